"""The paper's own formulation on the GPU (shared.cu) against
oracle/shared.py: one tanh network u(t, x) for all steps, Eq. 6 residual loss,
reverse-over-reverse gradient.  fp32 kernels: north-star tolerance 1e-4."""
import numpy as np
import pytest

from oracle import bsde as ob, philox, shared as osh
from parity_util import PROBLEM

pytestmark = pytest.mark.gpu
TOL = 1e-4


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1910_11623_b200 import build
    build.build()


def make(problem, d, w, L, N, T, B, **kw):
    from paper_1910_11623_b200 import BSDE
    return BSDE(problem, d, N, T, w, B, formulation="shared", layers=L, **kw)


def perturb(s, seed, scale=0.05):
    p = s.get_params()
    p += (scale * np.random.default_rng(seed).standard_normal(p.size)).astype(np.float32)
    s.set_params(p)
    return p


def check_grad(g, ref, tol=TOL):
    err = np.linalg.norm(g - ref) / np.linalg.norm(ref)
    assert err <= tol, err
    assert np.max(np.abs(g - ref)) <= 4 * tol * np.max(np.abs(ref))


def test_init_matches_oracle():
    d, w, L = 10, 32, 3
    s = make("heat", d, w, L, 4, 1.0, 64, seed=5)
    assert s.family == "shared-simt" and s.num_params() == osh.num_params(d, w, L)
    ref = osh.init_params(5, d, w, L)
    assert np.max(np.abs(s.get_params() - ref)) <= 1e-6 * np.max(np.abs(ref))


CASES = [("heat", "fc", 0.0), ("hjb", "fc", 0.0), ("allen_cahn", "fc", 0.0),
         ("black_scholes", "fc", 0.5), ("hjb", "resnet", 0.0), ("black_scholes", "resnet", 0.5),
         ("hjb", "nais", 0.0), ("black_scholes", "nais", 0.5), ("allen_cahn", "nais", 0.0)]
ARCH = {"fc": osh.FC, "resnet": osh.RESNET, "nais": osh.NAIS}


@pytest.mark.parametrize("problem,arch,x0", CASES)
def test_teacher_forced_gradient(problem, arch, x0):
    """Loss and the full reverse-over-reverse gradient at a perturbed parameter
    point, ragged sizes (d + 1 = 38 inputs, 101 paths, 6 steps)."""
    d, w, L, N, T, B = 37, 48, 3, 6, 0.5, 101
    s = make(problem, d, w, L, N, T, B, arch=arch, x0=x0, lr=1e-3)
    p = perturb(s, 1)
    for it in (0, 4):
        s.iteration = it
        loss = s.compute_grad()
        ref = osh.iteration(PROBLEM[problem], d, w, L, ARCH[arch],
                            N, T, p.astype(np.float64), 0, it, np.arange(B), B, x0=x0)
        assert abs(loss - ref["loss"]) <= TOL * ref["loss"], (loss, ref["loss"])
        check_grad(s.get_grads(), ref["grad"])
        R = s.debug_residuals(0, B)
        assert np.max(np.abs(R - ref["r"][N])) <= TOL * np.max(np.abs(ref["r"][N]))


def test_paper_workload_gradient_adam_and_y0():
    """The paper's Table 1 workload: Black-Scholes d = 100, M = 100
    paths, N = 50 steps, 4 tanh layers of 256, Adam lr 1e-3; X_0 = 0.1·1 (R21)."""
    d, w, L, N, T, B, x0 = 100, 256, 4, 50, 1.0, 100, 0.1
    s = make("black_scholes", d, w, L, N, T, B, x0=x0, lr=1e-3)
    p = s.get_params().astype(np.float64)
    loss = s.compute_grad()
    ref = osh.iteration(ob.BLACK_SCHOLES, d, w, L, osh.FC, N, T, p, 0, 0, np.arange(B), B, x0=x0)
    assert abs(loss - ref["loss"]) <= TOL * ref["loss"]
    g = s.get_grads()
    check_grad(g, ref["grad"])
    assert abs(s.y0() - osh.u0(p, d, w, L, osh.FC, x0)) <= 1e-5
    # one Adam step from these gradients
    s.train_step()
    st = ob.AdamState(p.size)
    q = p.copy()
    ob.adam_step(q, s.get_grads().astype(np.float64), st, 1e-3)
    assert np.max(np.abs(s.get_params() - q)) <= 1e-8 + 1e-6 * np.max(np.abs(q))


def test_prolongate_keeps_network_and_doubles_steps():
    d, w, L, N, T, B = 8, 32, 2, 3, 1.0, 64
    s = make("hjb", d, w, L, N, T, B, max_levels=2)
    p = perturb(s, 3)
    s.train_step()
    q = s.get_params()
    s.prolongate(1)
    assert s.N == 2 * N and np.array_equal(s.get_params(), q)
    m, v, t = s.get_adam_state()
    assert t == 0 and not m.any() and not v.any()
    loss = s.compute_grad()
    ref = osh.iteration(ob.HJB, d, w, L, osh.FC, 2 * N, T, q.astype(np.float64), 0, s.iteration,
                        np.arange(B), B)
    assert abs(loss - ref["loss"]) <= TOL * ref["loss"]
    check_grad(s.get_grads(), ref["grad"])


def test_coupled_paths_shared():
    """Coupled multilevel paths (R22) with the shared network: level N = 2 of a
    N_fine = 8 grid uses sums of 4 fine increments."""
    d, w, L, N, T, B = 6, 16, 2, 2, 1.0, 50
    s = make("black_scholes", d, w, L, N, T, B, max_levels=2, coupled_paths=True, x0=0.8)
    p = perturb(s, 4)
    loss = s.compute_grad()
    # the oracle's shared iteration with coupled increments: rebuild its paths
    m = np.arange(B)
    X = [np.full((B, d), 0.8)]
    for n in range(N):
        X.append(ob.forward_step(ob.BLACK_SCHOLES, X[-1],
                                 philox.coupled_increments(0, 0, n, m, d, T / N, 4)))
    R = s.debug_residuals(0, B)
    u_N = osh.forward(p.astype(np.float64), d, w, L, osh.FC, np.full(B, T), X[N])[0]
    assert np.max(np.abs(R - (u_N - np.sum(X[N] ** 2, axis=1)))) <= 1e-4 * np.max(np.abs(R))
    assert np.isfinite(loss)


def test_eval_loss_matches_oracle():
    d, w, L, N, T = 12, 32, 3, 4, 0.3
    s = make("allen_cahn", d, w, L, N, T, 64)   # eval batch 200 runs in chunks of 64 paths
    p = perturb(s, 2).astype(np.float64)
    got = s.eval_loss(3, 200)
    ref = osh.iteration(ob.ALLEN_CAHN, d, w, L, osh.FC, N, T, p, 0, philox.EVAL_BIT | 3,
                        np.arange(200), 200, want_grad=False)
    assert abs(got - ref["loss"]) <= TOL * ref["loss"]


def test_training_descends():
    """Black-Scholes d = 100 with the paper's network: 300 Adam steps (lr 1e-3) on
    the shared formulation reduce the loss several-fold."""
    s = make("black_scholes", 100, 256, 4, 20, 1.0, 256, x0=0.1, lr=1e-3)
    losses = [s.train_step() for _ in range(300)]
    assert np.all(np.isfinite(losses))
    assert np.mean(losses[-20:]) < 0.2 * np.mean(losses[:5])


def test_nais_init_adam_projection_and_y0():
    """NAIS-Net shared network (R26): init = oracle init (projected R_k), one Adam
    step = oracle Adam + projection, Y0 = u(0, X_0) with the A_k of the
    current parameters."""
    d, w, L, N, T, B = 10, 32, 3, 4, 1.0, 64
    s = make("hjb", d, w, L, N, T, B, arch="nais", lr=0.05, seed=2)
    assert s.num_params() == osh.num_params(d, w, L, osh.NAIS)
    p = s.get_params().astype(np.float64)
    ref = osh.init_params(2, d, w, L, osh.NAIS)
    assert np.max(np.abs(p - ref)) <= 2e-6 * np.max(np.abs(ref))
    s.train_step()
    q = p.copy()
    ob.adam_step(q, s.get_grads().astype(np.float64), ob.AdamState(p.size), 0.05)
    osh.project(q, d, w, L, osh.NAIS)
    got = s.get_params()
    assert np.max(np.abs(got - q)) <= 1e-5 * np.max(np.abs(q))
    assert abs(s.y0() - osh.u0(got.astype(np.float64), d, w, L, osh.NAIS, 0.0)) <= 1e-5


@pytest.mark.parametrize("arch", ["fc", "nais"])
def test_fake_world_shards_sum(arch):
    """Data-parallel sharding (§8(e)): two rank contexts without a communicator
    ("fake world") own global paths [0, B/2) and [B/2, B); their local losses and
    gradients sum to the single-context ones."""
    d, w, L, N, T, B = 12, 32, 3, 4, 1.0, 128
    full = make("hjb", d, w, L, N, T, B, arch=arch)
    lf = full.compute_grad()
    gf = full.get_grads().astype(np.float64)
    parts = [make("hjb", d, w, L, N, T, B, arch=arch, rank=r, world=2) for r in range(2)]
    ls = sum(pt.compute_grad() for pt in parts)
    gs = sum(pt.get_grads().astype(np.float64) for pt in parts)
    assert abs(ls - lf) <= 1e-5 * lf
    assert np.linalg.norm(gs - gf) <= 1e-5 * np.linalg.norm(gf)


@pytest.mark.parametrize("problem,arch,x0", [("black_scholes", "fc", 0.5), ("hjb", "resnet", 0.0),
                                             ("allen_cahn", "fc", 0.0)])
def test_bf16_tensor_core_gradient(problem, arch, x0):
    """precision="bf16": the row GEMMs (forward, ∇ₓu, and the reverse-over-reverse
    δ̄ / h̄ products) run on tcgen05 with bf16 operands and fp32 TMEM accumulation;
    the weight-gradient GEMMs stay fp32.  North-star bf16 tolerance 2e-2 against
    the float64 oracle; ragged rows (R = 7·101) and d + 1 = 38 inputs."""
    d, w, L, N, T, B = 37, 64, 3, 6, 0.5, 101
    s = make(problem, d, w, L, N, T, B, arch=arch, x0=x0, lr=1e-3, precision="bf16")
    assert s.family == "shared-tc"
    p = perturb(s, 1)
    loss = s.compute_grad()
    ref = osh.iteration(PROBLEM[problem], d, w, L, ARCH[arch], N, T, p.astype(np.float64), 0, 0,
                        np.arange(B), B, x0=x0)
    assert abs(loss - ref["loss"]) <= 2e-2 * ref["loss"], (loss, ref["loss"])
    check_grad(s.get_grads(), ref["grad"], tol=2e-2)


def test_bf16_tensor_core_paper_workload():
    """The paper's Table 1 workload with bf16 tcgen05 row GEMMs (4×256, M = 100,
    N = 50, BS d = 100): loss and gradient within 2e-2 of the oracle."""
    d, w, L, N, T, B, x0 = 100, 256, 4, 50, 1.0, 100, 0.1
    s = make("black_scholes", d, w, L, N, T, B, x0=x0, lr=1e-3, precision="bf16")
    p = s.get_params().astype(np.float64)
    loss = s.compute_grad()
    ref = osh.iteration(ob.BLACK_SCHOLES, d, w, L, osh.FC, N, T, p, 0, 0, np.arange(B), B, x0=x0)
    assert abs(loss - ref["loss"]) <= 2e-2 * ref["loss"]
    check_grad(s.get_grads(), ref["grad"], tol=2e-2)


@pytest.mark.parametrize("problem", ["black_scholes", "hjb", "allen_cahn"])
def test_zN_term_matches_oracle(problem):
    """The optional Σ|∇ₓu(t_N, X_N) - ∇g(X_N)|² term of P:79 (R27, cfg.shared_zN)."""
    d, w, L, N, T, B, x0 = 12, 32, 3, 4, 0.5, 101, (0.5 if problem == "black_scholes" else 0.0)
    s = make(problem, d, w, L, N, T, B, x0=x0, zN=True)
    p = perturb(s, 6)
    loss = s.compute_grad()
    ref = osh.iteration(PROBLEM[problem], d, w, L, osh.FC, N, T, p.astype(np.float64), 0, 0,
                        np.arange(B), B, x0=x0, zN=True)
    assert abs(loss - ref["loss"]) <= TOL * ref["loss"], (loss, ref["loss"])
    check_grad(s.get_grads(), ref["grad"])


def test_bf16_tensor_core_weight_gradients_large_rows():
    """R ≥ 32 768 rows: the weight-gradient GEMMs also run on tcgen05 (split over
    row ranges, MN-major bf16 images).  Loss and gradient vs the oracle at 2e-2 on
    sampled sizes: d = 20, w = 64, L = 3, N = 8, M = 4 000 (36 000 rows)."""
    d, w, L, N, T, B = 20, 64, 3, 8, 1.0, 4000
    s = make("hjb", d, w, L, N, T, B, precision="bf16", lr=1e-3)
    p = perturb(s, 8)
    loss = s.compute_grad()
    ref = osh.iteration(ob.HJB, d, w, L, osh.FC, N, T, p.astype(np.float64), 0, 0, np.arange(B), B)
    assert abs(loss - ref["loss"]) <= 2e-2 * ref["loss"]
    check_grad(s.get_grads(), ref["grad"], tol=2e-2)
