"""GPU ↔ oracle parity through the C-ABI (libbsde.so), DESIGN.md §Parity.

All inputs are seeded and synthetic (Philox counters); sizes span several tiles
and a ragged tail.  Tolerances: north_star (1e-4 fp32, 2e-2 bf16).
"""
import numpy as np
import pytest

from oracle import bsde as ob, closed_forms as cf, philox
from parity_util import (KINK_BAND, TOL, band_of, check_tc_against_emulation, compare_grads,
                         oracle_iteration)
from workloads import CONFIGS

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1910_11623_b200 import build
    build.build()


def make(problem, d, w, N, T, batch, **kw):
    from paper_1910_11623_b200 import BSDE
    return BSDE(problem, d, N, T, w, batch, **kw)


# ------------------------------------------------------------------ a1: Philox
def test_philox_bit_exact_on_device():
    s = make("heat", 4, 8, 2, 1.0, 64, kernel="simt")
    rng = np.random.default_rng(0)
    ctr = rng.integers(0, 2 ** 32, size=(4096, 4), dtype=np.uint64).astype(np.uint32)
    for key in ([0, 0], [0xDEADBEEF, 0x12345678]):
        out = s.debug_philox(ctr, np.array(key, np.uint32))
        ref = np.stack(philox.philox4x32_10(ctr[:, 0], ctr[:, 1], ctr[:, 2], ctr[:, 3], *key), 1)
        assert np.array_equal(out, ref)


@pytest.mark.parametrize("d,N,T", [(100, 20, 1.0), (10, 5, 1.0), (7, 3, 0.3)])
def test_dw_matches_oracle(d, N, T):
    s = make("hjb", d, 8, N, T, 64, kernel="simt", seed=0x1234567890ABCDEF)
    for it, n, m0 in ((0, 0, 0), (17, N - 1, 1000), (2 ** 31 - 1, 1, 2 ** 32 - 300)):
        gpu = s.debug_dw(it, n, m0, 257)
        ref = philox.brownian_increments(0x1234567890ABCDEF, it, n, np.arange(m0, m0 + 257), d,
                                         T / N)
        assert np.max(np.abs(gpu - ref)) <= 2e-6 * np.sqrt(T / N) * 6


@pytest.mark.parametrize("problem", ["hjb", "allen_cahn"])
def test_init_matches_oracle(problem):
    d, w, N = 100, 110, 3
    s = make(problem, d, w, N, 1.0, 64, kernel="simt", seed=5)
    p = s.get_params()
    ref = ob.init_params(5, d, w, N, zero_head=(problem == "allen_cahn"))
    assert np.max(np.abs(p - ref)) <= 1e-6 * np.max(np.abs(ref))


# ------------------------------------------------------------------ a2-a6 teacher-forced
CASES = [
    # (config, overrides)
    ("cfg1_heat", dict()),
    ("cfg2_hjb", dict(batch=1000)),
    ("cfg3_allen_cahn", dict(batch=1000, precision="fp32")),
    ("cfg4_hjb_multilevel", dict(batch=1000)),
    ("cfg2_hjb", dict(batch=300, N=3, d=37, w=45)),       # odd sizes, ragged tiles
    ("nx3_black_scholes", dict(batch=1000, precision="fp32")),
    ("nx3_black_scholes", dict(batch=300, N=3, d=37, w=45, x0=1.3, precision="fp32")),
]


@pytest.mark.parametrize("cfg,over", CASES, ids=[c + str(sorted(o.items())) for c, o in CASES])
@pytest.mark.parametrize("kernel", ["simt"])
def test_teacher_forced_iteration(cfg, over, kernel):
    wl = CONFIGS[cfg].with_(**over)
    tol = TOL[wl.precision]
    s = make(wl.problem, wl.d, wl.w, wl.N, wl.T, wl.batch, lr=wl.lr, precision=wl.precision,
             kernel=kernel, seed=wl.seed, x0=wl.x0)
    # move away from the zero-bias init so every tensor has a gradient (smaller
    # for Allen-Cahn, whose cubic driver explodes for a large Z, R7b)
    p = s.get_params()
    rng = np.random.default_rng(1)
    scale = 0.003 if wl.problem == "allen_cahn" else 0.02
    p[1:] += (scale * rng.standard_normal(p.size - 1)).astype(np.float32)
    s.set_params(p)
    for it in (0, 7):
        s.iteration = it
        loss = s.compute_grad()
        g = s.get_grads()
        ref = oracle_iteration(wl.problem, wl.d, wl.w, wl.N, wl.T, p, wl.seed, it,
                               np.arange(wl.batch), wl.batch, x0=wl.x0,
                               kink_band=KINK_BAND[wl.precision])
        assert np.isfinite(ref["loss"])
        assert abs(loss - ref["loss"]) <= tol * ref["loss"], (loss, ref["loss"])
        compare_grads(g, ref["grad"], wl.d, wl.w, wl.N, tol, ref["slack"])
    # Adam (a8): the step recomputes the same gradient (same it) and applies Adam
    loss2 = s.train_step()
    assert loss2 == pytest.approx(loss, rel=1e-6)
    g2 = s.get_grads()          # the gradient this step used (atomic order may differ)
    assert np.linalg.norm(g2 - g) <= 1e-5 * np.linalg.norm(g)
    st = ob.AdamState(p.size)
    q = p.astype(np.float64)
    ob.adam_step(q, g2.astype(np.float64), st, wl.lr)
    got = s.get_params()
    assert np.max(np.abs(got - q)) <= 1e-5 * wl.lr + 1e-6 * np.max(np.abs(q))
    m, v, t = s.get_adam_state()
    assert t == 1 and np.allclose(m, st.m, rtol=1e-5, atol=1e-6 * np.abs(st.m).max())
    assert s.iteration == 8


def test_full_size_cfg2_gradient_and_sampled_residuals():
    """Config 2 at its full batch (16384 paths, N = 20), launch as bench.py times it."""
    wl = CONFIGS["cfg2_hjb"]
    s = make(wl.problem, wl.d, wl.w, wl.N, wl.T, wl.batch, lr=wl.lr)
    p = s.get_params()
    loss = s.compute_grad()
    ref = oracle_iteration(wl.problem, wl.d, wl.w, wl.N, wl.T, p, 0, 0, np.arange(wl.batch),
                           wl.batch, kink_band=band_of(s))
    assert abs(loss - ref["loss"]) <= 1e-4 * ref["loss"]
    compare_grads(s.get_grads(), ref["grad"], wl.d, wl.w, wl.N, 1e-4, ref["slack"])
    idx = np.random.default_rng(3).choice(wl.batch, 64, replace=False)
    R = np.array([s.debug_residuals(int(i), 1)[0] for i in idx])
    assert np.allclose(R, ref["R"][idx], rtol=1e-4, atol=1e-4 * np.abs(ref["R"]).max())


def test_heat_optimum_identity_on_gpu():
    """Pin H1 on the device: at the exact optimum R = 2dT - 2Σ|ΔW|² per path."""
    d, T, N, B = 10, 1.0, 5, 256
    p, w = cf.heat_optimum_params(d, T, N)
    s = make("heat", d, w, N, T, B, kernel="simt")
    s.set_params(p.astype(np.float32))
    loss = s.compute_grad()
    R = s.debug_residuals(0, B)
    S = sum(np.sum(s.debug_dw(0, n, 0, B).astype(np.float64) ** 2, 1) for n in range(N))
    assert np.max(np.abs(R - (2 * d * T - 2 * S))) < 2e-4
    assert abs(loss - np.mean(R.astype(np.float64) ** 2)) < 1e-4 * loss


def test_cfg1_trajectory():
    """Config 1 end to end: 200 Adam iterations through the C-ABI (CUDA graph
    replay), teacher-forced parity at it = 50 and 199 and the free-running
    trajectory against the oracle's own 200 iterations (R19)."""
    wl = CONFIGS["cfg1_heat"]
    s = make(wl.problem, wl.d, wl.w, wl.N, wl.T, wl.batch, lr=wl.lr)
    p0 = s.get_params().astype(np.float64)
    losses = []
    for k in range(wl.iterations):
        if k in (50, 199):
            pk = s.get_params()
            lk = s.compute_grad()
            ref = oracle_iteration(wl.problem, wl.d, wl.w, wl.N, wl.T, pk, 0, k,
                                   np.arange(wl.batch), wl.batch, kink_band=band_of(s))
            assert abs(lk - ref["loss"]) <= 1e-4 * ref["loss"]
            compare_grads(s.get_grads(), ref["grad"], wl.d, wl.w, wl.N, 1e-4, ref["slack"])
        losses.append(s.train_step())
    po, _, lo = ob.train(ob.HEAT, wl.d, wl.w, wl.N, wl.T, p0.copy(), 0, wl.batch, wl.iterations,
                         wl.lr)
    assert abs(s.y0() - po[0]) <= 1e-3 * abs(po[0])
    assert np.allclose(losses[:20], lo[:20], rtol=1e-4)
    assert abs(np.mean(losses[-10:]) - np.mean(lo[-10:])) <= 1e-2 * np.mean(lo[-10:])


# ------------------------------------------------------------------ a9, eval, guards
@pytest.mark.parametrize("mode", ["copy", "interp"])
def test_prolongate_matches_oracle(mode):
    d, w, N = 6, 9, 5
    s = make("hjb", d, w, N, 1.0, 64, kernel="simt", max_levels=2, prolong=mode)
    s.train_step()
    p = s.get_params()
    s.prolongate(1)
    q = s.get_params()
    ref = ob.prolongate(p.astype(np.float64), d, w, N, ob.COPY if mode == "copy" else ob.INTERP)
    assert s.N == 2 * N and q.size == ref.size
    if mode == "copy":
        assert np.array_equal(q, ref.astype(np.float32))
    else:
        assert np.allclose(q, ref, rtol=1e-6, atol=1e-7)
    m, v, t = s.get_adam_state()
    assert t == 0 and not m.any() and not v.any()
    it = s.iteration
    loss = s.compute_grad()
    r = oracle_iteration("hjb", d, w, 2 * N, 1.0, q, 0, it, np.arange(64), 64)
    assert abs(loss - r["loss"]) <= 1e-4 * r["loss"]
    with pytest.raises(Exception):
        s.prolongate(3)


@pytest.mark.parametrize("mode,kernel", [("copy", "simt"), ("interp", "simt"), ("copy", "tc")])
def test_prolongate_keep_adam_matches_oracle(mode, kernel):
    """R14b (BSDE_PROLONG_KEEP_ADAM): the Adam moments follow the parameters'
    prolongation on the device (oracle.prolongate_adam of the pre-change state), t is
    kept, and the next update is Adam from that state (teacher-forced on the
    context's own gradient)."""
    d, w, N, B = (10, 20, 5, 64) if kernel == "tc" else (6, 9, 5, 64)   # tc: a built shape
    prec = "bf16" if kernel == "tc" else "fp32"
    s = make("hjb", d, w, N, 1.0, B, kernel=kernel, precision=prec, max_levels=2, prolong=mode,
             keep_adam=True)
    for _ in range(3):
        s.train_step()
    m, v, t = s.get_adam_state()
    s.prolongate(1)
    om = ob.COPY if mode == "copy" else ob.INTERP
    st = ob.AdamState(m.size)
    st.m, st.v, st.t = m.astype(np.float64), v.astype(np.float64), t
    ref = ob.prolongate_adam(st, d, w, N, om)
    m2, v2, t2 = s.get_adam_state()
    assert t2 == t == 3 and m2.size == ref.m.size
    if mode == "copy":
        assert np.array_equal(m2, ref.m.astype(np.float32)) and np.array_equal(v2, ref.v.astype(np.float32))
    else:
        assert np.allclose(m2, ref.m, rtol=1e-6, atol=1e-12) and np.allclose(v2, ref.v, rtol=1e-6, atol=1e-15)
    q = s.get_params().astype(np.float64)
    s.train_step()
    g = s.get_grads().astype(np.float64)
    st2 = ob.AdamState(q.size)
    st2.m, st2.v, st2.t = m2.astype(np.float64), v2.astype(np.float64), t2
    assert ob.adam_step(q, g, st2, 1e-2)
    got = s.get_params()
    assert np.allclose(got, q, rtol=0, atol=2e-6), np.abs(got - q).max()
    assert s.get_adam_state()[2] == t2 + 1


@pytest.mark.parametrize("keep", [False, True])
def test_multilevel_schedule_matches_oracle(keep):
    """The multilevel schedule end to end through the C-ABI (run_schedule: train
    steps, bsde_prolongate between levels N = 2 -> 4 -> 8) against the oracle's
    train_multilevel with the same Adam rule at the level changes (R14 reset or
    R14b kept): the per-iteration losses and the final parameters."""
    from paper_1910_11623_b200.multilevel import run_schedule
    d, w, B, T, iters = 6, 9, 64, 1.0, [6, 6, 4]
    s = make("hjb", d, w, 2, T, B, kernel="simt", max_levels=2, keep_adam=keep)
    p0 = s.get_params().astype(np.float64)
    res = run_schedule(s, iters, eval_every=0)
    pr, hist = ob.train_multilevel(ob.HJB, d, w, [2, 4, 8], T, p0.copy(), 0, B, iters, 1e-2,
                                   keep_adam=keep)
    got = np.array([r.train_loss for r in res.records])
    ref = np.array([h[2] for h in hist])
    assert np.allclose(got, ref, rtol=1e-4), np.abs(got / ref - 1).max()
    q = s.get_params().astype(np.float64)
    assert np.linalg.norm(q - pr) <= 1e-4 * np.linalg.norm(pr)
    assert s.get_adam_state()[2] == (sum(iters) if keep else iters[-1])


@pytest.mark.parametrize("problem,x0", [("hjb", 0.0), ("black_scholes", 0.7)])
def test_coupled_paths_match_oracle(problem, x0):
    """Coupled multilevel paths (NEXT-3): at every level of N = 5 -> 10 -> 20 the
    increments are sums of the N = 20 grid's (factor 4, 2, 1); teacher-forced
    loss and gradient against the oracle with the same coupling."""
    d, w, N, T, B = 12, 16, 5, 1.0, 200
    s = make(problem, d, w, N, T, B, kernel="simt", max_levels=2, coupled_paths=True, x0=x0)
    for level in range(3):
        if level:
            s.prolongate(level)
        p = s.get_params()
        p[1:] += (0.02 * np.random.default_rng(level).standard_normal(p.size - 1)).astype(np.float32)
        s.set_params(p)
        loss = s.compute_grad()
        ref = oracle_iteration(problem, d, w, s.N, T, p, 0, s.iteration, np.arange(B), B, x0=x0,
                               kink_band=KINK_BAND["fp32"], coupled_factor=20 // s.N)
        assert abs(loss - ref["loss"]) <= 1e-4 * ref["loss"], (level, loss, ref["loss"])
        compare_grads(s.get_grads(), ref["grad"], d, w, s.N, 1e-4, ref["slack"])
        s.train_step()


def test_coupled_paths_share_terminal_state_on_gpu():
    """Heat with Z ≡ 0: Y_N = Y0 and X_N = √2 W_T, so coupled levels give the same
    residuals (pin C2 of the oracle, on the device)."""
    d, w, N, T, B = 10, 20, 4, 1.0, 256
    s = make("heat", d, w, N, T, B, kernel="simt", max_levels=2, coupled_paths=True,
             zero_head=True)
    s.compute_grad()
    R0 = s.debug_residuals(0, B)
    for level in (1, 2):
        s.prolongate(level)
        s.compute_grad()
        assert np.max(np.abs(s.debug_residuals(0, B) - R0)) <= 1e-5 * np.max(np.abs(R0))


def test_eval_loss_matches_oracle():
    d, w, N, T = 20, 24, 4, 0.3
    s = make("allen_cahn", d, w, N, T, 128, kernel="simt")
    p = s.get_params()
    for eid, batch in ((0, 500), (3, 128)):
        got = s.eval_loss(eid, batch)
        ref = oracle_iteration("allen_cahn", d, w, N, T, p, 0, philox.EVAL_BIT | eid,
                               np.arange(batch), batch, want_grad=False)
        assert abs(got - ref["loss"]) <= 1e-5 * ref["loss"]


def test_divergence_guard_skips_update():
    from paper_1910_11623_b200 import BSDEError
    s = make("heat", 4, 8, 2, 1.0, 64, kernel="simt")
    p = s.get_params()
    p[0] = 3e6          # loss ≈ 9e12 > 1e12
    s.set_params(p)
    with pytest.raises(BSDEError) as e:
        s.train_step()
    assert e.value.code == -4
    assert np.array_equal(s.get_params(), p)


def test_fake_world_shards_sum_to_full_batch():
    """§8(e)/H10: rank r of G owns global paths [rB/G, (r+1)B/G); the shard
    gradients (no collective) sum to the single-rank gradient."""
    d, w, N, T, B = 12, 16, 4, 1.0, 512
    full = make("hjb", d, w, N, T, B, kernel="simt")
    lf = full.compute_grad()
    gf = full.get_grads().astype(np.float64)
    parts = [make("hjb", d, w, N, T, B, kernel="simt", rank=r, world=4) for r in range(4)]
    ls = sum(pt.compute_grad() for pt in parts)
    gs = sum(pt.get_grads().astype(np.float64) for pt in parts)
    assert abs(ls - lf) <= 1e-6 * lf
    assert np.linalg.norm(gs - gf) <= 1e-5 * np.linalg.norm(gf)


def test_graph_replay_equals_eager():
    a = make("allen_cahn", 16, 20, 4, 0.3, 300, kernel="simt", use_graph=True)
    b = make("allen_cahn", 16, 20, 4, 0.3, 300, kernel="simt", use_graph=False)
    la = [a.train_step() for _ in range(5)]
    lb = [b.train_step() for _ in range(5)]
    assert np.allclose(la, lb, rtol=1e-6)
    assert np.allclose(a.get_params(), b.get_params(), rtol=1e-5, atol=1e-7)


def test_torch_workspace_context_matches_own_allocations():
    """cfg.workspace: a context carved from a torch tensor of
    bsde_workspace_bytes() trains exactly like one with its own allocations."""
    import torch
    from paper_1910_11623_b200.solver import workspace_bytes
    d, w, N, B = 12, 16, 3, 128
    nbytes = workspace_bytes("hjb", d, N, w, B, kernel="simt")
    ws = torch.empty(nbytes + 256, dtype=torch.uint8, device="cuda")
    off = (-ws.data_ptr()) % 256
    view = ws[off:off + nbytes]
    a = make("hjb", d, w, N, 1.0, B, kernel="simt")
    b = make("hjb", d, w, N, 1.0, B, kernel="simt", workspace=view)
    for _ in range(3):
        assert a.train_step() == b.train_step()
    assert np.array_equal(a.get_params(), b.get_params())
    small = ws[off:off + nbytes // 2]
    with pytest.raises(Exception):
        make("hjb", d, w, N, 1.0, B, kernel="simt", workspace=small)


@pytest.mark.parametrize("kernel,problem,d,w,N,B", [
    ("simt", "heat", 1, 1, 1, 1),          # every dimension at its minimum
    ("simt", "hjb", 3, 2, 1, 65),          # one step, a 1-path ragged tail after a full tile
    ("tc", "allen_cahn", 100, 110, 1, 1),  # one path in a 128-row tcgen05 tile, one step
    ("tc", "hjb", 37, 45, 2, 129),         # ragged tail of one path, odd d and w
])
def test_degenerate_shapes(kernel, problem, d, w, N, B):
    """Edge cases: minimal sizes, single step, single path, one-path ragged tails."""
    prec = "bf16" if kernel == "tc" else "fp32"
    T = 0.3 if problem == "allen_cahn" else 1.0
    s = make(problem, d, w, N, T, B, kernel=kernel, precision=prec)
    p = s.get_params()
    p[1:] += (0.01 * np.random.default_rng(9).standard_normal(p.size - 1)).astype(np.float32)
    s.set_params(p)
    loss = s.compute_grad()
    ref = oracle_iteration(problem, d, w, N, T, p, 0, 0, np.arange(B), B,
                           kink_band=KINK_BAND[prec])
    tol = TOL[prec]
    assert abs(loss - ref["loss"]) <= tol * ref["loss"], (loss, ref["loss"])
    compare_grads(s.get_grads(), ref["grad"], d, w, N, tol, ref["slack"],
                  max_slack_share=None if prec == "bf16" else 0.1)
    if kernel == "tc":
        emu = oracle_iteration(problem, d, w, N, T, p, 0, 0, np.arange(B), B,
                               kink_band=KINK_BAND["fp32"], tc=True)
        check_tc_against_emulation(loss, s.get_grads(), None, emu, d, w, N)
    assert np.isfinite(s.train_step())
    with pytest.raises(Exception):
        make(problem, d, w, N, T, 0, kernel=kernel, precision=prec)   # empty batch: EINVAL
