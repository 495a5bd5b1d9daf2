"""The fp32-accurate tcgen05 family ("tc32": bf16x3 row GEMMs, rows_tc.cu, DESIGN
R18b) against the float64 oracle at the north-star fp32 tolerance 1e-4 (loss, Y0,
per-tensor gradients, R19), with the kink band of its ~2^-16 product precision.
Configs 1, 2, 4 (BASELINE.json fp32 configs) and the other problems, ragged sizes,
coupled multilevel paths, evaluation and Adam.
"""
import numpy as np
import pytest

from oracle import bsde as ob, philox
from parity_util import KINK_BAND, compare_grads, oracle_iteration
from workloads import CONFIGS

pytestmark = pytest.mark.gpu
TOL = 1e-4
BAND = KINK_BAND["fp32x3"]


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1910_11623_b200 import build
    build.build()


def make(problem, d, w, N, T, batch, **kw):
    from paper_1910_11623_b200 import BSDE
    kw.setdefault("kernel", "tc")
    return BSDE(problem, d, N, T, w, batch, precision="fp32", **kw)


CASES = [
    ("cfg1_heat", dict()),
    ("cfg2_hjb", dict(batch=1000)),
    ("cfg3_allen_cahn", dict(batch=1000, precision="fp32")),
    ("cfg4_hjb_multilevel", dict(batch=1000)),
    ("cfg2_hjb", dict(batch=300, N=3, d=37, w=45)),       # odd sizes, ragged row tile
    ("nx3_black_scholes", dict(batch=1000, precision="fp32")),
    ("nx3_black_scholes", dict(batch=129, N=3, d=7, w=9, x0=1.3, precision="fp32")),
]


@pytest.mark.parametrize("cfg,over", CASES, ids=[c + str(sorted(o.items())) for c, o in CASES])
def test_tc32_teacher_forced_iteration(cfg, over):
    wl = CONFIGS[cfg].with_(**over)
    s = make(wl.problem, wl.d, wl.w, wl.N, wl.T, wl.batch, lr=wl.lr, seed=wl.seed, x0=wl.x0)
    assert s.family == "tc32"
    p = s.get_params()
    scale = 0.003 if wl.problem == "allen_cahn" else 0.02
    p[1:] += (scale * np.random.default_rng(1).standard_normal(p.size - 1)).astype(np.float32)
    s.set_params(p)
    for it in (0, 7):
        s.iteration = it
        loss = s.compute_grad()
        g = s.get_grads()
        ref = oracle_iteration(wl.problem, wl.d, wl.w, wl.N, wl.T, p, wl.seed, it,
                               np.arange(wl.batch), wl.batch, x0=wl.x0, kink_band=BAND)
        assert abs(loss - ref["loss"]) <= TOL * ref["loss"], (loss, ref["loss"])
        compare_grads(g, ref["grad"], wl.d, wl.w, wl.N, TOL, ref["slack"],
                      step0_shared_x0=wl.x0 != 0.0)
        R = s.debug_residuals(0, wl.batch)
        assert np.max(np.abs(R - ref["R"])) <= TOL * np.max(np.abs(ref["R"]))
    # Adam (a8) on the gradient this step used
    s.train_step()
    st = ob.AdamState(p.size)
    q = p.astype(np.float64)
    ob.adam_step(q, s.get_grads().astype(np.float64), st, wl.lr)
    assert np.max(np.abs(s.get_params() - q)) <= 1e-5 * wl.lr + 1e-6 * np.max(np.abs(q))


def test_tc32_full_size_cfg2():
    """Config 2 at its full 16 384 paths, N = 20, in bench.py's launch configuration."""
    from parity_util import oracle_iteration_chunked
    wl = CONFIGS["cfg2_hjb"]
    s = make(wl.problem, wl.d, wl.w, wl.N, wl.T, wl.batch, lr=wl.lr, kernel="auto")
    assert s.family == "tc32"
    p = s.get_params()
    p[1:] += (0.02 * np.random.default_rng(3).standard_normal(p.size - 1)).astype(np.float32)
    s.set_params(p)
    s.iteration = 11
    loss = s.compute_grad()
    ref = oracle_iteration_chunked(wl.problem, wl.d, wl.w, wl.N, wl.T, p, 0, 11,
                                   np.arange(wl.batch), wl.batch, kink_band=BAND)
    assert abs(loss - ref["loss"]) <= TOL * ref["loss"]
    compare_grads(s.get_grads(), ref["grad"], wl.d, wl.w, wl.N, TOL, ref["slack"])


def test_tc32_full_size_cfg4():
    """Config 4's finest level at full size (65 536 paths, N = 80: 5.2 M rows) on tc32:
    (a) in bench_multilevel's launch configuration, residuals of sampled paths against
    the oracle path by path and the loss as the mean of all device residuals; (b) the
    gradient of one 1/64 shard of the same global batch (fake world: paths
    [17·1024, 18·1024), 1/B_global normalisation) against the oracle on those paths."""
    wl = CONFIGS["cfg4_hjb_multilevel"].with_(N=80)
    s = make(wl.problem, wl.d, wl.w, wl.N, wl.T, wl.batch, lr=wl.lr, kernel="auto")
    assert s.family == "tc32"
    p = s.get_params()
    p[1:] += (0.02 * np.random.default_rng(9).standard_normal(p.size - 1)).astype(np.float32)
    s.set_params(p)
    s.iteration = 5
    loss = s.compute_grad()
    assert np.isfinite(loss) and np.all(np.isfinite(s.get_grads()))
    idx = np.sort(np.random.default_rng(4).choice(wl.batch, 48, replace=False))
    ref = oracle_iteration(wl.problem, wl.d, wl.w, wl.N, wl.T, p, 0, 5, idx, wl.batch,
                           want_grad=False)
    R = np.array([s.debug_residuals(int(i), 1)[0] for i in idx])
    assert np.max(np.abs(R - ref["R"])) <= TOL * np.max(np.abs(ref["R"]))
    Rall = s.debug_residuals(0, wl.batch).astype(np.float64)
    assert abs(np.mean(Rall ** 2) - loss) <= 1e-5 * loss
    s.close()
    world, rank = 64, 17
    sh = make(wl.problem, wl.d, wl.w, wl.N, wl.T, wl.batch, lr=wl.lr, world=world, rank=rank)
    sh.set_params(p)
    sh.iteration = 5
    ls = sh.compute_grad()
    m0 = rank * (wl.batch // world)
    ref = oracle_iteration(wl.problem, wl.d, wl.w, wl.N, wl.T, p, 0, 5,
                           np.arange(m0, m0 + wl.batch // world), wl.batch, kink_band=BAND)
    assert abs(ls - ref["loss"]) <= TOL * ref["loss"], (ls, ref["loss"])
    compare_grads(sh.get_grads(), ref["grad"], wl.d, wl.w, wl.N, TOL, ref["slack"])


def test_tc32_fake_world_shards_sum():
    """Two ragged shards (300 paths each: two 128-row tiles and a 44-row tail, global
    path offsets m0 = 0, 300) of a 600-path batch add up to the full context's loss and
    gradient (§8(e)), through the tile-image buffers."""
    d, w, N, T, B = 100, 110, 4, 1.0, 600
    full = make("hjb", d, w, N, T, B)
    p = full.get_params()
    p[1:] += (0.02 * np.random.default_rng(12).standard_normal(p.size - 1)).astype(np.float32)
    full.set_params(p)
    lf = full.compute_grad()
    gf = full.get_grads().astype(np.float64)
    parts = [make("hjb", d, w, N, T, B, rank=r, world=2) for r in range(2)]
    for pt in parts:
        pt.set_params(p)
    ls = sum(pt.compute_grad() for pt in parts)
    gs = sum(pt.get_grads().astype(np.float64) for pt in parts)
    assert abs(ls - lf) <= 1e-6 * lf
    assert np.linalg.norm(gs - gf) <= 1e-5 * np.linalg.norm(gf)


def test_tc32_matches_simt_kernels():
    """Same parameters and paths on the FFMA kernels and the bf16x3 tensor-core rows:
    losses to 1e-5, gradients within the parity bound of each other."""
    d, w, N, T, B = 100, 110, 4, 1.0, 777
    a = make("hjb", d, w, N, T, B, kernel="simt")
    b = make("hjb", d, w, N, T, B)
    p = a.get_params()
    p[1:] += (0.02 * np.random.default_rng(5).standard_normal(p.size - 1)).astype(np.float32)
    a.set_params(p)
    b.set_params(p)
    la, lb = a.compute_grad(), b.compute_grad()
    assert abs(la - lb) <= 1e-5 * la
    ref = oracle_iteration("hjb", d, w, N, T, p, 0, 0, np.arange(B), B, kink_band=BAND)
    compare_grads(b.get_grads(), ref["grad"], d, w, N, TOL, ref["slack"])
    compare_grads(a.get_grads(), ref["grad"], d, w, N, TOL, ref["slack"])


def test_tc32_coupled_multilevel_matches_oracle():
    """Config-4 style schedule with coupled paths (NEXT-3) on tc32: N = 4 -> 8 -> 16,
    teacher-forced at each level (copy prolongation, R14)."""
    d, w, N, T, B = 100, 110, 4, 1.0, 500
    s = make("hjb", d, w, N, T, B, max_levels=2, coupled_paths=True)
    for level in range(3):
        if level:
            s.prolongate(level)
        p = s.get_params()
        p[1:] += (0.02 * np.random.default_rng(level).standard_normal(p.size - 1)).astype(np.float32)
        s.set_params(p)
        loss = s.compute_grad()
        ref = oracle_iteration("hjb", d, w, s.N, T, p, 0, s.iteration, np.arange(B), B,
                               kink_band=BAND, coupled_factor=16 // s.N)
        assert abs(loss - ref["loss"]) <= TOL * ref["loss"], (level, loss, ref["loss"])
        compare_grads(s.get_grads(), ref["grad"], d, w, s.N, TOL, ref["slack"])
        s.train_step()


def test_tc32_eval_loss_in_chunks():
    """bsde_eval_loss on a batch larger than the training batch (three row chunks)."""
    d, w, N, T = 100, 110, 3, 1.0
    s = make("hjb", d, w, N, T, 256)
    p = s.get_params()
    got = s.eval_loss(4, 700)
    ref = oracle_iteration("hjb", d, w, N, T, p, 0, philox.EVAL_BIT | 4, np.arange(700), 700,
                           want_grad=False)
    assert abs(got - ref["loss"]) <= TOL * ref["loss"]


def test_tc32_training_descends_and_graph_replays():
    """Config 2 shape, 30 Adam iterations through the captured CUDA graph: finite,
    decreasing, and identical to an eager (no-graph) context step for step."""
    wl = CONFIGS["cfg2_hjb"].with_(batch=4096, N=5)
    a = make(wl.problem, wl.d, wl.w, wl.N, wl.T, wl.batch, lr=wl.lr, use_graph=True)
    b = make(wl.problem, wl.d, wl.w, wl.N, wl.T, wl.batch, lr=wl.lr, use_graph=False)
    la = [a.train_step() for _ in range(30)]
    lb = [b.train_step() for _ in range(30)]
    assert np.all(np.isfinite(la)) and np.mean(la[-5:]) < np.mean(la[:5])
    assert np.allclose(la, lb, rtol=1e-4)
