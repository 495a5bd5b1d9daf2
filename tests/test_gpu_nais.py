"""NAIS-Net block in the per-step nets on the GPU
against oracle/nais.py: fp32 SIMT kernels, north-star tolerance 1e-4 (R19)."""
import numpy as np
import pytest

from oracle import bsde as ob, nais as onais
from parity_util import KINK_BAND, PROBLEM, compare_grads

pytestmark = pytest.mark.gpu
TOL = 1e-4


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1910_11623_b200 import build
    build.build()


def make(problem, d, w, N, T, B, **kw):
    from paper_1910_11623_b200 import BSDE
    return BSDE(problem, d, N, T, w, B, arch="nais", kernel="simt", **kw)


def test_init_matches_oracle_projected():
    d, w, N = 37, 45, 3
    s = make("hjb", d, w, N, 1.0, 64, seed=3)
    assert s.num_params() == onais.num_params(d, w, N)
    ref = onais.init_params(3, d, w, N)
    got = s.get_params()
    assert np.max(np.abs(got - ref)) <= 2e-6 * np.max(np.abs(ref))
    _, nets = onais.unpack(got.astype(np.float64), d, w, N)
    for net in nets:
        assert np.linalg.norm(net["R"].T @ net["R"]) <= 0.99 * (1 + 1e-5)


CASES = [("heat", 37, 45, 3, 300, 0.0), ("hjb", 37, 45, 3, 300, 0.0),
         ("allen_cahn", 37, 45, 3, 300, 0.0), ("black_scholes", 37, 45, 3, 300, 0.8),
         ("hjb", 100, 110, 20, 1000, 0.0)]


@pytest.mark.parametrize("problem,d,w,N,B,x0", CASES)
def test_teacher_forced_gradient(problem, d, w, N, B, x0):
    T = 0.3 if problem == "allen_cahn" else 1.0
    s = make(problem, d, w, N, T, B, x0=x0, lr=1e-3, zero_head=False)
    p = s.get_params()
    rng = np.random.default_rng(5)
    p[1:] += (0.01 * rng.standard_normal(p.size - 1)).astype(np.float32)
    s.set_params(p)
    for it in (0, 3):
        s.iteration = it
        loss = s.compute_grad()
        ref = onais.iteration(PROBLEM[problem], d, w, N, T, p.astype(np.float64), 0, it,
                              np.arange(B), B, x0=x0, kink_band=KINK_BAND["fp32"])
        assert abs(loss - ref["loss"]) <= TOL * ref["loss"], (loss, ref["loss"])
        compare_grads(s.get_grads(), ref["grad"], d, w, N, TOL, ref["slack"], nais=True)


def test_adam_step_projects_R():
    """One train step = oracle Adam on the device gradient followed by the
    projection of every R_n (R25); a large lr pushes R outside the ball."""
    d, w, N, B = 12, 20, 3, 128
    s = make("hjb", d, w, N, 1.0, B, lr=0.05)
    p = s.get_params().astype(np.float64)
    s.train_step()
    g = s.get_grads().astype(np.float64)
    st = ob.AdamState(p.size)
    q = p.copy()
    ob.adam_step(q, g, st, 0.05)
    _, before = onais.unpack(q.copy(), d, w, N)
    onais.project(q, d, w, N)
    got = s.get_params()
    assert np.max(np.abs(got - q)) <= 1e-5 * np.max(np.abs(q))
    assert any(np.linalg.norm(n["R"].T @ n["R"]) > 0.99 for n in before)   # the projection acted


def test_prolongate_matches_oracle():
    d, w, N, B = 10, 16, 2, 96
    s = make("allen_cahn", d, w, N, 0.3, B, max_levels=1, lr=1e-3)
    s.train_step()
    p = s.get_params().astype(np.float64)
    s.prolongate(1)
    q = s.get_params()
    ref = onais.prolongate(p, d, w, N, copy=True)
    assert np.array_equal(q, ref.astype(np.float32))
    loss = s.compute_grad()
    r = onais.iteration(ob.ALLEN_CAHN, d, w, 2 * N, 0.3, q.astype(np.float64), 0, s.iteration,
                        np.arange(B), B, kink_band=KINK_BAND["fp32"])
    assert abs(loss - r["loss"]) <= TOL * r["loss"]
    compare_grads(s.get_grads(), r["grad"], d, w, 2 * N, TOL, r["slack"], nais=True)


def test_nais_rejects_tensor_core_path():
    from paper_1910_11623_b200 import BSDE
    with pytest.raises(Exception):
        BSDE("hjb", 100, 4, 1.0, 110, 256, arch="nais", precision="bf16")
