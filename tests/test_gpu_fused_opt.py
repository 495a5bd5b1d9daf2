"""NEXT-4 (BASELINE north_star (e)): the reduce-scatter +
sharded Adam + all-gather as one peer-memory kernel (fused_opt.cu).  Only one GPU is
available to the tests: at world = 1 the kernel's peers are the context itself, and it
must reproduce the collective-free step and the NCCL sharded form bit for bit (same
fixed-order gradient, same Adam arithmetic).  World >= 2 over NVLink is not exercised
here."""
import numpy as np
import pytest

from workloads import CONFIGS

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1910_11623_b200 import build
    build.build()


def make(kernel, precision, **kw):
    from paper_1910_11623_b200 import BSDE
    wl = CONFIGS["cfg3_allen_cahn"].with_(batch=1024, N=3)
    return BSDE(wl.problem, wl.d, wl.N, wl.T, wl.w, wl.batch, lr=wl.lr, precision=precision,
                kernel=kernel, deterministic=True, **kw)


@pytest.mark.parametrize("kernel,precision", [("tc", "bf16"), ("simt", "fp32")])
def test_fused_optimizer_world1_is_bit_exact(kernel, precision):
    from paper_1910_11623_b200 import nccl_unique_id
    ref = make(kernel, precision)
    fus = make(kernel, precision)
    fus.enable_fused_optimizer()
    sh = make(kernel, precision, nccl_id=nccl_unique_id(), world=1, rank=0, sharded_adam=True)
    p = ref.get_params()
    for s in (fus, sh):
        s.set_params(p)
    for _ in range(4):
        la, lb, lc = ref.train_step(), fus.train_step(), sh.train_step()
        assert la == lb == lc
    assert np.array_equal(ref.get_params(), fus.get_params())
    assert np.array_equal(sh.get_params(), fus.get_params())
    ma, va, ta = ref.get_adam_state()
    mb, vb, tb = fus.get_adam_state()
    assert ta == tb == 4 and np.array_equal(ma, mb) and np.array_equal(va, vb)
    assert fus.iteration == ref.iteration == 4


def test_fused_optimizer_skips_a_diverged_step():
    """The divergence guard inside the fused kernel: a non-finite loss leaves
    parameters and Adam state untouched and raises EDIVERGED, like the unfused step."""
    from paper_1910_11623_b200 import BSDEError
    s = make("tc", "bf16")
    s.enable_fused_optimizer()
    p = s.get_params()
    p[0] = np.float32(1e30)    # Y0 -> R ~ 1e30 -> loss > 1e12
    s.set_params(p)
    with pytest.raises(BSDEError):
        s.train_step()
    assert np.array_equal(s.get_params(), p)
    m, v, t = s.get_adam_state()
    assert t == 0 and not m.any() and not v.any()
