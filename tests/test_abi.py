"""CPU checks of the boundary: libbsde.so builds for sm_100a, loads, and exports
every symbol include/bsde.h declares; argument validation without a GPU."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def libpath():
    from paper_1910_11623_b200 import build
    return build.build()


def header_symbols():
    src = open(os.path.join(ROOT, "include", "bsde.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bsde_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported(libpath):
    syms = header_symbols()
    assert len(syms) >= 20
    L = ctypes.CDLL(libpath)
    for s in syms:
        assert hasattr(L, s), s
    from paper_1910_11623_b200 import _lib
    assert sorted(_lib.SYMBOLS) == syms


def test_library_is_sm100a_and_uses_tensor_memory(libpath):
    out = subprocess.run(["cuobjdump", "--list-elf", libpath], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_config_struct_layout_matches_header(libpath):
    """The ctypes mirror of bsde_config has the C layout: defaults round-trip."""
    from paper_1910_11623_b200 import _lib
    cfg = _lib.Config()
    _lib.lib().bsde_config_default(ctypes.byref(cfg))
    assert cfg.batch_global == 256 and cfg.lam == 1.0 and cfg.lr == 1e-2
    assert cfg.beta1 == 0.9 and cfg.beta2 == 0.999 and cfg.eps == 1e-8
    assert cfg.world == 1 and cfg.rank == 0 and cfg.use_graph == 1 and cfg.kernel == 0


@pytest.mark.parametrize("kw,msg", [
    (dict(problem="heat", d=0), "d >= 1"),
    (dict(problem="heat", width=0), "widths"),
    (dict(problem="hjb", batch=10, world=3), "divisible"),
    (dict(problem="allen_cahn", kernel="simt", precision="bf16"), "bf16"),
])
def test_create_rejects_bad_arguments(libpath, kw, msg):
    """Validation happens before any device call, so it runs on the CPU box."""
    from paper_1910_11623_b200 import BSDE, BSDEError
    args = dict(problem="heat", d=4, N=2, T=1.0, width=8, batch=16)
    args.update(kw)
    world = args.pop("world", 1)
    with pytest.raises(BSDEError) as e:
        BSDE(args.pop("problem"), args.pop("d"), args.pop("N"), args.pop("T"), args.pop("width"),
             args.pop("batch"), world=world, stream=0, **args)
    assert msg in str(e.value) and e.value.code == -1


def test_workspace_bytes_without_gpu(libpath):
    """bsde_workspace_bytes: sizes a context with the create-time
    validation and no allocation, so it runs on the CPU box; it grows with the
    batch and the time grid and rejects what bsde_create rejects."""
    from paper_1910_11623_b200 import BSDEError
    from paper_1910_11623_b200.solver import workspace_bytes
    a = workspace_bytes("allen_cahn", 100, 80, 110, 524288, precision="bf16")
    b = workspace_bytes("allen_cahn", 100, 80, 110, 262144, precision="bf16")
    c = workspace_bytes("allen_cahn", 100, 40, 110, 524288, precision="bf16")
    assert a > b > 0 and a > c > 0
    # config 5 holds the X̃ and ΔW images: 2 × 224 B per path-step at least
    assert a >= 2 * 224 * 524288 * 80
    s = workspace_bytes("black_scholes", 100, 50, 256, 100, formulation="shared", layers=4)
    assert s > 0
    with pytest.raises(BSDEError):
        workspace_bytes("heat", 0, 2, 8, 16)
    # the shared net's activation rows are read as float4: a width not divisible by 4 is
    # refused at create time instead of misaligning the GEMM loads
    with pytest.raises(BSDEError, match="multiple of 4"):
        workspace_bytes("black_scholes", 100, 50, 30, 100, formulation="shared", layers=4)


def test_missing_library_fails_loudly(tmp_path):
    """No CPU fallback: without libbsde.so the binding refuses to construct a solver."""
    import subprocess
    import sys
    code = ("from paper_1910_11623_b200 import BSDE\n"
            "try:\n"
            "    BSDE('heat', 10, 5, 1.0, 20, 256)\n"
            "except ImportError as e:\n"
            "    print('raised:', e)\n")
    env = dict(os.environ, BSDE_LIB=str(tmp_path / "nope" / "libbsde.so"))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))), timeout=120)
    assert "raised:" in r.stdout and "no CPU fallback" in r.stdout, (r.stdout, r.stderr)
