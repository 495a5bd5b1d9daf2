"""Per-tensor parity of the bf16 tcgen05 gradient against the oracle's tensor-core
emulation (tc=True, fp32 kink band) at larger N and small batches: prints the worst
tensors by elementwise error (max |diff| beyond the slack / max |ref|), their relative
L2 error and slack share.  Used to size tests/test_gpu_tc.py's cases: over 240 steps a
few masked tensors (W1, W2, b1, b2 of single steps) exceed the elementwise bound
whichever Philox path generated the increments.

    python tools/diag_parity_largeN.py      (GPU)
"""
import sys, numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from parity_util import *  # noqa
from test_gpu_tc import make, oracle_iteration, KINK_BAND, TOL
from workloads import CONFIGS
for N, B in ((240, 256), (240, 1024), (80, 256)):
    wl = CONFIGS["cfg5_allen_cahn_scaleout"].with_(batch=B, N=N)
    s = make(wl.problem, wl.d, wl.w, wl.N, wl.T, wl.batch, lr=wl.lr, precision="bf16", kernel="tc", seed=wl.seed, x0=wl.x0)
    p = s.get_params(); rng = np.random.default_rng(1)
    p[1:] += (0.003 * rng.standard_normal(p.size - 1)).astype(np.float32); s.set_params(p)
    s.iteration = 0
    loss = s.compute_grad(); g = s.get_grads()
    emu = oracle_iteration(wl.problem, wl.d, wl.w, wl.N, wl.T, p, wl.seed, 0, np.arange(B), B, x0=wl.x0, kink_band=KINK_BAND["fp32"], tc=True)
    rows = []
    for name, sl in tensor_slices(wl.d, wl.w, wl.N):
        a = np.asarray(g[sl], np.float64); b = np.asarray(emu["grad"][sl], np.float64); sk = np.asarray(emu["slack"][sl], np.float64)
        nb = np.linalg.norm(b)
        if nb == 0: continue
        diff = np.maximum(np.abs(a - b) - sk, 0.0)
        rows.append((name, np.linalg.norm(diff) / nb, np.max(diff) / np.max(np.abs(b)), np.linalg.norm(sk)/nb))
    rows.sort(key=lambda r: -r[2])
    print("N", N, "B", B, "loss", loss, emu["loss"])
    for r in rows[:8]: print("   %-8s rel %.2e  elem %.3f  slack %.2e" % r)
