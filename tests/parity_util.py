"""Helpers shared by the GPU parity tests (test-side: may import the oracle)."""
import numpy as np

from oracle import bsde as ob

PROBLEM = dict(ob.PROBLEM_NAMES)

# north_star: "GPU losses, Y0 and gradients must match the oracle to relative 1e-4
# (fp32) or 2e-2 (bf16 operands with fp32 accumulate)"
TOL = {"fp32": 1e-4, "bf16": 2e-2}


def tensor_slices(d, w, N, nais=False):
    """(name, slice) of every parameter tensor in the flat layout (NAIS-Net: the
    W2/b2 slots hold R/C and B (w×d) follows b3, R25)."""
    out = [("Y0", slice(0, 1))]
    off = 1
    for n in range(N):
        tensors = [("W1", w * d), ("b1", w), ("W2", w * w), ("b2", w), ("W3", d * w), ("b3", d)]
        if nais:
            tensors.append(("B", w * d))
        for name, size in tensors:
            out.append(("%s_%d" % (name, n), slice(off, off + size)))
            off += size
    return out


# Width of the band around the ReLU kink in which a finite-precision evaluation
# of the pre-activation may land on either side (R15/R19): relative to Σ|W x|+|b|.
KINK_BAND = {"fp32": 2e-6, "bf16": 8e-3}


def oracle_iteration(problem, d, w, N, T, params, seed, it, paths, batch, x0=0.0, lam=1.0,
                     want_grad=True, kink_band=0.0, coupled_factor=1):
    return ob.iteration(PROBLEM[problem], d, w, N, T, np.asarray(params, np.float64), seed, it,
                        np.asarray(paths), batch, x0=x0, lam=lam, want_grad=want_grad,
                        kink_band=kink_band, coupled_factor=coupled_factor)


def compare_grads(g_gpu, g_orc, d, w, N, tol, slack=None, nais=False):
    """R19: per tensor ‖Δ‖₂/‖g‖₂ ≤ tol and max|Δ| ≤ 4·tol·max|g|, where Δ is the
    GPU-oracle difference beyond the kink slack (both ReLU masks are valid for a
    pre-activation inside the rounding band).  Returns the worst relative L2
    error; raises AssertionError naming the tensor."""
    worst = 0.0
    for name, sl in tensor_slices(d, w, N, nais):
        a = np.asarray(g_gpu[sl], np.float64)
        b = np.asarray(g_orc[sl], np.float64)
        s = 0.0 if slack is None else np.asarray(slack[sl], np.float64)
        diff = np.maximum(np.abs(a - b) - s, 0.0)
        nb = np.linalg.norm(b)
        if nb == 0.0:
            assert np.all(diff <= 1e-30), (name, "oracle gradient is exactly 0")
            continue
        rel = np.linalg.norm(diff) / nb
        worst = max(worst, rel)
        assert rel <= tol, (name, rel)
        assert np.max(diff) <= tol * np.max(np.abs(b)) * 4, (name, np.max(diff))
    return worst
