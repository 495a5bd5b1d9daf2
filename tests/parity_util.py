"""Helpers shared by the GPU parity tests (test-side: may import the oracle)."""
import os

import numpy as np

from oracle import bsde as ob

PROBLEM = dict(ob.PROBLEM_NAMES)

# north_star: "GPU losses, Y0 and gradients must match the oracle to relative 1e-4
# (fp32) or 2e-2 (bf16 operands with fp32 accumulate)"
TOL = {"fp32": 1e-4, "bf16": 2e-2}
# The tensor-core path against the oracle's evaluation of the same roundings
# (R17: bf16 operands incl. the folded biases, bf16 H1 and residual
# sum, binary16 ΔW_n).  What is left is fp32 accumulation order and the device
# normals' ~1e-6 relative error (fast Box-Muller, R8), which move an operand
# across a bf16 rounding boundary now and then; downstream of such a flip a
# ReLU mask can change sign, so the tensors whose gradient goes through a mask
# (W1, b1, W2, b2 at n >= 1) carry that noise (measured on the B200, up to
# 7e-3 relative L2 at config-5 size, profiles/r02_parity_stats.txt).
# Everything else (loss, Y0, W3, b3, the constant-input step n = 0) has no mask
# flips: measured <= 1.4e-3.  A 5% error in any tensor fails either bound.  A flip
# moves one path's share of a sum over the batch, so the masked bound grows as
# √(1000/B) below 1000 paths.
TOL_TC_EMU = 2e-3            # loss/R bound is TOL_TC_LOSS; mask-free tensors
TOL_TC_EMU_STEP0 = 4e-3      # n = 0 tensors (sums over paths that nearly cancel)
TOL_TC_EMU_MASKED = 1.5e-2   # W1, b1, W2, b2 at n >= 1
TOL_TC_LOSS = 1e-4           # measured <= 5.4e-6
MASK_FREE = ("Y0", "W3", "b3")


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
# fp32: accumulation order of fp32 sums; bf16: bf16 operand rounding (used only
# against the exact oracle; against the tc emulation the operands are the same
# and the fp32 band applies).
# fp32x3: the fp32-accurate tcgen05 family ("tc32", bf16x3 operands, DESIGN R18b),
# whose products carry ~2^-16 relative error: a band ten times the fp32 one.
KINK_BAND = {"fp32": 2e-6, "bf16": 8e-3, "fp32x3": 2e-5}


def band_of(s, precision="fp32"):
    """The kink band R19 for a context's kernel family."""
    return KINK_BAND["fp32x3"] if s.family == "tc32" else KINK_BAND[precision]


def oracle_iteration(problem, d, w, N, T, params, seed, it, paths, batch, x0=0.0, lam=1.0,
                     want_grad=True, kink_band=0.0, coupled_factor=1, tc=False, kink_flip=0.0):
    return ob.iteration(PROBLEM[problem], d, w, N, T, np.asarray(params, np.float64), seed, it,
                        np.asarray(paths), batch, x0=x0, lam=lam, want_grad=want_grad,
                        kink_band=kink_band, coupled_factor=coupled_factor, tc=tc,
                        kink_flip=kink_flip)


def _chunk(args):
    kw, paths = args
    r = oracle_iteration(paths=paths, **kw)
    return r


def oracle_iteration_chunked(problem, d, w, N, T, params, seed, it, paths, batch,
                             chunk_path_steps=150000, workers=None, **kw):
    """oracle_iteration over ``paths`` in shards (the shard results add up, §8(e):
    loss_sum and gradient are sums over paths), in worker processes, so that
    full-size configurations fit in host memory and finish in tens of seconds."""
    import concurrent.futures as cf
    import multiprocessing as mp
    paths = np.asarray(paths)
    c = max(64, chunk_path_steps // N)
    parts = [paths[i:i + c] for i in range(0, paths.size, c)]
    base = dict(problem=problem, d=d, w=w, N=N, T=T, params=np.asarray(params, np.float64),
                seed=seed, it=it, batch=batch, **kw)
    workers = workers or min(len(parts), max(1, (os.cpu_count() or 2) // 2))
    if workers == 1:
        res = [_chunk((base, p)) for p in parts]
    else:
        with cf.ProcessPoolExecutor(workers, mp_context=mp.get_context("spawn"),
                                    initializer=_limit_threads) as ex:
            res = list(ex.map(_chunk, [(base, p) for p in parts]))
    out = dict(loss_sum=sum(r["loss_sum"] for r in res), R=np.concatenate([r["R"] for r in res]))
    out["loss"] = out["loss_sum"] / float(batch)
    for k in ("grad", "slack"):
        if k in res[0]:
            out[k] = sum(r[k] for r in res)
    return out


def _limit_threads():
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(2)
    except Exception:
        pass


def compare_grads(g_gpu, g_orc, d, w, N, tol, slack=None, nais=False, max_slack_share=0.1,
                  elem_tol=None, step0_shared_x0=False):
    """R19: per tensor ‖Δ‖₂/‖g‖₂ ≤ tol and max|Δ| ≤ tol·max|g|, where Δ is the
    GPU-oracle difference beyond the kink slack (both ReLU masks are valid for a
    pre-activation inside the rounding band).  max_slack_share bounds
    ‖slack‖/‖g‖ per tensor, so that the slack cannot hide a real error (None
    only for the secondary bf16-vs-exact checks, whose bf16-wide band is
    larger than some tensors: the binding bf16 check is the tc emulation).
    elem_tol (default tol) is the elementwise bound relative to max|g|.
    step0_shared_x0: X_0 = x0·1 with x0 != 0, so at n = 0 every path evaluates the
    same pre-activation and a unit inside the band flips for the whole batch; the
    slack-share cap then does not apply to the step-0 tensors (the slack still does).
    Returns the worst relative L2 error; raises AssertionError naming the tensor."""
    worst = 0.0
    elem_tol = tol if elem_tol is None else elem_tol
    for name, sl in tensor_slices(d, w, N, nais):
        a = np.asarray(g_gpu[sl], np.float64)
        b = np.asarray(g_orc[sl], np.float64)
        s = 0.0 if slack is None else np.asarray(slack[sl], np.float64)
        diff = np.maximum(np.abs(a - b) - s, 0.0)
        nb = np.linalg.norm(b)
        if nb == 0.0:
            assert np.all(diff <= 1e-30), (name, "oracle gradient is exactly 0")
            continue
        if max_slack_share is not None and slack is not None and not (
                step0_shared_x0 and name.endswith("_0")):
            share = np.linalg.norm(s) / nb
            assert share < max_slack_share, (name, "slack share", share)
        rel = np.linalg.norm(diff) / nb
        worst = max(worst, rel)
        assert rel <= tol, (name, rel)
        assert np.max(diff) <= elem_tol * np.max(np.abs(b)), (name, np.max(diff) / np.max(np.abs(b)))
    return worst


def check_tc_against_emulation(loss, g, R, ref, d, w, N, scale=1.0):
    """The binding bf16 check: GPU loss, residuals and gradient against the
    oracle's tensor-core rounding model (tc=True, fp32 kink band), per tensor:
    relative L2 beyond the slack (slack share < 0.1) within TOL_TC_EMU (mask-free
    tensors), TOL_TC_EMU_STEP0 (n = 0) or TOL_TC_EMU_MASKED (W1, b1, W2, b2);
    elementwise 5x those.  ``scale`` multiplies the bounds (mutation tests use
    it to show the margin)."""
    assert abs(loss - ref["loss"]) <= TOL_TC_LOSS * scale * ref["loss"], (loss, ref["loss"])
    # a mask flip moves one path's share of a sum over the batch: relative noise ~ 1/√B
    R_paths = len(ref["R"])
    if R is not None:
        err = np.max(np.abs(R - ref["R"])) / np.max(np.abs(ref["R"]))
        assert err <= TOL_TC_EMU * scale, ("R", err)
    worst = 0.0
    for name, sl in tensor_slices(d, w, N):
        fam, _, n = name.partition("_")
        tol = (TOL_TC_EMU if fam in MASK_FREE else
               TOL_TC_EMU_STEP0 if n == "0" else
               TOL_TC_EMU_MASKED * max(1.0, np.sqrt(1000.0 / R_paths))) * scale
        a = np.asarray(g[sl], np.float64)
        b = np.asarray(ref["grad"][sl], np.float64)
        s = np.asarray(ref["slack"][sl], np.float64)
        nb = np.linalg.norm(b)
        diff = np.maximum(np.abs(a - b) - s, 0.0)
        if nb == 0.0:
            assert np.all(diff <= 1e-30), (name, "oracle gradient is exactly 0")
            continue
        share = np.linalg.norm(s) / nb
        assert share < 0.1, (name, "slack share", share)
        rel = np.linalg.norm(diff) / nb
        worst = max(worst, rel / tol)
        assert rel <= tol, (name, rel, tol)
        assert np.max(diff) <= 5 * tol * np.max(np.abs(b)), (name, np.max(diff) / np.max(np.abs(b)))
    return worst
