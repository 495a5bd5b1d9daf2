"""Diagnostic (test-side): per-tensor statistics of the tcgen05 gradient against
the oracle's tensor-core rounding model, for calibrating the parity comparator.

    python tools/parity_stats.py [case ...]

Prints, per case and tensor family, the worst over steps n >= 1 (and n = 0
separately) of: relative L2 difference beyond the slack, elementwise difference
/ max|g|, and ‖slack‖/‖g‖, for the kink bands (fp32, flip 0) and (fp32, 2^-8).
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from parity_util import oracle_iteration_chunked, tensor_slices  # noqa: E402
from workloads import CONFIGS  # noqa: E402

CASES = {
    "cfg3_b1000": ("cfg3_allen_cahn", dict(batch=1000), 0.003, 0),
    "cfg3_b1000_it5": ("cfg3_allen_cahn", dict(batch=1000), 0.003, 5),
    "cfg2bf16_b1000": ("cfg2_hjb", dict(batch=1000, precision="bf16"), 0.02, 0),
    "cfg3_full": ("cfg3_allen_cahn", dict(), 0.003, 3),
    "cfg5_b16384": ("cfg5_allen_cahn_scaleout", dict(batch=16384), 0.003, 3),
}


def stats(g, ref, d, w, N):
    out = {}
    for name, sl in tensor_slices(d, w, N):
        if name == "Y0":
            continue
        fam, n = name.split("_")
        key = fam + ("0" if n == "0" else "")
        a = np.asarray(g[sl], np.float64)
        b = np.asarray(ref["grad"][sl], np.float64)
        s = np.asarray(ref["slack"][sl], np.float64)
        nb = np.linalg.norm(b)
        if nb == 0:
            continue
        diff = np.maximum(np.abs(a - b) - s, 0.0)
        r = (np.linalg.norm(diff) / nb, np.max(diff) / np.max(np.abs(b)), np.linalg.norm(s) / nb,
             np.linalg.norm(a - b) / nb)
        o = out.get(key, (0, 0, 0, 0))
        out[key] = tuple(max(x, y) for x, y in zip(o, r))
    return {k: ["%.2e" % x for x in v] for k, v in out.items()}


def main():
    from paper_1910_11623_b200 import BSDE
    names = sys.argv[1:] or list(CASES)
    for cname in names:
        cfg, over, scale, it = CASES[cname]
        wl = CONFIGS[cfg].with_(**over)
        s = BSDE(wl.problem, wl.d, wl.N, wl.T, wl.w, wl.batch, lr=wl.lr, precision="bf16", kernel="tc")
        p = s.get_params()
        p[1:] += (scale * np.random.default_rng(1).standard_normal(p.size - 1)).astype(np.float32)
        s.set_params(p)
        s.iteration = it
        loss = s.compute_grad()
        g = s.get_grads()
        for flip in (0.0, 2.0 ** -8):
            ref = oracle_iteration_chunked(wl.problem, wl.d, wl.w, wl.N, wl.T, p, 0, it,
                                           np.arange(wl.batch), wl.batch, kink_band=2e-6, tc=True,
                                           kink_flip=flip)
            print(json.dumps({"case": cname, "flip": flip, "loss_rel": abs(loss / ref["loss"] - 1),
                              "stats[l2,elem,slack,raw_l2]": stats(g, ref, wl.d, wl.w, wl.N)}),
                  flush=True)
        s.close()


if __name__ == "__main__":
    main()
