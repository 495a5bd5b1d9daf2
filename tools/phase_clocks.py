"""clock64() phase trace of CTA 0 of the tcgen05 forward / adjoint kernels on the
config-5 workload (tc_fwd.cuh / tc_bwd.cuh CLK points), cycles per phase.
The stamps are compiled in only with -DBSDE_PHASE_CLOCKS:

    tools/build_variant.sh clocks -DBSDE_PHASE_CLOCKS
    BSDE_LIB=build_variants/clocks.so python tools/phase_clocks.py

Slots 0-7 of a row: consumer / adjoint phases; slots 8-11: forward producer
(8 before the empty wait, 9 after it, 10 slot filled).

    python tools/phase_clocks.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_11623_b200 import BSDE  # noqa: E402

s = BSDE("allen_cahn", 100, 80, 0.3, 110, 524288, precision="bf16", lr=5e-4)
for _ in range(3):
    try:
        s.train_step()
    except Exception as e:   # experiment builds may diverge (timing only)
        print("train_step:", str(e)[:80])
for which, name in ((0, "fwd (per step)"), (1, "bwd (per item)")):
    c = s.debug_phase_clocks(which, 1024).astype(np.int64).reshape(-1, 16)
    rows = [r for r in c if r[0] != 0]
    lim = 8 if which == 0 else 12
    npts = max(int(np.max(np.nonzero(r[:lim])[0])) + 1 for r in rows)
    d = np.array([np.diff(r[:npts]) for r in rows[2:40]])
    tot = np.array([rows[i + 1][0] - rows[i][0] for i in range(2, min(40, len(rows) - 1))])
    print("%s: %d traced, mean cycles %.0f" % (name, len(rows), tot.mean()))
    print("  phase deltas:", " ".join("%d" % x for x in d.mean(0)))
    if which == 0 and c[2:40, 8].any():
        p = c[2:40]
        print("  producer: wait-empty %.0f  fill %.0f  period %.0f  (fill start - consumer step start %.0f)"
              % ((p[:, 9] - p[:, 8]).mean(), (p[:, 10] - p[:, 9]).mean(),
                 np.diff(p[:, 8]).mean(), (p[:, 9] - p[:, 0]).mean()))
    if False:
        p = c[2:40].astype(np.int64)
        base = p[:, 8]
        print("  issuer (from I0 start): " + " ".join("%d" % (p[:, j] - base).mean() for j in range(9, 16))
              + "  | epilogue CLK0 %d" % (p[:, 0] - base).mean())
    if which == 0 and c[2:40, 12].any():
        p = c[2:40]
        print("  issuer: G2 seen %.0f, W2 reload issued %.0f, E2 done %.0f, barrier passed %.0f | others: G2 seen %.0f, E2 barrier issued %.0f"
              % ((p[:, 12] - p[:, 0]).mean(), (p[:, 13] - p[:, 0]).mean(), (p[:, 14] - p[:, 0]).mean(),
                 (p[:, 15] - p[:, 0]).mean(), (p[:, 3] - p[:, 0]).mean(), (p[:, 4] - p[:, 0]).mean()))
