"""clock64() phase trace of CTA 0 of the tcgen05 forward / adjoint kernels on the
config-5 workload (tc_fwd.cuh / tc_bwd.cuh CLK points), cycles per phase.
The stamps are compiled in only with -DBSDE_PHASE_CLOCKS:

    tools/build_variant.sh clocks -DBSDE_PHASE_CLOCKS
    BSDE_LIB=build_variants/clocks.so python tools/phase_clocks.py

Forward: worker warp 0 stamps slots 0-9 of a step row, the control warp 12-14
(see tc_fwd.cuh); adjoint: slots 0-10 of an item row.

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
    if which == 0:
        # worker warp 0: 0 step start | 1 slice 1 | 2 G1 waited | 3 E1 | 4 slice 2 | 5 G2 waited
        # | 6 E2 | 7 slice 3 | 8 G3 waited | 9 E3 + X̃_{n+1};  control: 12 B_X, 13 B_E1, 14 B_E2
        p = np.array(rows[2:40])
        tot = np.diff(p[:, 0])
        d = np.diff(p[:, :10], axis=1).mean(0)
        print("%s: %d traced, mean cycles %.0f" % (name, len(rows), tot.mean()))
        print("  worker: S1 %d  waitG1 %d  E1 %d  S2 %d  waitG2 %d  E2 %d  S3 %d  waitG3 %d  E3 %d" % tuple(d))
        print("  control (from worker step start): B_X %.0f  B_E1 %.0f  B_E2 %.0f"
              % tuple((p[:, j] - p[:, 0]).mean() for j in (12, 13, 14)))
        if p[:, 10].any():
            print("  E1 loads %.0f | E3: loads+sums %.0f  part %.0f  X~ put %.0f"
                  % ((p[:, 15] - p[:, 2]).mean(), (p[:, 10] - p[:, 8]).mean(), (p[:, 11] - p[:, 10]).mean(),
                     (p[:, 9] - p[:, 11]).mean()))
        continue
    lim = 12
    npts = max(int(np.max(np.nonzero(r[:lim])[0])) + 1 for r in rows)
    d = np.array([np.diff(r[:npts]) for r in rows[2:40]])
    tot = np.array([rows[i + 1][0] - rows[i][0] for i in range(2, min(40, len(rows) - 1))])
    print("%s: %d traced, mean cycles %.0f" % (name, len(rows), tot.mean()))
    print("  phase deltas:", " ".join("%d" % x for x in d.mean(0)))
