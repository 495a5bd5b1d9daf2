import numpy as np, sys
sys.path.insert(0, '.')
from paper_1910_11623_b200 import BSDE
s = BSDE("allen_cahn", 100, 80, 0.3, 110, 524288, precision="bf16", lr=5e-4)
for _ in range(3): s.train_step()
for which, npts in ((0, 14), (1, 13)):
    c = s.debug_phase_clocks(which, 1024).astype(np.int64)
    rows = [r for r in c if r[0] != 0]
    d = np.array([np.diff(r[:npts]) for r in rows[2:40]])
    tot = np.array([rows[i + 1][0] - rows[i][0] for i in range(2, min(40, len(rows) - 1))])
    print("which", which, "steps", len(rows), "mean cycles per step/item", tot.mean())
    print("  phase deltas:", " ".join("%d" % x for x in d.mean(0)))
