"""Run a few training steps of a workload (for ncu / compute-sanitizer captures).

    python tools/prof_step.py [workload] [steps] [batch]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1910_11623_b200 import BSDE  # noqa: E402
from workloads import CONFIGS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5_allen_cahn_scaleout"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
wl = CONFIGS[name]
if len(sys.argv) > 3:
    wl = wl.with_(batch=int(sys.argv[3]))
s = BSDE(wl.problem, wl.d, wl.N, wl.T, wl.w, wl.batch, lr=wl.lr, precision=wl.precision,
         x0=wl.x0, seed=wl.seed)
for _ in range(steps):
    print(s.train_step())
s.close()
