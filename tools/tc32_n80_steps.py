"""Three eager training steps of config 4's finest grid (HJB d = 100, N = 80,
B = 65 536, fp32-accurate tc32 kernels), for an ncu launch list:

    ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file launches.csv python tools/tc32_n80_steps.py
"""
import sys
sys.path.insert(0, '.')
from paper_1910_11623_b200 import BSDE
s = BSDE("hjb", 100, 80, 1.0, 110, 65536, precision="fp32", lr=1e-2, use_graph=False)
for _ in range(3):
    s.train_step()
