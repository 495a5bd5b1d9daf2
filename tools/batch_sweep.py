"""Throughput of the tcgen05 step against the batch (config-5 network, N = 80):
path-steps/s and ms per step from CUDA events, one line per batch."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_11623_b200 import BSDE  # noqa: E402

for B in (16384, 65536, 131072, 262144, 524288, 1048576):
    s = BSDE("allen_cahn", 100, 80, 0.3, 110, B, precision="bf16", lr=5e-4)
    for _ in range(3):
        s.train_step(sync=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s.stream)
    for _ in range(5):
        s.train_step(sync=False)
    e1.record(s.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print("B %8d  %7.3f ms/step  %.3e path-steps/s  tiles/SM %.1f" % (B, ms, B * 80 / ms * 1e3,
                                                                       B / 128 / 148), flush=True)
    s.close()
