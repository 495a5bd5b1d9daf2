"""Shared-network (paper's own) formulation: per-iteration time and time-to-solution."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1910_11623_b200 import BSDE

def timed(s, iters):
    st = s.stream
    for _ in range(5):
        s.train_step(sync=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(iters):
        s.train_step(sync=False)
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters

u0 = np.exp(0.21) * 100 * 0.01
for M, N in ((100, 50), (1000, 50), (4096, 50)):
    s = BSDE("black_scholes", 100, N, 1.0, 256, M, formulation="shared", layers=4, x0=0.1, lr=1e-3)
    ms = timed(s, 50)
    print("M %5d N %d: %.3f ms/iter  %.3e path-steps/s  launches %d" % (M, N, ms, M * N / ms * 1e3, s.launches_per_step()), flush=True)
# the paper's run: 20000 iterations, M=100, N=50, lr 1e-3
s = BSDE("black_scholes", 100, 50, 1.0, 256, 100, formulation="shared", layers=4, x0=0.1, lr=1e-3)
t0 = time.time()
hist = []
for k in range(20000):
    if k % 2000 == 0 or k == 19999:
        l = s.train_step()
        hist.append((k, l, s.y0()))
    else:
        s.train_step(sync=False)
torch.cuda.synchronize()
print("20000 iterations: %.1f s wall" % (time.time() - t0))
for k, l, y in hist:
    print("  it %5d loss %.3e Y0 %.5f (rel %.4f)" % (k, l, y, y / u0 - 1))
