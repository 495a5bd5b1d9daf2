"""Black-Scholes workload: Y0 trajectory under training (tc bf16 and simt fp32)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from workloads import CONFIGS
from paper_1910_11623_b200 import BSDE
wl = CONFIGS["nx3_black_scholes"]
u0 = np.exp((0.05 + 0.16) * wl.T) * wl.d * wl.x0 ** 2
print("closed form u0", u0)
for kern, prec, B, lr in (("tc", "bf16", 65536, 1e-2), ("tc", "bf16", 16384, 1e-2), ("simt", "fp32", 16384, 1e-2)):
    s = BSDE(wl.problem, wl.d, wl.N, wl.T, wl.w, B, lr=lr, precision=prec, kernel=kern, x0=wl.x0)
    t0 = time.time()
    for k in range(1501):
        l = s.train_step()
        if k % 100 == 0:
            print(kern, prec, B, k, "loss %.5f Y0 %.5f rel %.4f" % (l, s.y0(), s.y0() / u0 - 1), flush=True)
    print("time", time.time() - t0)
