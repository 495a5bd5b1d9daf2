"""The paper's Table 1 run (BS d = 100, M = 100, N = 50, 4 × 256, Adam 1e-3, 20 000
iterations) on the shared formulation: FC fp32, FC bf16 tcgen05, ResNet, NAIS-Net.
Y0 = u(0, X_0) against the closed form; wall time of the 20 000 iterations."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_11623_b200 import BSDE  # noqa: E402

u0 = float(np.exp(0.21) * 100 * 0.01)
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
for arch, prec in (("fc", "fp32"), ("fc", "bf16"), ("resnet", "fp32"), ("nais", "fp32")):
    s = BSDE("black_scholes", 100, 50, 1.0, 256, 100, formulation="shared", layers=4, arch=arch,
             precision=prec, x0=0.1, lr=1e-3)
    torch.cuda.synchronize()
    t0 = time.time()
    ys = []
    for k in range(iters):
        if k >= iters - 1000 and k % 100 == 0:
            s.train_step()
            ys.append(s.y0())
        else:
            s.train_step(sync=False)
    torch.cuda.synchronize()
    sec = time.time() - t0
    y = float(np.mean(ys))
    print(json.dumps({"arch": arch, "precision": prec, "iterations": iters, "seconds": sec,
                      "y0_mean_last_1000": y, "closed_form": u0, "rel_err": y / u0 - 1,
                      "eval_loss": s.eval_loss(7, 100)}), flush=True)
    s.close()
