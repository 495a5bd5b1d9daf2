"""End-to-end training of the BASELINE configs on the GPU: Y0 and the loss after
each config's iteration budget, against the reference values of SURVEY Appendix A
(Allen-Cahn u(0,0) ≈ 0.05278-0.05282, HJB Cole-Hopf 4.590162, heat 2dT = 20).

    python tools/train_configs.py [cfg3_allen_cahn cfg5_allen_cahn_scaleout ...]
Prints one JSON line per config (wall time includes host loss reads every 100 steps).
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from workloads import CONFIGS  # noqa: E402

REF = {"heat": 20.0, "hjb": 4.590161724605, "allen_cahn": 0.0528151,
       "black_scholes": None}

names = sys.argv[1:] or ["cfg1_heat", "cfg2_hjb", "cfg3_allen_cahn", "cfg5_allen_cahn_scaleout"]
from paper_1910_11623_b200 import BSDE  # noqa: E402

for name in names:
    wl = CONFIGS[name]
    s = BSDE(wl.problem, wl.d, wl.N, wl.T, wl.w, wl.batch, lr=wl.lr, precision=wl.precision,
             seed=wl.seed, x0=wl.x0)
    t0 = time.time()
    curve = []
    for k in range(wl.iterations):
        if k % 100 == 0 or k == wl.iterations - 1:
            curve.append((k, s.train_step(), s.y0()))
        else:
            s.train_step(sync=False)
    s.stream.synchronize()
    y0 = s.y0()
    ref = REF[wl.problem] if wl.problem != "black_scholes" else 1.2336780599567434
    print(json.dumps({"config": name, "kernel": s.family, "iterations": wl.iterations,
                      "seconds": time.time() - t0, "y0": y0, "reference_u0": ref,
                      "rel_err": (y0 - ref) / ref, "final_loss": curve[-1][1],
                      "curve": [[k, l, y] for k, l, y in curve[:: max(1, len(curve) // 10)]]}),
          flush=True)
    s.close()
