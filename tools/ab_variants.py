"""A/B timing of experiment builds (tools/build_variant.sh) on the config-5 workload:
each variant runs in its own process (BSDE_LIB=build_variants/NAME.so), the order
alternating over the repeats; prints the best forward / adjoint / step ms of each.

    python tools/ab_variants.py base new [--reps 3] [--workload cfg2_hjb --precision fp32]
"""
import argparse
import os
import subprocess
import sys

CODE = r'''
import sys
sys.path.insert(0, %r)
from paper_1910_11623_b200 import BSDE
from workloads import CONFIGS
wl = CONFIGS[%r]
if %r: wl = wl.with_(N=%r)
s = BSDE(wl.problem, wl.d, wl.N, wl.T, wl.w, wl.batch, lr=wl.lr, precision=%r, kernel=%r)
for _ in range(3):
    try: s.train_step()
    except Exception: pass
r = [s.profile_steps(5) for _ in range(3)]
print("%%.4f %%.4f %%.4f" %% (min(x["fwd"] for x in r), min(x["bwd"] for x in r), min(sum(x.values()) for x in r)))
'''

ap = argparse.ArgumentParser()
ap.add_argument("variants", nargs="+")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--workload", default="cfg5_allen_cahn_scaleout")
ap.add_argument("--precision", default="bf16")
ap.add_argument("--kernel", default="auto")
ap.add_argument("--N", type=int, default=0, help="override the workload's number of steps")
args = ap.parse_args()
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
res = {v: [] for v in args.variants}
for rep in range(args.reps):
    for v in (args.variants if rep % 2 == 0 else args.variants[::-1]):
        env = dict(os.environ, BSDE_LIB=os.path.join(root, "build_variants", v + ".so"))
        r = subprocess.run([sys.executable, "-c", CODE % (root, args.workload, args.N, args.N, args.precision, args.kernel)], env=env, capture_output=True, text=True)
        try:
            res[v].append([float(x) for x in r.stdout.split()])
        except ValueError:
            print(v, "failed:", r.stderr[-400:])
for v, xs in res.items():
    xs = [x for x in xs if len(x) == 3]
    if xs:
        print("%-12s fwd %.3f  bwd %.3f  step %.3f   (best of %d; fwd runs %s; bwd runs %s)"
              % (v, min(x[0] for x in xs), min(x[1] for x in xs), min(x[2] for x in xs), len(xs),
                 " ".join("%.3f" % x[0] for x in xs), " ".join("%.3f" % x[1] for x in xs)))
