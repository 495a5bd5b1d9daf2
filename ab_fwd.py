import os, sys, subprocess
code = r'''
from paper_1910_11623_b200 import BSDE
from workloads import CONFIGS
wl = CONFIGS["cfg5_allen_cahn_scaleout"]
s = BSDE(wl.problem, wl.d, wl.N, wl.T, wl.w, wl.batch, lr=wl.lr, precision="bf16")
for _ in range(3): s.train_step()
r = [s.profile_steps(5) for _ in range(3)]
print("%.3f" % min(x["fwd"] for x in r))
'''
res = {"cur": [], "alt": []}
for rep in range(5):
    for v in (("cur", "alt") if rep % 2 == 0 else ("alt", "cur")):
        env = dict(os.environ, BSDE_LIB="build_variants/%s.so" % v)
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True).stdout.strip()
        res[v].append(float(out))
for k, v in res.items(): print(k, "mean %.3f min %.3f" % (sum(v) / len(v), min(v)), v)
