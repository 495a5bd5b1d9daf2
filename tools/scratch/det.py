import sys, os, numpy as np
sys.path.insert(0, os.getcwd())
from paper_1910_11623_b200 import BSDE
s = BSDE("allen_cahn", 100, 4, 0.3, 110, 2048, precision="bf16", lr=5e-4)
for _ in range(2): s.train_step()
p = s.get_params()
res = []
for r in range(4):
    s.set_params(p); s.iteration = 5
    l = s.compute_grad(); g = s.get_grads().astype(np.float64); res.append((l, g))
g0 = res[0][1]
for l, g in res[1:]:
    d = np.abs(g - g0)
    print("loss diff", l - res[0][0], "max|dg|", d.max(), "max|g|", np.abs(g0).max(), "frac>1e-6*max", np.mean(d > 1e-6 * np.abs(g0).max()), "n_exact_diff", np.count_nonzero(d))
# per-tensor: where do diffs live
d, w, N = 100, 110, 4
P = 2*d*w + w*w + 2*w + d
names = [("W1", w*d), ("b1", w), ("W2", w*w), ("b2", w), ("W3", d*w), ("b3", d)]
g1 = res[1][1]
for n in range(N):
    off = 1 + n * P
    for nm, sz in names:
        a, b = g0[off:off+sz], g1[off:off+sz]
        print(n, nm, "max|g| %.3e maxdiff %.3e ndiff %d" % (np.abs(a).max(), np.abs(a-b).max(), np.count_nonzero(a != b)))
        off += sz
