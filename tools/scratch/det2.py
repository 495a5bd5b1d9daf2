import sys, os, numpy as np
sys.path.insert(0, os.getcwd())
from paper_1910_11623_b200 import BSDE
d, w, N = 100, 110, 4
mk = lambda: BSDE("allen_cahn", d, N, 0.3, w, 2048, precision="bf16", lr=5e-4)
a, b = mk(), mk()
for k in range(3):
    la, lb = a.train_step(), b.train_step()
    ga, gb = a.get_grads().astype(np.float64), b.get_grads().astype(np.float64)
    pa, pb = a.get_params(), b.get_params()
    print("step", k, la, lb, "grad maxdiff", np.abs(ga-gb).max(), "param frac>1e-6", np.mean(np.abs(pa-pb) > 1e-6))
P = 2*d*w + w*w + 2*w + d
names = [("W1", w*d), ("b1", w), ("W2", w*w), ("b2", w), ("W3", d*w), ("b3", d)]
m, v, t = a.get_adam_state()
for n in range(N):
    off = 1 + n * P
    for nm, sz in names:
        x, y = pa[off:off+sz], pb[off:off+sz]
        dd = np.abs(x - y)
        i = np.argmax(dd)
        print(n, nm, "ndiff>1e-6 %d maxdiff %.3e at |g|=%.3e v=%.3e" % (np.count_nonzero(dd > 1e-6), dd.max(), abs(ga[off+i]), v[off+i]))
        off += sz
