"""Small runs of every kernel family for compute-sanitizer (SURVEY §5 race
detection): per-step SIMT (heat, HJB, NAIS-Net), per-step tcgen05 (Allen-Cahn
d = 100, deterministic and atomics), and the shared formulation (FC, NAIS-Net).

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
    compute-sanitizer --tool racecheck python tools/sanitize_run.py simt
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_11623_b200 import BSDE  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
runs = []
if which in ("all", "simt"):
    runs += [("heat", 10, 20, 3, 256, {}), ("hjb", 37, 45, 3, 200, {}),
             ("hjb", 20, 24, 2, 128, dict(arch="nais"))]
if which in ("all", "tc"):
    runs += [("allen_cahn", 100, 110, 2, 300, dict(precision="bf16")),
             ("allen_cahn", 100, 110, 2, 300, dict(precision="bf16", deterministic=True))]
if which in ("all", "tc32"):
    runs += [("hjb", 100, 110, 2, 300, dict(kernel="tc")), ("hjb", 37, 45, 3, 200, dict(kernel="tc")),
             ("black_scholes", 100, 110, 2, 130, dict(kernel="tc", x0=1.0))]
if which in ("all", "fused"):
    runs += [("allen_cahn", 100, 110, 2, 300, dict(precision="bf16", fused_opt=True))]
if which in ("all", "shared"):
    runs += [("black_scholes", 16, 32, 3, 64, dict(formulation="shared", layers=3, x0=0.5)),
             ("hjb", 16, 32, 3, 64, dict(formulation="shared", layers=3, arch="nais"))]
for prob, d, w, N, B, kw in runs:
    kw = dict(kw)
    fused = kw.pop("fused_opt", False)
    kern = kw.pop("kernel", None) or ("simt" if kw.get("precision", "fp32") == "fp32"
                                      and kw.get("formulation") != "shared" else "auto")
    s = BSDE(prob, d, N, 1.0, w, B, kernel=kern, use_graph=False, **kw)
    if fused:
        s.enable_fused_optimizer()
    for _ in range(2):
        s.train_step()
    s.eval_loss(1, B)
    print("ok", prob, d, w, N, B, kw, s.family, flush=True)
    s.close()
print("sanitize runs done")
