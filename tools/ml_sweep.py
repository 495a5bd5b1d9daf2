"""Multilevel schedule sweep on config 4 (experiment tool, not the product path):
one single-level N = 80 run sets the target (bench rule: 1.01 x the mean of its last
five evaluation losses), then multilevel variants are timed to the same target.

Variants: iterations per coarse level, and the Adam state at a level change —
'reset' (R14) or 'carry' (BSDE_PROLONG_KEEP_ADAM, R14b: m, v prolonged on the device by
the parameters' copy rule, t kept).

    python tools/ml_sweep.py [--iters 10000] [--variants 400:reset,400:carry,...]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=10000)
    ap.add_argument("--variants", default="400:reset,400:carry,1000:reset,1000:carry,2000:carry")
    ap.add_argument("--precision", default="bf16")
    ap.add_argument("--eval-every", type=int, default=50)
    ap.add_argument("--reps", type=int, default=1)
    args = ap.parse_args()
    import torch
    from paper_1910_11623_b200 import BSDE
    from paper_1910_11623_b200.multilevel import run_schedule
    from workloads import CONFIGS
    wl = CONFIGS["cfg4_hjb_multilevel"]
    levels = list(wl.levels)
    Nf, B = levels[-1], wl.batch
    kw = dict(lr=wl.lr, precision=args.precision, seed=wl.seed)
    single = BSDE(wl.problem, wl.d, Nf, wl.T, wl.w, B, **kw)
    rs = run_schedule(single, [args.iters], eval_every=args.eval_every, eval_batch=B)
    ev = [(r.train_seconds, r.iteration, r.eval_loss) for r in rs.records if r.eval_loss is not None]
    target = 1.01 * float(np.mean([e[2] for e in ev[-5:]]))
    t_s = next(e[0] for e in ev if e[2] <= target)
    print(json.dumps({"single": {"target": target, "time_to_target_s": t_s,
                                 "iteration_at_target": next(e[1] for e in ev if e[2] <= target),
                                 "total_s": rs.records[-1].train_seconds, "y0": single.y0()}}), flush=True)
    single.close()
    torch.cuda.synchronize()
    for var in args.variants.split(",") * args.reps:
        per, mode, *pro = var.split(":")   # per-level:reset|carry[:copy|interp]
        per = int(per)
        s = BSDE(wl.problem, wl.d, levels[0], wl.T, wl.w, B, max_levels=len(levels) - 1,
                 keep_adam=(mode == "carry"), prolong=(pro[0] if pro else "copy"), **kw)
        rm = run_schedule(s, [per] * (len(levels) - 1) + [per], eval_every=args.eval_every, eval_batch=B,
                          target_loss=target, final_N=Nf, extend_last=args.iters)
        coarse = next((r.train_seconds for r in rm.records if r.N == Nf), None)
        print(json.dumps({"variant": var, "time_to_target_s": rm.time_to_target,
                          "iteration_at_target": rm.iteration_at_target,
                          "speedup": (t_s / rm.time_to_target) if rm.time_to_target else None,
                          "coarse_levels_s": coarse, "y0_per_level": rm.y0_per_level,
                          "final_eval": rm.final_eval_loss}), flush=True)
        s.close()
        torch.cuda.synchronize()


if __name__ == "__main__":
    main()
