"""Multilevel (coarse-to-fine time grid) training schedule, §3.2 of the paper.

PAPER.md:237-252: "we start with samples of small number of time steps (low
accuracy) and then gradually increase the number of time steps", with step
sizes h_l = h_0 M^{-l}; the experiments use 2, 4, 8, 16 and 32 steps
(PAPER.md:463), i.e. M = 2.  BASELINE.json config 4 uses N = 5 -> 10 -> 20 ->
40 -> 80 with a fixed iteration budget per level.

This is host-side control only: each level runs `bsde_train_step` on the
device, and a level change is one `bsde_prolongate` call (copy or midpoint
prolongation of the per-step nets; the Adam state reset, R14, or prolonged with the
parameters when the context was created with keep_adam, R14b).  Evaluation uses a
fixed evaluation stream (`bsde_eval_loss`) so that losses at different
iterations are comparable; evaluation time is excluded from the training clock.
"""
import time
from dataclasses import dataclass, field
from typing import List, Optional


@dataclass
class LevelRecord:
    level: int
    N: int
    iteration: int          # global iteration index (continues across levels, R9)
    train_loss: float
    eval_loss: Optional[float]
    train_seconds: float    # wall clock spent in training steps so far (evals excluded)


@dataclass
class MultilevelResult:
    records: List[LevelRecord] = field(default_factory=list)
    time_to_target: Optional[float] = None
    iteration_at_target: Optional[int] = None
    y0_per_level: List[float] = field(default_factory=list)
    final_eval_loss: Optional[float] = None


def _sync(solver):
    if getattr(solver, "stream", None) is not None:
        solver.stream.synchronize()


def run_schedule(solver, iters_per_level, *, eval_every=25, eval_batch=None, eval_id=0,
                 target_loss=None, final_N=None, extend_last=0, clock=time.perf_counter):
    """Train `solver` over len(iters_per_level) levels starting at its current N.

    After level l (except the last) the solver is prolonged to level l+1.
    `target_loss` (optional) is checked on evaluations at N == final_N; the
    last level may run `extend_last` extra iterations until it is reached.
    Returns a MultilevelResult.
    """
    res = MultilevelResult()
    t_train = 0.0
    L = len(iters_per_level)
    for li, iters in enumerate(iters_per_level):
        N = solver.N
        budget = iters + (extend_last if li == L - 1 else 0)
        k = 0
        while k < budget:
            _sync(solver)
            t0 = clock()
            loss = solver.train_step(sync=True)
            t_train += clock() - t0
            k += 1
            ev = None
            if eval_every and (k % eval_every == 0 or k == budget):
                ev = solver.eval_loss(eval_id, eval_batch)
                res.final_eval_loss = ev
                if (target_loss is not None and res.time_to_target is None
                        and (final_N is None or N == final_N) and ev <= target_loss):
                    res.time_to_target = t_train
                    res.iteration_at_target = solver.iteration
            res.records.append(LevelRecord(li, N, solver.iteration, loss, ev, t_train))
            if k >= iters and res.time_to_target is not None:
                break
        res.y0_per_level.append(solver.y0())
        if li + 1 < L:
            solver.prolongate(li + 1)
    return res


def write_loss_csv(result, path):
    """Loss curve as CSV (SURVEY §5 metrics; SPEC S:502 columns iteration, level,
    loss, elapsed_seconds, plus N and the evaluation loss where one was taken)."""
    with open(path, "w") as f:
        f.write("iteration,level,N,loss,eval_loss,elapsed_seconds\n")
        for r in result.records:
            f.write("%d,%d,%d,%.9g,%s,%.6f\n" % (r.iteration, r.level, r.N, r.train_loss,
                                                 "" if r.eval_loss is None else "%.9g" % r.eval_loss,
                                                 r.train_seconds))
