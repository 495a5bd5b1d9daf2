"""Benchmark of the deep-BSDE training step (BASELINE.json metric: path-steps/s
and % of roofline).  Prints ONE JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--impl reference]

N = 1 runs in-process; N > 1 is launched by torchrun (one rank per GPU over
NCCL).  The default workload is config 5 (Allen-Cahn, d = 100, N = 80,
524288 paths, bf16 operands), the configuration the metric is quoted on at
1/2/4/8 GPUs (global batch fixed: strong scaling).  A "step" is one full
training iteration: Philox ΔW, forward rollout, terminal loss, adjoint,
gradient allreduce, Adam.

--impl reference runs the float64 CPU oracle (the reference arm of this tier)
on a bounded sample of the same workload.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads import CONFIGS  # noqa: E402

# the paper's single-level solution times of its Table 1 workloads
PAPER_MINUTES = {"nx1_shared_bs_paper": 59.0, "nx1_shared_bs_resnet_paper": 73.0,
                 "nx2_shared_bs_nais_paper": 123.0}
METRIC = "BSDE train path-steps/sec & % roofline at d=100 (1/2/4/8 B200); multilevel time-to-loss"
UNIT = "path-steps/s"
# algorithmic flop per path-step: forward 2(dw + w² + wd),
# adjoint without dX 6dw + 4w² (replay and padding are implementation work)
def fwd_flops(d, w):
    return 2 * (d * w + w * w + w * d)


def bwd_flops(d, w):
    return 6 * d * w + 4 * w * w


# Shared-network formulation (NEXT-1, R23): per row (path, time point) the forward
# (K0 = d+1 inputs, L tanh layers of w) and the input gradient each cost
# 2(K0 w + (L-1) w²); the reverse-over-reverse gradient costs three such passes
# (δᵀḡ, ḡWᵀ, āᵀh) plus the hidden-state back-propagation 2(L-1)w².  N+1 rows per
# N path-steps.
def shared_flops(wl):
    K0, w, L = wl.d + 1, wl.w, wl.layers
    one = 2 * (K0 * w + (L - 1) * w * w)
    if wl.arch == "nais":   # + the input injection B_k u of every block (R26)
        one += 2 * (L - 1) * w * K0
    rows = (wl.N + 1) / wl.N
    return rows * 2 * one, rows * (3 * one + 2 * (L - 1) * w * w)   # (fwd + ∇ₓu, gradient)


def flops_per_path_step(wl):
    if wl.formulation == "shared":
        return shared_flops(wl)
    return fwd_flops(wl.d, wl.w), bwd_flops(wl.d, wl.w)


def shared_row_bytes(wl):
    K0p = (wl.d + 1 + 3) // 4 * 4
    L, w = wl.layers, wl.w
    floats = 3 * K0p + wl.d + w * (2 * L + (L - 1) + L + 4) + 6
    if wl.arch in ("resnet", "nais"):
        floats += w * (L - 1 + 2)
    return 4 * floats


def peaks():
    p = {"hbm_gbs": 6558.4, "bf16_tflops": 1675.8, "bf16_tflops_sustained": 1400.3,
         "sm_max_mhz": 1965.0, "source": "fallback"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        p.update({k: m[k] for k in ("hbm_gbs", "bf16_tflops", "bf16_tflops_sustained",
                                     "sm_max_mhz") if k in m})
        p["source"] = "measured"
    except Exception:
        pass
    return p


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index, interval_ms=100):
        self.index = index
        self.interval_ms = interval_ms
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                 "--format=csv,noheader,nounits", "-lms", str(self.interval_ms)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            parts = [x.strip() for x in l.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(max(mx)) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_info():
    model = "unknown"
    try:
        for l in open("/proc/cpuinfo"):
            if l.startswith("model name"):
                model = l.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return model


def oracle_rate(wl, paths, iters):
    """The float64 oracle as it stands on a bounded path sample; path-steps/s."""
    from threadpoolctl import threadpool_info
    from oracle import bsde as ob
    from oracle import shared as osh
    prob = ob.PROBLEM_NAMES[wl.problem]
    if wl.formulation == "shared":
        arch = {"fc": osh.FC, "resnet": osh.RESNET, "nais": osh.NAIS}[wl.arch]
        p = osh.init_params(wl.seed, wl.d, wl.w, wl.layers, arch)

        def one(k):
            return osh.iteration(prob, wl.d, wl.w, wl.layers, arch, wl.N, wl.T, p, wl.seed, k,
                                 np.arange(paths), wl.batch, x0=wl.x0)
    else:
        p = ob.init_params(wl.seed, wl.d, wl.w, wl.N,
                           zero_head=(wl.problem == "allen_cahn"))   # R7b, as the GPU init

        def one(k):
            return ob.iteration(prob, wl.d, wl.w, wl.N, wl.T, p, wl.seed, k, np.arange(paths),
                                wl.batch, x0=wl.x0)
    st = ob.AdamState(p.size)
    times = []
    for k in range(iters):
        t0 = time.perf_counter()
        r = one(k)
        ob.adam_step(p, r["grad"], st, wl.lr, loss=r["loss"])
        times.append(time.perf_counter() - t0)
    threads = max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    return paths * wl.N / float(np.median(times)), threads, times


def run_reference(args, wl, rank):
    if rank != 0:
        return
    paths = args.ref_paths or max(256, min(wl.batch, int(2.4e5 // wl.N)))
    rate, threads, times = oracle_rate(wl, paths, args.warmup + args.steps)
    timed = times[args.warmup:] or times
    sample = "%d of %d paths x N=%d, full network, fp64 numpy; median of %d iterations" % (
        paths, wl.batch, wl.N, len(timed))
    line = {"impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * float(np.median(timed)) * wl.batch / paths,
            "ms_per_step_extrapolated": True,
            "ms_per_step_note": "median sample-iteration time x batch / sample paths (the "
                                "oracle's cost is linear in the path count)",
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (Philox Brownian increments, R8)",
            "config": config_dict(wl, args.gpus, "oracle"),
            "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads, "kind": "oracle",
                             "sample": sample, "cpu": cpu_info()},
            "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_dict(wl, gpus, family):
    c = {"workload": wl.name, "problem": wl.problem, "d": wl.d, "w": wl.w, "N": wl.N,
         "T": wl.T, "batch_global": wl.batch, "precision": wl.precision, "kernel": family,
         "parallelism": "dp%d" % gpus, "formulation": wl.formulation}
    if wl.formulation == "shared":
        c.update({"arch": wl.arch, "layers": wl.layers, "x0": wl.x0})
        ws = (wl.N + 1) * wl.batch // gpus * shared_row_bytes(wl) / 2 ** 20
        c["l2"] = ("working set %.0f MiB per GPU; %s" % (ws, "L2 flushed between timed steps "
                   "(256 MiB memset outside the per-step events)" if ws < 256 else
                   "larger than L2, no explicit flush"))
    else:
        c["l2"] = ("inputs larger than L2: per-step X_n store (N*B*d*4 bytes) >> 126 MB; "
                   "no explicit flush")
    return c


def spawn_ranks(args):
    """Re-launch this script under torch.distributed.run with --gpus ranks on
    127.0.0.1 (rank 0 prints the JSON line); NCCL logs its ranks on stderr."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           "--nproc-per-node", str(args.gpus), "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    r = subprocess.run(cmd, env=env)
    if r.returncode:
        raise SystemExit(r.returncode)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default 40: >= 0.5 s under load, several 100 ms clock samples; 10 for --impl reference)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="cfg5_allen_cahn_scaleout", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--kernel", default="auto")
    ap.add_argument("--precision", default=None)
    ap.add_argument("--ref-paths", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--deterministic", action="store_true",
                    help="fixed-order reductions instead of atomics (cfg.deterministic)")
    ap.add_argument("--no-multilevel", action="store_true",
                    help="skip the config-4 multilevel time-to-target sub-object (rank 0, N = 1)")
    ap.add_argument("--ml-iters", type=int, default=10000,
                    help="single-level iterations of the multilevel experiment")
    ap.add_argument("--ml-precision", default="fp32",
                    help="config 4 is fp32 in BASELINE.json (as config 2): the fp32-accurate "
                         "tc32 kernels by default; bf16 for a quick run")
    ap.add_argument("--sharded-adam", action="store_true",
                    help="reduce-scatter + sharded Adam + all-gather (NEXT-4) for N > 1")
    ap.add_argument("--fused-opt", action="store_true",
                    help="NEXT-4 as one peer-memory kernel (fused_opt.cu) instead of NCCL + Adam")
    args = ap.parse_args()
    if args.steps is None:
        args.steps = 10 if args.impl == "reference" else 40
    wl = CONFIGS[args.workload]
    if args.precision:
        wl = wl.with_(precision=args.precision)

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N`: start the N ranks (one process per GPU, NCCL)
        # ourselves, as the driver's torchrun launch would
        return spawn_ranks(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        raise SystemExit("bench.py: --gpus %d but WORLD_SIZE=%d" % (args.gpus, world))
    if args.impl == "reference":
        run_reference(args, wl, rank)
        return

    import torch
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    from paper_1910_11623_b200 import BSDE

    kw = dict(lr=wl.lr, precision=wl.precision, kernel=args.kernel, seed=wl.seed,
              device=local_rank, x0=wl.x0)
    if wl.formulation == "shared":
        kw.update(formulation="shared", arch=wl.arch, layers=wl.layers)
    if args.sharded_adam:
        kw.update(sharded_adam=True)
    if args.deterministic:
        kw.update(deterministic=True)
    if world > 1:
        s = BSDE.distributed(wl.problem, wl.d, wl.N, wl.T, wl.w, wl.batch, **kw)
    else:
        s = BSDE(wl.problem, wl.d, wl.N, wl.T, wl.w, wl.batch, **kw)
    if args.fused_opt:
        s.enable_fused_optimizer()
    family = s.family
    stream = s.stream          # the stream libbsde enqueues on

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(max(3, args.warmup)):
        s.train_step(sync=False)
    barrier()
    clocks = ClockSampler(local_rank if "CUDA_VISIBLE_DEVICES" not in os.environ else
                          os.environ["CUDA_VISIBLE_DEVICES"].split(",")[local_rank])
    clocks.start()
    time.sleep(0.3)
    flush = None
    if wl.formulation == "shared" and (wl.N + 1) * wl.batch // world * shared_row_bytes(wl) < 2 ** 28:
        flush = torch.empty(2 ** 26, dtype=torch.float32, device="cuda")   # 256 MiB > L2
    barrier()
    if flush is None:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            s.train_step(sync=False)
        e1.record(stream)
        barrier()
        ms = e0.elapsed_time(e1) / args.steps
    else:   # working set < L2: flush between steps, time each step with its own events
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        with torch.cuda.stream(stream):
            for a0, a1 in evs:
                flush.fill_(1.0)
                a0.record(stream)
                s.train_step(sync=False)
                a1.record(stream)
        barrier()
        ms = sum(a0.elapsed_time(a1) for a0, a1 in evs) / args.steps
    clk = clocks.stop()
    if dist is not None:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    launches = s.launches_per_step()
    path_steps = wl.batch * wl.N
    value = path_steps / (ms * 1e-3)

    # per-phase CUDA-event timing of the same step (eager replay of the step), with the
    # SM clock sampled over it: the replay is short, so it usually runs above the
    # power-capped clock of the long timed region, which is most of the gap between
    # ms_per_step and the sum of the phases
    pclocks = ClockSampler(local_rank if "CUDA_VISIBLE_DEVICES" not in os.environ else
                           os.environ["CUDA_VISIBLE_DEVICES"].split(",")[local_rank], 20)
    pclocks.start()
    phase = s.profile_steps(max(2, min(args.steps, 5)))
    pclk = pclocks.stop()

    # e2e: the public API call per step with the loss read back to the host
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        s.train_step(sync=True)
    barrier()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / args.steps
    if dist is not None:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())

    if rank == 0:
        pk = peaks()
        B_local = wl.batch // world
        # burst: the kernels are timed in a short eager replay at ~1.9 GHz, not under
        # the seconds-long power-capped clock the sustained figure was measured at
        if family in ("tc", "shared-tc") and wl.precision == "bf16":
            bound, peak, pk_name = "tensor", pk["bf16_tflops"], "bf16 burst (measured)"
            peak_sus = pk["bf16_tflops_sustained"]
        elif family == "tc32":
            bound, peak = "tensor", pk["bf16_tflops"] / 3.0
            pk_name = ("bf16 burst / 3 (bf16x3 fp32-accurate split: three bf16 MMAs per product, "
                       "DESIGN R18b)")
            peak_sus = pk["bf16_tflops_sustained"] / 3.0
        else:
            bound, peak = "alu", 148 * 128 * 2 * pk["sm_max_mhz"] * 1e6 / 1e12
            pk_name = "fp32 FFMA: 148 SM x 128 lanes x 2 flop x sm_max_mhz (derived)"
            peak_sus = peak
        dom = "bwd" if phase["bwd"] >= phase["fwd"] else "fwd"

        def kernel_traffic(k):   # dram bytes per launch from one `ncu --set full` capture
            try:                 # (tools/ncu_traffic.py)
                with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
                    tr = json.load(f).get(wl.name, {}).get("bsde_" + k)
                if tr and world == 1:
                    return tr["bytes_per_launch"], "profiles/" + tr["source"]
            except Exception:
                pass
            return None, None

        traffic, traffic_src = kernel_traffic(dom)
        ffw, fbw = flops_per_path_step(wl)

        def kernel_roof(k):   # the same figures for each of the two pass kernels
            fl = B_local * wl.N * (fbw if k == "bwd" else ffw)
            ach = fl / (phase[k] * 1e-3) / 1e12
            tb, _ = kernel_traffic(k)
            return {"ms": phase[k], "achieved": ach, "frac": ach / peak, "frac_sustained": ach / peak_sus,
                    "algorithmic_flop_per_path_step": fbw if k == "bwd" else ffw, "traffic": tb,
                    "hbm_frac": (tb / (phase[k] * 1e-3) / 1e9 / pk["hbm_gbs"]) if tb else None}
        flops = B_local * wl.N * (fbw if dom == "bwd" else ffw)
        achieved = flops / (phase[dom] * 1e-3) / 1e12
        step_flops = wl.batch * wl.N * (ffw + fbw) / world
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16" if (family in ("tc", "shared-tc") and wl.precision == "bf16") else "f32",
            "dtype_note": ("fp32-accurate: bf16x3 split operands (hi·hi + hi·lo + lo·hi), fp32 "
                           "accumulation" if family == "tc32" else
                           "bf16 GEMM operands (biases folded; H1, H2 = bf16(H1 + bf16(ReLU(A2))); "
                           "binary16 dW copy), fp32 accumulation, X/Y/reductions/Adam fp32"
                           if family == "tc" else "fp32"),
            "data": "synthetic (Philox4x32-10 Brownian increments generated on device, R8)",
            "config": dict(config_dict(wl, world, family),
                           optimizer=("fused peer-memory kernel" if args.fused_opt else
                                      "NCCL reduce-scatter + sharded Adam + all-gather"
                                      if args.sharded_adam else "NCCL allreduce + Adam"
                                      if world > 1 else "Adam")),
            "roofline": {"bound": bound, "kernel": "bsde_" + dom, "achieved": achieved,
                         "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                         "peak_sustained": peak_sus, "frac_sustained": achieved / peak_sus,
                         "traffic": traffic, "traffic_source": traffic_src,
                         "peak_source": pk_name + "; " + pk["source"],
                         "algorithmic_flop_per_path_step": fbw if dom == "bwd" else ffw,
                         # the other roofline axis: the kernel's DRAM bytes (ncu) over its
                         # live duration against the measured copy bandwidth
                         "hbm": ({"achieved_gbs": traffic / (phase[dom] * 1e-3) / 1e9,
                                  "peak_gbs": pk["hbm_gbs"],
                                  "frac": traffic / (phase[dom] * 1e-3) / 1e9 / pk["hbm_gbs"]}
                                 if traffic else None),
                         # the dominant kernel is whichever pass took longer in this run; the
                         # two are within a few percent of each other at config 5
                         "per_kernel": {"bsde_fwd": kernel_roof("fwd"), "bsde_bwd": kernel_roof("bwd")}},
            "step_roofline": {"achieved_tflops": step_flops / (ms * 1e-3) / 1e12,
                              "frac": step_flops / (ms * 1e-3) / 1e12 / peak,
                              "frac_sustained": step_flops / (ms * 1e-3) / 1e12 / peak_sus,
                              "flop_per_path_step": ffw + fbw},
            "phase_ms": phase,
            "phase_clocks": {"sm_mhz": pclk.get("sm_mhz"), "samples": pclk.get("samples"),
                             "note": "SM clock during the eager per-phase replay; ms_per_step's "
                                     "region is in 'clocks'"},
            "gpu_launches": launches * args.steps,
            "clocks": clk,
            "e2e": {"value": path_steps / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 8,
                    "note": "bsde_train_step(ctx, &loss) per step, loss read back and stream "
                            "synchronised every step; the step's inputs are Philox counters "
                            "held on the device (no host input data exists, R8)"},
        }
        if family in ("tc", "tc32") and wl.formulation == "per_step":
            # the forward's other bound: the Philox4x32-10 + Box-Muller increments, 1 Philox
            # block per 4 normals, ceil(d/4) per path and (fine) step, against the
            # standalone generator's best measured rate (profiles/r02_ubench_philox.txt, lane
            # blocks per cycle per SM with the MUFU Box-Muller): 1.162 for the forward's
            # generator (rounds 0-2 from the per-launch table: eight rounds' multiplies per
            # lane), 1.039 for the full ten rounds of the tc32 path kernel, at the SM clock
            # of the phase replay the forward's time comes from
            blocks = B_local * wl.N * ((wl.d + 3) // 4)
            rng_ach = blocks / (phase["fwd"] * 1e-3)
            mhz = pclk.get("sm_mhz") or clk.get("sm_mhz") or pk["sm_max_mhz"]
            rate = 1.162 if family == "tc" else 1.039
            rng_peak = rate * 148 * mhz * 1e6
            line["rng_roofline"] = {
                "kernel": "bsde_fwd", "bound": "alu", "unit": "Philox4x32-10 blocks/s",
                "achieved": rng_ach, "peak": rng_peak, "frac": rng_ach / rng_peak,
                "peak_source": "%.3f blocks/cycle/SM (Philox + MUFU Box-Muller, standalone, best "
                               "measured, profiles/r02_ubench_philox.txt) x 148 SM x SM clock of "
                               "the phase replay (%s MHz)" % (rate, mhz),
                "note": "the forward kernel also runs the three chain epilogues between its "
                        "random-number slices (DESIGN §6, §8 step floor)"}
        if wl.name in PAPER_MINUTES:
            # the paper's own timing of this workload: context only
            line["paper_context"] = {
                "solution_time_min": PAPER_MINUTES[wl.name], "hardware": "Tesla T4 (PyTorch)",
                "iterations": wl.iterations, "derived_path_steps_per_s": 2.8e4,
                "ours_solution_time_min": ms * wl.iterations / 6e4,
                "source": "BASELINE.md section 1; PAPER.md:488 (single-level, %s)" % wl.arch}
        if not args.no_cpu_baseline and world == 1:
            paths = max(256, min(wl.batch, int(2.4e5 // wl.N)))
            rate, threads, _ = oracle_rate(wl, paths, 2)
            line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": threads, "kind": "oracle",
                                    "sample": "%d of %d paths x N=%d, fp64 numpy oracle, median "
                                              "of 2 iterations" % (paths, wl.batch, wl.N),
                                    "cpu": cpu_info()}
        if not args.no_multilevel and world == 1 and args.workload == "cfg5_allen_cahn_scaleout":
            # the metric's second half (BASELINE.json): config 4's multilevel schedule
            # against single-level training, wall clock to the same target loss, this run
            s.close()
            s = None
            from bench_multilevel import run_cfg4
            ml = run_cfg4(args.ml_precision, args.ml_iters,
                          alt=[(1000, False, "copy"), (1000, True, "copy")])
            ml["note"] = ("config 4 (HJB d=100, N 5->80, B=65536), precision %s on the %s kernels "
                          "(tc32 = fp32-accurate bf16x3 split operands, R18b); time-to-target = "
                          "training wall clock (evaluations excluded) until the eval loss <= target"
                          % (args.ml_precision, ml["kernel"]))
            line["multilevel"] = ml
        print(json.dumps(line), flush=True)
    if s is not None:
        s.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
