"""Summarise an ncu report (raw page) into the metrics the bench/DESIGN cite.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/<name>.txt
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("duration_ms", "gpu__time_duration.sum"),
    ("sm_clock_ghz", "sm__cycles_elapsed.avg.per_second"),
    ("regs", "launch__registers_per_thread"),
    ("threads", "launch__block_size"),
    ("grid", "launch__grid_size"),
    ("dram_read_GB", "dram__bytes_read.sum"),
    ("dram_write_GB", "dram__bytes_write.sum"),
    ("dram_pct_peak", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("tensor_pipe_pct", "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"),
    ("tensor_mem_pct", "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
    ("sm_throughput_pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("issue_active_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
    ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("ipc", "sm__inst_executed.avg.per_cycle_active"),
    ("alu_pipe_pct", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
    ("fma_pipe_pct", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
    ("xu_pipe_pct", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
    ("lsu_pipe_pct", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
    ("uniform_pipe_pct", "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active"),
    ("inst_executed", "smsp__inst_executed.sum"),
]
STALL_PREFIX = "smsp__average_warp_latency_issue_stalled_"
STALL_PREFIX2 = "smsp__pcsamp_warps_issue_stalled_"


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    for d in data:
        print("kernel:", d[idx["Kernel Name"]])
        for name, key in KEYS:
            k = key if key in idx else next((h for h in idx if h.endswith("." + key)), None)
            if k is not None:
                print("  %-18s %s %s" % (name, d[idx[k]], units[idx[k]]))
        stalls = []
        for h, i in idx.items():
            if h.startswith(STALL_PREFIX2) and not h.endswith("not_issued") and d[i]:
                try:
                    stalls.append((float(d[i].replace(",", "")), h[len(STALL_PREFIX2):]))
                except ValueError:
                    pass
        if stalls:
            tot = sum(s for s, _ in stalls) or 1.0
            print("  stall samples (top):",
                  ", ".join("%s %.0f%%" % (n, 100 * s / tot) for s, n in sorted(stalls)[::-1][:8]))
        print()


if __name__ == "__main__":
    main(sys.argv[1])
