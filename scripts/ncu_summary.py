"""Summarise an ncu launch-list CSV and a --set full report into markdown.

usage: ncu_summary.py <launches.csv> <full.ncu-rep> > profiles/<name>.md
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sectors_op_read.sum", "lts__t_sectors_op_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__occupancy_limit_shared_mem",
        "sm__maximum_warps_per_active_cycle_pct",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio"]


def launches(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    H = rows[h]
    ki, vi, ui = H.index("Kernel Name"), H.index("Metric Value"), H.index("Metric Unit")
    d = defaultdict(list)
    unit = "ns"
    for r in rows[h + 1:]:
        if len(r) > vi:
            d[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")))
            unit = r[ui]
    scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1e-3)
    tot = sum(sum(v) for v in d.values())
    out = ["| kernel | launches | total us | mean us | share |", "|---|---|---|---|---|"]
    for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
        out.append(f"| `{k}` | {len(v)} | {sum(v)*scale:.1f} | {sum(v)/len(v)*scale:.2f} | "
                   f"{sum(v)/tot:.3f} |")
    return "\n".join(out)


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    H, U = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        name = r[H.index("Kernel Name")]
        out.append(f"\n### `{name[:90]}`\n\n| metric | value | unit |\n|---|---|---|")
        for k in KEYS:
            if k in H:
                i = H.index(k)
                out.append(f"| {k} | {r[i]} | {U[i]} |")
    return "\n".join(out)


if __name__ == "__main__":
    print("## Launch list (ncu --metrics gpu__time_duration.sum, cold-cache, serialised)\n")
    print(launches(sys.argv[1]))
    if len(sys.argv) > 2:
        print("\n## Full capture (--set full --clock-control none)")
        print(full(sys.argv[2]))
