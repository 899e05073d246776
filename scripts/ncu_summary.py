"""Summarise ncu outputs for profiles/: per-kernel launch times (from a --metrics
gpu__time_duration.sum CSV) and key metrics of a --set full report.
Usage: python scripts/ncu_summary.py launches.csv [full.ncu-rep] > profiles/<name>.md"""
import csv
import subprocess
import sys
from collections import defaultdict


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[start]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    d = defaultdict(list)
    for r in rows[start + 1:]:
        if len(r) > vi:
            v = float(r[vi].replace(",", ""))
            scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(r[ui], 1e-6)
            d[r[ki].split("(")[0]].append(v * scale)
    tot = sum(sum(v) for v in d.values())
    print(f"## launch list: {path}\n")
    print("| kernel | launches | avg ms | total ms | share |\n|---|---|---|---|---|")
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        print(f"| `{k}` | {len(v)} | {sum(v)/len(v):.4f} | {sum(v):.2f} | {sum(v)/tot:.1%} |")
    print()


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__block_size", "launch__grid_size", "launch__occupancy_limit_registers",
        "smsp__inst_executed.sum", "lts__t_bytes.sum",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard",
        "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
        "smsp__warp_issue_stalled_barrier_per_warp_active.pct",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    print(f"## ncu --set full: {path}\n")
    for r in rows[2:]:
        name = r[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print(f"### `{name[:90]}`\n\n| metric | value | unit |\n|---|---|---|")
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f"| {k} | {r[i]} | {units[i]} |")
        print()


if __name__ == "__main__":
    launches(sys.argv[1])
    for p in sys.argv[2:]:
        full(p)
