"""Stall-reason breakdown (pc sampling) + key throughput metrics of an ncu report.
usage: python profiles/ncu_stalls.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, u, v = r[0], r[1], r[2]
items = []
for i, k in enumerate(h):
    if "smsp__pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued"):
        try:
            items.append((float(v[i]), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
items.sort(reverse=True)
tot = sum(x for x, _ in items) or 1.0
print("stall reasons (share of pc samples):")
for x, k in items[:12]:
    print(f"  {100 * x / tot:5.1f}%  {k}")
for k in ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "smsp__warps_active.avg.per_cycle_active", "smsp__warps_eligible.avg.per_cycle_active",
          "dram__bytes_read.sum", "lts__t_sector_hit_rate.pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]:
    if k in h:
        print(f"{k:60s} {v[h.index(k)]} {u[h.index(k)]}")
