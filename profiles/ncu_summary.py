"""One-screen summary of an ncu report: key raw metrics + top source lines by stall samples
and by executed instructions.  usage: python profiles/ncu_summary.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, units, v = r[0], r[1], r[2]
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.avg.per_cycle_active", "smsp__inst_executed.sum", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__grid_size",
        "launch__block_size", "launch__shared_mem_per_block_dynamic"]
for k in keys:
    if k in h:
        i = h.index(k)
        print(f"{k:60s} {v[i]} {units[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = None
by_stall, by_inst = [], []
ts = ti = 0
fname = "?"
for row in rows:
    if row and row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row and row[0] == "Line No":
        hdr = row
        si = hdr.index("Warp Stall Sampling (All Samples)")
        ii = hdr.index("Instructions Executed")
        continue
    if hdr is None or not row or not row[0]:
        continue
    try:
        s, n = int(float(row[si])), int(float(row[ii]))
    except (ValueError, IndexError):
        continue
    ts += s
    ti += n
    tag = f"{fname}:{row[0]}"
    by_stall.append((s, tag, row[1].strip()[:90]))
    by_inst.append((n, tag, row[1].strip()[:90]))
for title, items, tot in [("stall samples", by_stall, ts), ("warp instructions", by_inst, ti)]:
    items.sort(reverse=True)
    print(f"\n-- top source lines by {title} (total {tot}) --")
    for s, tag, line in items[:top]:
        print(f"{100.0 * s / max(tot, 1):5.1f}%  {tag:>18}  {line}")
