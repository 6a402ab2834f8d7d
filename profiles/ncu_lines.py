"""Aggregate ncu warp-stall samples of a report by CUDA source line (needs -lineinfo).
usage: python profiles/ncu_lines.py report.ncu-rep [top] [kernel-substring]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
items = []
tot = 0
fname = "?"
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        si = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or not r or not r[0]:
        continue
    try:
        s = int(float(r[si]))
    except (ValueError, IndexError):
        continue
    tot += s
    items.append((s, f"{fname}:{r[0]}", r[1].strip()[:100]))
items.sort(reverse=True)
print(f"total samples {tot}")
for s, ln, src in items[:top]:
    print(f"{100.0 * s / max(tot, 1):5.1f}%  {ln:>16}  {src}")
