"""Instruction / stall-sample shares by code region of the search kernel.
usage: python profiles/ncu_regions.py report.ncu-rep search.cu
(search.cu = the exact source the report was compiled from, -lineinfo).  Regions: the function
whose definition precedes the line, and inside search_kernel the beam sections by their comment
markers."""
import collections
import csv
import io
import re
import subprocess
import sys

rep, srcpath = sys.argv[1], sys.argv[2]
src = open(srcpath).read().split("\n")
MARK = [("// 1. quantize", "query setup"), ("// 2. greedy", "greedy upper layers"),
        ("// 3. layer-0 beam", "beam: pick + row + dists call"), ("// filter against", "beam: filter + dedupe"),
        ("// the next expansion is", "beam: next pick + prefetch"), ("// merge", "beam: merge (sort + shift)"),
        ("// debug: C with", "beam end: C trace + stage 2-3 call")]
FN = re.compile(r"\b(\w+)\s*\(")
region_of = {}
region = "file scope"
for i, ln in enumerate(src, 1):
    s = ln.strip()
    if (s.startswith("__device__") or s.startswith("__global__") or s.startswith("template")) and "(" in s:
        names = [n for n in FN.findall(s) if n not in ("__launch_bounds__", "template", "constexpr")]
        if names:
            region = names[0]
    for mk, nm in MARK:
        if mk in s:
            region = nm
    region_of[i] = region
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
acc, accs = collections.Counter(), collections.Counter()
fname, hdr = "?", None
tot = tots = 0
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        si, ii = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
        continue
    if hdr is None or not r or not r[0]:
        continue
    try:
        ln, n, s = int(r[0]), int(float(r[ii])), int(float(r[si]))
    except (ValueError, IndexError):
        continue
    key = region_of.get(ln, "?") if fname == "search.cu" else f"intrinsics ({fname})"
    acc[key] += n
    accs[key] += s
    tot += n
    tots += s
print(f"{'region':40s} {'instr%':>7s} {'stall%':>7s}")
for k, v in acc.most_common():
    if v:
        print(f"{k:40s} {100 * v / max(tot, 1):7.1f} {100 * accs[k] / max(tots, 1):7.1f}")
print("total instructions", tot)
