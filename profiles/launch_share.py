"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv).
usage: python profiles/launch_share.py launches.csv"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[0].isdigit()]
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows:
    name = r[4].split("(")[0][:90]
    v = float(r[14].replace(",", ""))
    unit = r[13]
    ns = v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(unit, 1)
    tot[name] += ns
    cnt[name] += 1
all_ns = sum(tot.values())
print(f"{len(rows)} launches, {all_ns / 1e6:.2f} ms total (cold-cache, serialised)")
for k, v in sorted(tot.items(), key=lambda z: -z[1])[:15]:
    print(f"{100 * v / all_ns:6.2f}%  {v / 1e6:10.3f} ms  {cnt[k]:5d} x  {k}")
