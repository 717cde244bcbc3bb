"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.
usage: python tools/launch_summary.py launches.csv"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = collections.defaultdict(list)
for r in rows[1:]:
    agg[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")))
tot = sum(sum(v) for v in agg.values())
print(f"{'kernel':50s} {'launches':>8s} {'total ms':>12s} {'mean us':>12s} {'share':>7s}")
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{k[:50]:50s} {len(v):8d} {sum(v)/1e6:12.3f} {sum(v)/len(v)/1e3:12.1f} {sum(v)/tot:7.4f}")
