"""Per-source-line executed instructions (per unit) and stall samples from an
ncu 'cuda,sass' source export.  usage: python tools/ncu_inst.py x.csv UNITS [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 45
cur = None
hdr = None
inst = collections.Counter()
samp = collections.Counter()
text = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ii = hdr.index("Instructions Executed")
        si = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or not r[0].strip():
        continue
    try:
        k = (cur, int(r[0]))
    except ValueError:
        continue
    text[k] = r[1].strip()[:80]
    try:
        inst[k] += int(r[ii] or 0)
        samp[k] += int(r[si] or 0)
    except (ValueError, IndexError):
        pass
ti, ts = sum(inst.values()), sum(samp.values())
print(f"instructions/unit {ti/units:.1f}  samples {ts}")
for k, v in sorted(inst.items(), key=lambda x: -x[1])[:top]:
    print(f"{v/units:8.1f} inst {100*samp[k]/max(ts,1):5.1f}% smp  {k[0]}:{k[1]}  {text[k]}")
