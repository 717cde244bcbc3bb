"""Per-round SASS view of an ncu source export (development aid).
usage: ncu -i X.ncu-rep --page source --csv --print-source sass > x.csv
       python tools/sass_hot.py x.csv <units> [min_per_unit] [--ops]"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = rows[2:]
U = float(sys.argv[2]); mn = float(sys.argv[3]) if len(sys.argv) > 3 and not sys.argv[3].startswith('-') else 0.5
ai = hdr.index("Instructions Executed"); si = hdr.index("Warp Stall Sampling (All Samples)")
tot_s = sum(int(r[si] or 0) for r in data) or 1
ops = collections.Counter(); tot = 0; prev = -5
for i, r in enumerate(data):
    n = int(r[ai] or 0) / U
    if n >= 0.01:
        op = r[1].strip().split()
        if op and op[0].startswith('@'): op = op[1:]
        ops[op[0].split('.')[0] if op else '?'] += n; tot += n
    if n >= mn and '--ops' not in sys.argv:
        if i != prev + 1: print('----')
        prev = i
        print(f"{i:6d} {n:5.2f} {100*int(r[si])/tot_s:5.1f}% {r[1].strip()[:96]}")
print(f"total warp-instructions per unit: {tot:.1f}")
print(' '.join(f"{o}:{n:.0f}" for o, n in ops.most_common(24)))
