"""Hottest SASS instructions (by stall samples) with preceding context from an
ncu 'cuda,sass' source export.  usage: python tools/ncu_hot.py x.csv [top] [ctx]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 10
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 5
sass, cur, seen = [], None, set()
for r in rows[3:]:
    if not r:
        continue
    if r[0].strip():
        cur = r[0]
        continue
    if len(r) > 7 and r[2].startswith("0x"):
        a = int(r[2], 16)
        if a in seen:
            continue
        seen.add(a)
        sass.append((a, cur, r[3].strip(), int(r[4] or 0), int(r[7] or 0)))
sass.sort()
tot = sum(s[3] for s in sass)
print("total samples", tot)
for i in sorted(range(len(sass)), key=lambda i: -sass[i][3])[:top]:
    print(f"---- {sass[i][3]} ({100*sass[i][3]/tot:.1f}%)")
    for j in range(max(0, i - ctx), i + 1):
        a, l, t, smp, ex = sass[j]
        print(f"  {a & 0xfffff:6x} L{l:>4} {smp:6d} {ex:10d}  {t}")
