"""Aggregate an ncu 'cuda,sass' source export per CUDA source line.
usage: ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > x.csv
       python tools/ncu_lines.py x.csv [top]"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur_file = None; hdr = None
agg_i = collections.Counter(); agg_s = collections.Counter(); text = {}
line_key = None
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur_file = r[1].split("/")[-1]; continue
    if r[0] == "Function Name": continue
    if r[0] == "Line No": hdr = r; ii = hdr.index("Instructions Executed"); si = hdr.index("Warp Stall Sampling (All Samples)"); continue
    if hdr is None: continue
    # a source row has a line number in col 0; sass rows have empty col 0
    if r[0].strip():
        line_key = (cur_file, int(r[0])); text[line_key] = r[1].strip()[:70]
        # some exports put line-level totals on the source row
        try:
            agg_i[line_key] += int(r[ii] or 0); agg_s[line_key] += int(r[si] or 0)
        except (ValueError, IndexError): pass
tot_i = sum(agg_i.values()); tot_s = sum(agg_s.values())
print(f"total inst {tot_i}  samples {tot_s}")
for k, v in agg_s.most_common(top):
    print(f"{v:7d} {100*v/max(tot_s,1):5.1f}%  inst {agg_i[k]:10d}  {k[0]}:{k[1]}  {text.get(k,'')}")
