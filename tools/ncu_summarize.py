"""Summarize an ncu report into small text files (run where the .ncu-rep is):
details page (SOL, memory, occupancy, launch stats, warp state), the raw
DRAM/L2 byte counters, and the top source lines by stall samples.

usage: python tools/ncu_summarize.py X.ncu-rep OUT_PREFIX
"""
import csv
import io
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


det = ncu("--page", "details", "--csv")
keep = []
for r in csv.reader(io.StringIO(det)):
    if len(r) >= 15 and r[0] != "ID":
        keep.append(f"{r[4][:60]} | {r[12]} | {r[13]} = {r[15] if len(r) > 15 else ''} {r[14]}")
raw = ncu("--page", "raw", "--csv", "--metrics",
          "dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,gpu__time_duration.sum,"
          "sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum")
with open(out + "_details.txt", "w") as f:
    f.write("\n".join(keep) + "\n\n== raw\n" + raw)
src = ncu("--page", "source", "--csv", "--print-source", "cuda,sass")
with open("/tmp/_src.csv", "w") as f:
    f.write(src)
lines = subprocess.run([sys.executable, "tools/ncu_lines.py", "/tmp/_src.csv", "40"],
                       capture_output=True, text=True).stdout
with open(out + "_lines.txt", "w") as f:
    f.write(lines)
print(open(out + "_details.txt").read()[:3000])
