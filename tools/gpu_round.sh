set -x
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sssp_bank -c 1 -o gpurun_out/bank_final python tools/probe.py band_small > gpurun_out/bank_final.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum -k regex:k_trace_bank --csv --log-file gpurun_out/tb_l.csv python tools/probe_trace.py c1 > /dev/null 2>&1
SKIP=$(python -c "
import csv
rows=[r for r in csv.reader(open('gpurun_out/tb_l.csv')) if len(r)>10]
h=rows[0]; vi=h.index('Metric Value')
d=[float(r[vi].replace(',','')) for r in rows[1:]]
print(max(range(len(d)), key=lambda i:d[i]))")
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_trace_bank --launch-skip $SKIP -c 1 -o gpurun_out/tbank_final python tools/probe_trace.py c1 > gpurun_out/tbank_final.log 2>&1
timeout 900 python tools/bench_suite.py c1 --c1-ops 1000000 --c1-cpu-ops 2000 > gpurun_out/suite_c1m.json 2> gpurun_out/suite_c1m.log
tail -n 2 gpurun_out/*.log | cut -c1-400
