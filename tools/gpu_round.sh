set -x
timeout 1200 python tools/bench_suite.py thr > gpurun_out/suite_thr.json 2> gpurun_out/suite_thr.log
tail -n 4 gpurun_out/suite_thr.log | cut -c1-400
