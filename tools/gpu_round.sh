timeout 1200 python tools/bench_suite.py bf > /dev/null 2> gpurun_out/bf_final.jsonl; grep '^{' gpurun_out/bf_final.jsonl | cut -c1-400
