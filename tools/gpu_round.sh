timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -1
timeout 1200 python tools/bench_suite.py c2 c3 > /dev/null 2> gpurun_out/suite_c2c3_final.jsonl; grep '^{' gpurun_out/suite_c2c3_final.jsonl | cut -c1-220
