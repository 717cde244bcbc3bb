timeout 1500 python tools/bench_suite.py c1 --c1-ops 1000000 > /dev/null 2> gpurun_out/c1_full_r1c.jsonl; grep '^{' gpurun_out/c1_full_r1c.jsonl | cut -c1-250
timeout 2400 python tools/bench_suite.py c4 --c4-n 26 > /dev/null 2> gpurun_out/c4_26_r1c.jsonl; grep '^{' gpurun_out/c4_26_r1c.jsonl | grep -o '"d": [0-9]*\|"updates_per_s": [0-9.]*\|"us_per_batch": [0-9.]*' | paste - - -
