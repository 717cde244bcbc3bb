timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
timeout 2400 python tools/bench_suite.py c4 --c4-n 26 > /dev/null 2> gpurun_out/c4_26_final.jsonl; grep '^{' gpurun_out/c4_26_final.jsonl | grep -o '"d": [0-9]*\|"updates_per_s": [0-9.]*\|"us_per_batch": [0-9.]*' | paste - - -
