timeout 400 python -m pytest tests/test_heap_gpu.py tests/test_heap_big_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -2
PBH_PROF=1 timeout 300 python tools/probe_c4.py --ds 1024,65536 --c1 20000 2>&1 | grep "cfg\|C1\|jobprof\[run_ops\|jobprof\[destroy"
