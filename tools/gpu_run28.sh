timeout 600 python -m pytest tests/test_heap_gpu.py tests/test_heap_big_gpu.py tests/test_full_size_gpu.py -q -x -k "not c1 and not c2 and not c3 and not c5" -p no:cacheprovider 2>&1 | tail -2
for r in 1 2; do timeout 300 python tools/probe_c4.py --ds 8192,65536 --c1 20000 2>&1 | grep cfg | cut -c1-160; done
PBH_PROF=1 timeout 300 python tools/probe_c4.py --ds 65536 2>&1 | grep "jobprof\[run_ops"
