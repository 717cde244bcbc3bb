timeout 400 python -m pytest tests/test_heap_big_gpu.py tests/test_heap_gpu.py tests/test_boundary_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -2
PBH_PROF=1 timeout 300 python tools/probe_c4.py --ds 32,1024,8192,65536 --c1 20000 2>&1 | grep "run_ops\]\|cfg\|C1\|jobprof\[run_ops"
timeout 900 python -m pytest tests/test_acceptance_gpu.py tests/test_full_size_gpu.py -q -x -k "not density and not c2 and not c5 and not c3" -p no:cacheprovider 2>&1 | tail -2
