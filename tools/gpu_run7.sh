PBH_PROF=1 timeout 600 python tools/probe_c4.py --ds 32,256,1024,8192,65536 --c1 20000 2>&1 | grep "run_ops\|cfg\|C1\|run_trace"
timeout 900 python -m pytest tests/test_heap_gpu.py tests/test_heap_big_gpu.py tests/test_boundary_gpu.py tests/test_acceptance_gpu.py -q -x -k "not density" 2>&1 | tail -2
timeout 600 python -m pytest tests/test_full_size_gpu.py -q -x -k c4 2>&1 | tail -2
