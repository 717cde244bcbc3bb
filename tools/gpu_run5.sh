timeout 600 python tools/probe_c4.py --ds 32,256,1024,8192,65536 --batches 0 --c1 20000 2>&1 | grep cfg
timeout 900 python -m pytest tests/test_heap_gpu.py tests/test_heap_big_gpu.py tests/test_boundary_gpu.py tests/test_full_size_gpu.py -q -x -k "not c1_full and not c2 and not c5 and not c3" 2>&1 | tail -3
PBH_PROF=1 timeout 600 python tools/probe_c4.py --ds 8192,65536 2>&1 | grep "run_trace\|cfg" | tail -3
