timeout 600 python -m pytest tests/test_heap_gpu.py tests/test_heap_big_gpu.py tests/test_boundary_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -2
PBH_PROF=1 timeout 300 python tools/probe_c4.py --ds 32,1024,65536 --c1 20000 2>&1 | grep "cfg\|jobprof\[run_ops"
timeout 300 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python tools/sanitize.py big storm 2>&1 | tail -4
