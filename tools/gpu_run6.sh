PBH_PROF=1 timeout 600 python tools/probe_c4.py --ds 32,1024,65536 --c1 20000 2>&1 | grep "run_ops\|cfg\|C1\|run_trace"
timeout 600 python -m pytest tests/test_heap_gpu.py -q -x -k run_ops 2>&1 | tail -2
