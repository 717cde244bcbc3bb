PBH_PROF=1 timeout 600 python tools/probe_trace.py c1 fill 2>&1 | grep -o '"us_per_op": [0-9.]*\|push_down [0-9]*\|sort [0-9]*'
timeout 600 python -m pytest tests/test_heap_gpu.py -x -q 2>&1 | tail -1
