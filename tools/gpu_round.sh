timeout 900 python -m pytest tests/test_heap_gpu.py tests/test_heap_big_gpu.py -q -x 2>&1 | tail -2
timeout 600 python tools/probe_trace.py c1 fill 2>&1 | grep -o '"name": "[a-z0-9_^]*"\|"us_per_op": [0-9.]*'
