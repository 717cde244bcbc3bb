timeout 600 python -m pytest tests/test_multi_gpu.py tests/test_trace_io.py tests/test_bf_gpu.py -x -q 2>&1 | tail -15
