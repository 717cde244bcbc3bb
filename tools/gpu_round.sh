timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
PBH_SSSP_ENGINE=cta PBH_TRACE_ENGINE=cta timeout 900 python -m pytest tests/test_sssp_gpu.py tests/test_heap_gpu.py -q 2>&1 | tail -2
