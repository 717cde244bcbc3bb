timeout 900 python -m pytest tests/test_heap_gpu.py tests/test_heap_big_gpu.py tests/test_sssp_gpu.py tests/test_sssp_threshold_gpu.py -q -x 2>&1 | tail -2
PBH_PROF=1 timeout 600 python tools/probe_trace.py c1 fill 2>&1 | grep -o '"us_per_op": [0-9.]*\|pbh_prof.*' | cut -c1-300
timeout 300 python tools/probe.py band_small grid_small 2>&1 | grep -o '"name": "[a-zA-Z0-9_^]*"\|"ns_per_round": [0-9.]*'
