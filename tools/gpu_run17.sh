timeout 300 python -c "
import sys, json; sys.path.insert(0,'.')
import bench, paper_1908_09378_b200 as P
print(json.dumps(bench.leg_api_latency(P, 0, 1000)))
"
timeout 600 python -m pytest tests/test_heap_gpu.py tests/test_heap_big_gpu.py tests/test_boundary_gpu.py tests/test_cpp_shim.py -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 300 python tools/probe_c4.py --ds 32,1024,65536 --c1 20000 2>&1 | grep "cfg"
