timeout 700 python -m pytest tests/test_heap_gpu.py tests/test_heap_big_gpu.py tests/test_boundary_gpu.py tests/test_acceptance_gpu.py -v -x -k "not density" --durations=10 -p no:cacheprovider > gpurun_out/r02_t8.log 2>&1; echo "rc=$?" >> gpurun_out/r02_t8.log
tail -40 gpurun_out/r02_t8.log
