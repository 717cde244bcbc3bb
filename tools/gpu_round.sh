timeout 900 python -m pytest tests/test_sssp_gpu.py -x -q 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; tail -c 200 gpurun_out/bench_final.json; tail -3 gpurun_out/bench_final.err
