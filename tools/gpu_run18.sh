timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider --durations=10 > gpurun_out/r02_gputest2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_gputest2.log
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/r02_bench2.json 2> gpurun_out/r02_bench2.err; echo "bench rc=$?" >> gpurun_out/r02_bench2.err
timeout 600 python __graft_entry__.py smoke > gpurun_out/r02_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r02_smoke.log
tail -15 gpurun_out/r02_gputest2.log; tail -3 gpurun_out/r02_bench2.err; tail -2 gpurun_out/r02_smoke.log
