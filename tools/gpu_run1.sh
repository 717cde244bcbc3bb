set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider --durations=15 > gpurun_out/r02_gputest1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_gputest1.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02_bench1.log 2> gpurun_out/r02_bench1.err; echo "bench rc=$?" >> gpurun_out/r02_bench1.log
timeout 600 python bench.py --gpus 2 --steps 2 --warmup 1 --legs none --no-cpu-baseline > gpurun_out/r02_bench2.log 2> gpurun_out/r02_bench2.err; echo "bench2 rc=$?" >> gpurun_out/r02_bench2.log
tail -5 gpurun_out/r02_gputest1.log; tail -c 3000 gpurun_out/r02_bench1.log; tail -c 1500 gpurun_out/r02_bench2.log; tail -20 gpurun_out/r02_bench2.err
