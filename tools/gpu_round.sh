timeout 900 python bench.py > gpurun_out/bench.log 2>&1
tail -c 2500 gpurun_out/bench.log
