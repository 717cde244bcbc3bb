set -x
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --clock-control none -k regex:k_sssp_bank --launch-skip 2 -c 1 --csv --log-file gpurun_out/bank_c5_dram.csv python tools/probe.py band band64 > gpurun_out/bank_c5_dram.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_ncu.log 2>&1
cat gpurun_out/bench.log
