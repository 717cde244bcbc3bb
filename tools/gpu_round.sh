timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --clock-control none -k regex:k_sssp_bank -c 3 --csv --log-file gpurun_out/c5_dram_r2.csv python tools/probe.py band band64 > gpurun_out/c5_dram_r2.log 2>&1
tail -3 gpurun_out/c5_dram_r2.log
