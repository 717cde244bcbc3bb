# ncu --set full of the C4 d = 65536 op-engine launches (prefill run_trace + drain, timed run_ops)
export PYTHONPATH=.
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_trace_bank -c 4 -o /tmp/c4v2 -f python tools/probe_c4.py --ds 65536 --batches 64 --c1 0 > gpurun_out/c4v2.log 2>&1; echo ncu=$?
python tools/ncu_summarize.py /tmp/c4v2.ncu-rep gpurun_out/r02_ncu_c4_d65536_v2
ncu -i /tmp/c4v2.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum > gpurun_out/r02_ncu_c4_d65536_v2_raw.csv 2>&1
ls -la gpurun_out | grep c4
