timeout 300 python -m pytest tests/test_heap_big_gpu.py tests/test_heap_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1
PBH_PROF=1 timeout 300 python tools/probe_c4.py --ds 1024,65536 --c1 20000 2>&1 | grep "run_ops\]\|cfg\|C1\|jobprof\[run_ops"
ncu --set full --import-source on --clock-control none -k regex:k_trace_bank --launch-skip 2 --launch-count 1 -o gpurun_out/r02_ncu_c4_d65536_tma python tools/probe_c4.py --ds 65536 --batches 16 > gpurun_out/r02_ncu_c4_tma.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_trace_bank --launch-count 1 -o gpurun_out/r02_ncu_c1_20k python tools/probe_c4.py --ds "" --c1 20000 > gpurun_out/r02_ncu_c1.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_sssp_multi --launch-count 1 -o gpurun_out/r02_ncu_k_sssp_multi_grid1024 python tools/probe_sssp.py threshold grid 1024 > gpurun_out/r02_ncu_multi.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_bellman_ford --launch-count 1 -o gpurun_out/r02_ncu_k_bellman_ford_grid1024 python tools/probe_sssp.py bf grid 1024 > gpurun_out/r02_ncu_bf.log 2>&1
python tools/probe_sssp.py threshold grid 1024 2; python tools/probe_sssp.py bf grid 1024 2; python tools/probe_sssp.py exact grid 1024 2
ls -la gpurun_out/*.ncu-rep
