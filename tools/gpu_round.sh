ncu --set full --import-source on --clock-control none -k regex:k_sssp_bank -c 1 -o gpurun_out/grid5 python tools/probe.py grid_small > gpurun_out/grid5.log 2>&1
tail -1 gpurun_out/grid5.log
