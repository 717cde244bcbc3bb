set -x
export PBH_PROF=1
timeout 600 python tools/probe_c4.py --ds 32,256,1024,8192,65536 --c1 20000 > gpurun_out/r02_prof_c4.log 2>&1
unset PBH_PROF
timeout 600 python tools/probe_c4.py --ds 32,1024,65536 --c1 20000 > gpurun_out/r02_probe_c4.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_trace_bank --launch-skip 2 --launch-count 1 -o gpurun_out/r02_ncu_c4_d65536 python tools/probe_c4.py --ds 65536 --batches 16 > gpurun_out/r02_ncu_c4_d65536.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_trace_bank --launch-skip 2 --launch-count 1 -o gpurun_out/r02_ncu_c4_d1024 python tools/probe_c4.py --ds 1024 --batches 256 > gpurun_out/r02_ncu_c4_d1024.log 2>&1
cat gpurun_out/r02_prof_c4.log gpurun_out/r02_probe_c4.log; tail -3 gpurun_out/r02_ncu_c4_d65536.log gpurun_out/r02_ncu_c4_d1024.log
