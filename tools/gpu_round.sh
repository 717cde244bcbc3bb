# one GPU round-trip: tests, probes, profiles (outputs under gpurun_out/)
set -x
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
PBH_XP=16 PBH_PHASES=1 timeout 300 python tools/probe.py band_small band > gpurun_out/phases.log 2>&1
timeout 600 python tools/probe_trace.py c1 fill > gpurun_out/trace_probe.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sssp -c 1 -o gpurun_out/sssp_small_full python tools/probe.py band_small > gpurun_out/sssp_small_full.log 2>&1
tail -n 3 gpurun_out/*.log
