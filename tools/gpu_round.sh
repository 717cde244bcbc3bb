set -x
for nw in 4 1 8; do
PBH_SSSP_NW=$nw timeout 900 python -m pytest tests/test_sssp_gpu.py -x -q > gpurun_out/pytest_sssp_nw$nw.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_sssp_nw$nw.log
PBH_SSSP_NW=$nw timeout 300 python tools/probe.py band_small band band64 grid_small > gpurun_out/probe_nw$nw.log 2>&1
done
tail -n 6 gpurun_out/*.log
