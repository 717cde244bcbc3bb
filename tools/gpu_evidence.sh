# evidence after the merge-tile and check+classify changes: GPU tests, smoke, bench N=1, launch list
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r02_final4_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_final4_gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_final4_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r02_final4_smoke.log
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_final4_bench.json 2> gpurun_out/r02_final4_bench.err; echo "bench rc=$?" >> gpurun_out/r02_final4_bench.err
tail -n2 gpurun_out/r02_final4_gputest.log; tail -n2 gpurun_out/r02_final4_smoke.log; tail -n1 gpurun_out/r02_final4_bench.err
