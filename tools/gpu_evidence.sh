# evidence of the final state (tests, smoke, bench): GPU tests, smoke, bench N=1, launch list
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r02_final5_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_final5_gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_final5_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r02_final5_smoke.log
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_final5_bench.json 2> gpurun_out/r02_final5_bench.err; echo "bench rc=$?" >> gpurun_out/r02_final5_bench.err
tail -n2 gpurun_out/r02_final5_gputest.log; tail -n2 gpurun_out/r02_final5_smoke.log; tail -n1 gpurun_out/r02_final5_bench.err
