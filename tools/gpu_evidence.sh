# evidence of the final state (tests, smoke, bench): GPU tests, smoke, bench N=1, launch list
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r02_final6_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_final6_gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_final6_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r02_final6_smoke.log
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_final6_bench.json 2> gpurun_out/r02_final6_bench.err; echo "bench rc=$?" >> gpurun_out/r02_final6_bench.err
timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02_final6_ref.json 2> gpurun_out/r02_final6_ref.err; echo "ref rc=$?" >> gpurun_out/r02_final6_ref.err
tail -n2 gpurun_out/r02_final6_gputest.log; tail -n2 gpurun_out/r02_final6_smoke.log; tail -n1 gpurun_out/r02_final6_bench.err
