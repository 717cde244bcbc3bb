# round-end style evidence: GPU tests, smoke, bench N=1 (driver-like K/W), reference arm,
# 2-rank functional bench on one GPU, ncu launch list of the bench command
set -x
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r02_final2_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_final2_gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_final2_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r02_final2_smoke.log
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_final2_bench.json 2> gpurun_out/r02_final2_bench.err; echo "bench rc=$?" >> gpurun_out/r02_final2_bench.err
timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02_final2_ref.json 2> gpurun_out/r02_final2_ref.err; echo "ref rc=$?" >> gpurun_out/r02_final2_ref.err
timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --legs none --no-cpu-baseline > gpurun_out/r02_final2_bench_2rank.json 2> gpurun_out/r02_final2_bench_2rank.err; echo "bench2 rc=$?" >> gpurun_out/r02_final2_bench_2rank.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_final2_launches.csv python bench.py --steps 3 --warmup 3 --legs none --no-cpu-baseline > gpurun_out/r02_final2_launches.log 2>&1
tail -2 gpurun_out/r02_final2_gputest.log; tail -2 gpurun_out/r02_final2_smoke.log; tail -1 gpurun_out/r02_final2_bench.err; tail -1 gpurun_out/r02_final2_ref.err; tail -1 gpurun_out/r02_final2_bench_2rank.err
python tools/launch_summary.py gpurun_out/r02_final2_launches.csv > gpurun_out/r02_final2_launches.txt 2>&1
