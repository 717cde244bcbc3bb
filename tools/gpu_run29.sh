export PYTHONPATH=$PWD
for w in big storm api; do
  timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard --error-exitcode 9 python tools/sanitize.py $w > gpurun_out/r02_racecheck_$w.log 2>&1; echo "racecheck $w rc=$?"
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard" gpurun_out/r02_racecheck_$w.log | sort | uniq -c | head -8
done
timeout 1200 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python tools/sanitize.py big storm api sssp trace thr > gpurun_out/r02_memcheck_all.log 2>&1; echo "memcheck all rc=$?"; tail -2 gpurun_out/r02_memcheck_all.log
