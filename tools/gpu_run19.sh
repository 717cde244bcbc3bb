export PYTHONPATH=$PWD
for w in big storm api sssp trace thr; do
  timeout 900 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python tools/sanitize.py $w > gpurun_out/r02_memcheck_$w.log 2>&1; echo "memcheck $w rc=$?" | tee -a gpurun_out/r02_sanitizer.txt
  tail -3 gpurun_out/r02_memcheck_$w.log >> gpurun_out/r02_sanitizer.txt
done
for w in big api; do
  timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize.py $w > gpurun_out/r02_synccheck_$w.log 2>&1; echo "synccheck $w rc=$?" | tee -a gpurun_out/r02_sanitizer.txt
  tail -3 gpurun_out/r02_synccheck_$w.log >> gpurun_out/r02_sanitizer.txt
done
cat gpurun_out/r02_sanitizer.txt
