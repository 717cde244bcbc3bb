timeout 900 compute-sanitizer --tool racecheck --print-limit 40 python tools/sanitize.py sssp > gpurun_out/race.log 2>&1
grep -c "Race reported" gpurun_out/race.log
grep -A1 "Race reported" gpurun_out/race.log | grep -o "at [^ ]*+0x[0-9a-f]* in [a-z_.]*:[0-9]*" | sort | uniq -c | sort -rn | head -20
