for r in 1 2; do
  timeout 900 python bench.py --steps 3 --warmup 3 --legs c1 --no-cpu-baseline 2>/dev/null | python -c "
import sys, json
d=json.loads(sys.stdin.readline()); print('bench c1', d['c1_op_trace']['us_per_op'])"
done
for v in 0 5; do PBH_AB_OFF=$v timeout 900 python bench.py --steps 3 --warmup 3 --legs c2,c1 --no-cpu-baseline 2>/dev/null | python -c "
import sys, json
d=json.loads(sys.stdin.readline()); print('bench c2,c1 ab=$v', d['c1_op_trace']['us_per_op'])"; done
