timeout 300 python -c "
import sys, json; sys.path.insert(0,'.')
import bench, paper_1908_09378_b200 as P
print(json.dumps(bench.leg_api_latency(P, 0, 1000)))
"
