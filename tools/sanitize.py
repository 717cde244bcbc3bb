"""Small SSSP / op-trace / threshold runs for compute-sanitizer (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1908_09378_b200 as P
from oracle import oracle as O
which = sys.argv[1:] or ["sssp", "trace", "thr"]
if "sssp" in which:
    for g, s in [(O.gen_band(2048, 64, 2), 0), (O.gen_random(1500, 12000, 100, 3), 1), (O.gen_grid(40, 40, 1), 0)]:
        r = P.par_dijkstra(g, s)
        assert np.array_equal(r.dist, O.dijkstra(g, s)["dist"])
    print("sssp ok")
if "trace" in which:
    tr = O.gen_legal_trace(3000, 64, 5)
    e = P.Engine(P.EngineConfig(d=64, debug_assertions=True))
    got = e.run_trace(tr)
    wv, wp = O.run_oracle(tr)
    assert np.array_equal(got.extracted_values, wv)
    print("trace ok")
if "thr" in which:
    g = O.gen_grid(40, 40, 1)
    r = P.threshold_sssp(g, 0)
    assert np.array_equal(r.dist, O.dijkstra(g, 0)["dist"])
    print("thr ok")
