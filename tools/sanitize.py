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
if "big" in which:
    # grid paths: big batches (check+classify, bucket sort), grid / streamed
    # merges with TMA windows, flush bucket sorts
    tr = O.gen_mixed_trace(60, 1 << 15, 9000, 3)
    e = P.Engine(P.EngineConfig(d=9000, debug_assertions=False, key_universe=1 << 15))
    got = e.run_trace(tr)
    wv, wp = O.run_oracle(tr)
    assert np.array_equal(got.extracted_values, wv)
    e.close()
    tr = O.gen_mixed_trace(300, 1 << 16, 1024, 4)
    e = P.Engine(P.EngineConfig(d=1024, debug_assertions=False, key_universe=1 << 16))
    got = e.run_trace(tr)
    wv, wp = O.run_oracle(tr)
    assert np.array_equal(got.extracted_values, wv)
    e.close()
    print("big ok")
if "storm" in which:
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
    from test_heap_gpu import _decrease_storm
    tr = _decrease_storm(1 << 12, 1024, 6, 7)
    e = P.Engine(P.EngineConfig(d=1024, debug_assertions=False, key_universe=1 << 12))
    got = e.run_trace(tr)
    wv, wp = O.run_oracle(tr)
    assert np.array_equal(got.extracted_values, wv)
    print("storm ok", e.stats())
if "api" in which:
    e = P.Engine(P.EngineConfig(d=32, debug_assertions=True, key_universe=1 << 10))
    for i in range(200):
        e.update((i, 1000 - i))
    for i in range(0, 200, 3):
        e.delete_value(i)
    e.bulk_update(values=np.arange(300, 332, dtype=np.uint32), priorities=np.arange(32, dtype=np.uint64) + 5)
    n = e.live_size()
    for _ in range(n):
        e.extract_min()
    print("api ok")
