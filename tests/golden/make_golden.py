"""Generate the golden fixtures from the UNMODIFIED reference (oracle/_ref).

Run in the build container (needs /root/reference to build oracle/_ref):
    python tests/golden/make_golden.py
Writes tests/golden/traces.npz and tests/golden/sssp.npz. Every array comes
from the reference library itself: traces from pbh::testing::gen_legal_trace
(tests/oracle.hpp:82-155), extraction sequences from pbh::Engine::run_trace
(engine.cpp:207-226) cross-checked against pbh::testing::run_oracle, graphs
from the reference generators (graphs.cpp:74-186) and distances / settled
order from pbh::par_dijkstra (sssp.cpp:21-69) cross-checked against
pbh::reference_dijkstra (sssp.cpp:71-97).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import oracle as O  # noqa: E402


def traces():
    out = {}
    cases = [("legal_d1_s977", 2000, 1, 977), ("legal_d3_s1954", 2000, 3, 1954),
             ("legal_d8_s2931", 2000, 8, 2931), ("legal_d64_s1002", 5000, 64, 1002),
             ("legal_d4_s321", 10000, 4, 321)]
    for name, n, d, seed in cases:
        tr = O.ref_gen_legal_trace(n, d, seed)
        v, p, m = O.ref_run_trace(tr, d)
        ov, op = O.ref_run_oracle(tr)
        assert np.array_equal(v, ov) and np.array_equal(p, op), name
        out[name + "_kinds"] = tr.kinds
        out[name + "_offsets"] = tr.offsets
        out[name + "_vals"] = tr.vals
        out[name + "_prios"] = tr.prios
        out[name + "_out_v"] = v
        out[name + "_out_p"] = p
        out[name + "_d"] = np.array(d)
        out[name + "_ops"] = np.array(m["ops"])
    np.savez_compressed(os.path.join(HERE, "traces.npz"), **out)


def sssp():
    out = {}
    cases = [("random_200_1600_s1", ("random", 200, 1600, 50, 1), False),
             ("random_128_1024_s9", ("random", 128, 1024, 30, 9), False),
             ("highdiam_1024", ("highdiam", 1024, 10240, 100, 3), False),
             ("dag_512_4", ("dag", 512, 4, 40, 9), True),
             ("complete_64", ("complete", 64, 0, 1000, 64), False),
             ("random_tie_2000", ("random", 2000, 16000, 3, 100), False)]
    for name, args, dag in cases:
        g = O.ref_graph(*args)
        r = O.ref_sssp(g, 0, "par", dag_mode=dag)
        w = O.ref_sssp(g, 0, "ref")
        assert np.array_equal(r["dist"], w["dist"]) and np.array_equal(r["settled_order"], w["settled_order"])
        out[name + "_off"] = g.off
        out[name + "_tgt"] = g.tgt
        out[name + "_w"] = g.w
        out[name + "_dist"] = r["dist"]
        out[name + "_settled"] = r["settled_order"]
        out[name + "_ops"] = np.array(r["ops"])
        out[name + "_dag"] = np.array(dag)
        out[name + "_gen"] = np.array(args[1:], dtype=np.uint64)
    np.savez_compressed(os.path.join(HERE, "sssp.npz"), **out)


if __name__ == "__main__":
    traces()
    sssp()
    print("golden fixtures written")
