"""The reference's acceptance gate at its stated sizes, on the B200.

Criterion 1 (acceptance_main.cpp:57-107): 100 legal traces x 100k ops,
d = {1, 4, 64}[t % 3], seeds 1000 + t; the extraction sequence must equal
the model's (run_oracle, tests/oracle.hpp:55-75 — restated in oracle/ and
pinned to the reference by tests/test_oracle.py) and the structure must pass
its invariant audit at rest. (The workers column of the reference only
varies its thread count; results are worker-independent.)

Criterion 5 (acceptance_main.cpp:140-181): the random density grid
v in {256, 1024, 4096} x e/v in {4, 32, 256} exactly, plus the families of
tests/test_sssp_gpu.py.
"""
import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.mark.parametrize("block", range(10))
def test_criterion1_trace_suite(pbh, O, block):
    for t in range(10 * block, 10 * block + 10):
        d = (1, 4, 64)[t % 3]
        tr = O.gen_legal_trace(100_000, d, 1000 + t)
        want_v, want_p = O.run_oracle(tr)
        eng = pbh.Engine(pbh.EngineConfig(d=d, workers=(1, 4)[t % 2], debug_assertions=True))
        try:
            got = eng.run_trace(tr)
            assert np.array_equal(got.extracted_values, want_v), f"trace {t} diverged"
            assert np.array_equal(got.extracted_priorities, want_p), f"trace {t} diverged"
            assert eng.check_invariants() == [], f"trace {t}"
        finally:
            eng.close()


@pytest.mark.parametrize("v", [256, 1024, 4096])
@pytest.mark.parametrize("epv", [4, 32, 256])
def test_criterion5_random_density_grid(pbh, O, v, epv):
    e = min(epv * v, v * (v - 1))
    g = O.gen_random(v, e, 1000, v + epv)
    want = O.dijkstra(g, 0)
    got = pbh.par_dijkstra(g, 0)
    assert np.array_equal(got.dist, want["dist"])
    assert np.array_equal(got.settled_order, want["settled_order"])
    assert (got.rounds, got.ops) == (want["rounds"], want["ops"])
    assert pbh.validate_parent_tree(g, 0, got.dist, got.parent, optimal=True) is None
