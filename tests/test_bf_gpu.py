"""Device Bellman-Ford baseline (bellman_ford, sssp.cpp:99-129) on the B200.

The reference uses bellman_ford as the cross-check of par_dijkstra
(test_sssp.cpp:92-100: Bellman-Ford's stable sort by distance equals
Dijkstra's settle order). The same checks here: distances bit-exact vs the
oracle's reference_dijkstra, settle order = reached vertices by (dist, vid),
parent tree valid, and agreement with the reference's own bellman_ford
(oracle/_ref) where it is available.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def check(pbh, O, g, source=0):
    want = O.dijkstra(g, source)
    got, scanned, ms = pbh.bellman_ford(g, source)
    assert np.array_equal(got.dist, want["dist"])
    assert np.array_equal(got.settled_order, want["settled_order"])
    assert pbh.validate_parent_tree(g, source, got.dist, got.parent) is None
    assert scanned >= 0 and ms >= 0
    return got


def test_tiny(pbh, O):
    g = O.make_graph(3, [(0, 1, 5), (0, 2, 1), (2, 1, 1)])
    assert check(pbh, O, g).dist.tolist() == [0, 2, 1]


def test_unreachable(pbh, O):
    g = O.make_graph(4, [(0, 1, 3)])
    r = check(pbh, O, g)
    assert int(r.dist[2]) == pbh.K_INF_DIST and int(r.parent[2]) == 0xFFFFFFFF


def test_source_out_of_range(pbh, O):
    g = O.make_graph(2, [(0, 1, 1)])
    with pytest.raises(pbh.PreconditionError):
        pbh.bellman_ford(g, 5)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_random(pbh, O, seed):
    check(pbh, O, O.gen_random(3000, 24000, 1000, seed), source=seed)


def test_tie_heavy(pbh, O):
    check(pbh, O, O.gen_random(2000, 16000, 3, 7))


def test_high_diameter(pbh, O):
    check(pbh, O, O.gen_high_diameter(2000, 10000, 50, 4))


def test_grid(pbh, O):
    check(pbh, O, O.gen_grid(64, 64, 1))


def test_band(pbh, O):
    r = check(pbh, O, O.gen_band(4096, 64, 2))
    assert int(r.dist[4095]) == 4095  # the weight-1 spine


def test_matches_reference_bellman_ford(pbh, O):
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    g = O.gen_random(1500, 9000, 100, 11)
    want = O.ref_sssp(g, 0, algo="bf")
    got, _, _ = pbh.bellman_ford(g, 0)
    assert np.array_equal(got.dist, want["dist"])
    assert np.array_equal(got.settled_order, want["settled_order"])
