"""Boundary behaviour on the B200 through the C-ABI: the CSR input contract
(validate_graph, graphs.cpp:55-72, and the SSSP entry points' out-of-bounds
guard), max_out_degree (graphs.cpp:47-53), load_graph's shape check before
any state changes, remembered out-of-index deletes (bucket_heap.cpp:55-58,
113-125) and the batch limit."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def csr(V, rows):
    """rows: {u: [(t, w), ...]} -> (offsets, targets, weights) as given (no sorting)."""
    off = [0]
    tgt, w = [], []
    for u in range(V):
        for t, x in rows.get(u, []):
            tgt.append(t)
            w.append(x)
        off.append(len(tgt))
    from paper_1908_09378_b200 import CsrGraph
    return CsrGraph(V, np.array(off, np.uint64), np.array(tgt, np.uint32), np.array(w, np.uint32))


@pytest.mark.parametrize("rows,msg", [
    ({0: [(1, 1), (5, 1)]}, "graph: target out of range"),
    ({0: [(0, 1)]}, "graph: self-loop"),
    ({0: [(2, 1), (1, 1)]}, "graph: row not sorted or parallel edge"),
    ({0: [(1, 1), (1, 2)]}, "graph: row not sorted or parallel edge"),
    ({1: [(2, 0)]}, "graph: zero weight"),
])
def test_validate_graph_messages(pbh, rows, msg):
    g = csr(4, rows)
    with pytest.raises(pbh.InvariantError, match=msg):
        pbh.validate_graph(g)


def test_validate_graph_first_violation_wins(pbh):
    # vertex 1 has a zero weight, vertex 3 a bad target: the reference's
    # sequential loop reports vertex 1 first
    g = csr(4, {1: [(2, 0)], 3: [(9, 1)]})
    with pytest.raises(pbh.InvariantError, match="zero weight"):
        pbh.validate_graph(g)


def test_validate_graph_sizes_and_monotone(pbh):
    from paper_1908_09378_b200 import CsrGraph
    g = CsrGraph(3, np.array([0, 2, 1, 2], np.uint64), np.array([1, 2], np.uint32),
                 np.array([1, 1], np.uint32))
    with pytest.raises(pbh.InvariantError, match="offsets not monotone"):
        pbh.validate_graph(g)
    g = CsrGraph(2, np.array([1, 1, 1], np.uint64), np.array([1], np.uint32), np.array([1], np.uint32))
    with pytest.raises(pbh.InvariantError, match="inconsistent array sizes"):
        pbh.validate_graph(g)


def test_validate_graph_clean_generators(pbh, O):
    for g in (O.gen_random(500, 4000, 9, 1), O.gen_high_diameter(300, 3000, 9, 2),
              O.gen_dag(400, 8, 9, 3), O.gen_complete(64, 9, 4), O.gen_grid(32, 32, 1),
              O.gen_band(1024, 64, 2)):
        pbh.validate_graph(g)


def test_max_out_degree_host_and_device(pbh, O):
    import torch
    g = O.gen_random(500, 4000, 9, 1)
    want = int(np.max(np.diff(g.off)))
    assert pbh.max_out_degree(g) == want
    from paper_1908_09378_b200.gen import DeviceCsr
    dg = DeviceCsr(g.V, torch.from_numpy(g.off.view(np.int64)).cuda(),
                   torch.from_numpy(g.tgt.view(np.int32)).cuda(),
                   torch.from_numpy(g.w.view(np.int32)).cuda())
    assert pbh.max_out_degree(dg) == want


def test_sssp_rejects_out_of_range_target(pbh):
    g = csr(4, {0: [(1, 1)], 1: [(7, 2)]})
    with pytest.raises(pbh.PreconditionError, match="target out of range"):
        pbh.par_dijkstra(g, 0)
    # the device is still usable (no illegal-address fault)
    r = pbh.par_dijkstra(csr(3, {0: [(1, 1)], 1: [(2, 2)]}), 0)
    assert r.dist.tolist() == [0, 1, 3]


def test_bellman_ford_rejects_out_of_range_target(pbh):
    with pytest.raises(pbh.PreconditionError, match="target out of range"):
        pbh.bellman_ford(csr(3, {0: [(3, 1)]}), 0)


def test_load_graph_shape_check_keeps_context(pbh, O):
    g = O.gen_band(2048, 32, 2)
    ctx = pbh.SsspContext(g, max_sources=1)
    try:
        # same V and E, different max out-degree: rejected before any copy
        off = np.arange(g.V + 1, dtype=np.uint64) * 32
        off[1:g.V // 2 + 1] = np.arange(1, g.V // 2 + 1, dtype=np.uint64) * 31
        off[g.V // 2 + 1:] = off[g.V // 2] + np.arange(1, g.V // 2 + 1, dtype=np.uint64) * 33
        bad = pbh.CsrGraph(g.V, off, g.tgt, g.w)
        with pytest.raises(pbh.PreconditionError, match="max out-degree"):
            ctx.load_graph(bad)
        ctx.run([0])
        assert np.array_equal(ctx.fetch(0).dist, O.dijkstra(g, 0)["dist"])
        # same shape, a target out of range: the context refuses to run until
        # a valid graph is loaded again
        t2 = g.tgt.copy()
        t2[5] = g.V + 3
        with pytest.raises(pbh.PreconditionError, match="target out of range"):
            ctx.load_graph(pbh.CsrGraph(g.V, g.off, t2, g.w))
        with pytest.raises(pbh.PreconditionError, match="no valid graph"):
            ctx.run([0])
        ctx.load_graph(g)
        ctx.run([0])
        assert np.array_equal(ctx.fetch(0).dist, O.dijkstra(g, 0)["dist"])
    finally:
        ctx.close()


def test_out_of_universe_delete_is_remembered(pbh):
    eng = pbh.Engine(pbh.EngineConfig(d=4, key_universe=64))
    try:
        eng.delete_value(1000)  # absent: a no-op ...
        assert eng.live_size() == 0
        eng.update((5, 7))
        with pytest.raises(pbh.PreconditionError):  # ... but a dead value afterwards
            eng.update((1000, 3))
        assert tuple(eng.extract_min()) == (5, 7)
        eng.update((2000, 1))  # never deleted: the index grows, insert succeeds
        assert tuple(eng.extract_min()) == (2000, 1)
    finally:
        eng.close()


def test_many_out_of_universe_deletes(pbh):
    # more remembered deletes than the list holds: the index grows instead
    eng = pbh.Engine(pbh.EngineConfig(d=8, key_universe=64))
    try:
        class T:
            pass
        t = T()
        n = 5000
        t.kinds = np.full(n, ord("D"), np.uint8)
        t.offsets = np.arange(n + 1, dtype=np.uint64)
        t.vals = (np.arange(n, dtype=np.uint32) * 3 + 100)
        t.prios = np.zeros(n, np.uint64)
        eng.run_trace(t)
        for v in (100, 103, 100 + 3 * (n - 1)):
            with pytest.raises(pbh.PreconditionError):
                eng.update((v, 1))
        eng.update((101, 1))
        assert tuple(eng.extract_min()) == (101, 1)
    finally:
        eng.close()


def test_batch_limit(pbh):
    eng = pbh.Engine(pbh.EngineConfig(d=(1 << 26) + 8, key_universe=1 << 10))
    try:
        class T:
            pass
        t = T()
        n = (1 << 26) + 1
        t.kinds = np.array([ord("B")], np.uint8)
        t.offsets = np.array([0, n], np.uint64)
        t.vals = np.arange(n, dtype=np.uint32)
        t.prios = np.ones(n, np.uint64)
        with pytest.raises(pbh.TraceError, match="batch limit") as ei:
            eng.run_trace(t)
        assert ei.value.op_index == 0
        with pytest.raises(pbh.PreconditionError, match="batch limit"):
            eng.bulk_update(values=t.vals, priorities=t.prios)
        assert eng.live_size() == 0
    finally:
        eng.close()


def test_bulk_update_pairs_not_columnar(pbh):
    # a 2-element batch of pairs is two elements, not (values, priorities)
    eng = pbh.Engine(pbh.EngineConfig(d=4))
    try:
        eng.bulk_update(((1, 5), (2, 6)))
        assert tuple(eng.extract_min()) == (1, 5)
        assert tuple(eng.extract_min()) == (2, 6)
    finally:
        eng.close()
