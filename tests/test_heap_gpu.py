"""Priority-queue parity on the B200 through the C-ABI.

Restates the reference's own heap and engine tests
(/root/reference/proj/tests/test_bucket_heap.cpp, test_engine.cpp) against
paper_1908_09378_b200.Engine, and checks extraction sequences bit-exactly
against the CPU oracle (run_oracle, tests/oracle.hpp:55-75) on legal random
traces (gen_legal_trace, tests/oracle.hpp:82-155) and BASELINE C1 traces.
"""
import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def E(v, p):
    return (v, p)


def engine(P, d, debug=True, **kw):
    return P.Engine(P.EngineConfig(d=d, workers=1, debug_assertions=debug, **kw))


def settle(eng):
    eng.drain()


# ---- test_bucket_heap.cpp:71-160 ------------------------------------------
def test_construction_rejects_zero_d(pbh):
    with pytest.raises(pbh.PreconditionError):
        engine(pbh, 0)
    with pytest.raises(pbh.PreconditionError):
        engine(pbh, (1 << 40) + 1)


def test_find_min_composite_key(pbh):
    r = engine(pbh, 2)
    r.update(E(7, 3))
    r.update(E(9, 1))
    assert tuple(r.find_min()) == (9, 1)
    tie = engine(pbh, 2)
    tie.update(E(8, 5))
    tie.update(E(2, 5))
    assert tuple(tie.find_min()) == (2, 5)  # equal priorities: smaller value
    empty = engine(pbh, 1)
    with pytest.raises(pbh.EmptyHeapError):
        empty.find_min()
    with pytest.raises(pbh.EmptyHeapError):
        empty.extract_min()


def test_extract_order(pbh):
    r = engine(pbh, 2)
    for v, p in [(10, 3), (11, 1), (12, 2)]:
        r.update(E(v, p))
    assert [tuple(r.extract_min()) for _ in range(3)] == [(11, 1), (12, 2), (10, 3)]
    assert r.live_size() == 0


def test_decrease_takes_effect(pbh):
    r = engine(pbh, 1)
    r.update(E(4, 9))
    r.update(E(4, 5))
    assert r.live_size() == 1
    assert tuple(r.extract_min()) == (4, 5)
    assert r.live_size() == 0


def test_rejects_increase_and_reinsert(pbh):
    r = engine(pbh, 1)
    r.update(E(4, 5))
    with pytest.raises(pbh.PreconditionError):
        r.update(E(4, 9))
    r.extract_min()
    with pytest.raises(pbh.PreconditionError):
        r.update(E(4, 7))


def test_increase_without_checks_keeps_min(pbh):
    # delete_duplicates keeps the min-priority copy (primitives.cpp:25-57)
    r = engine(pbh, 1, debug=False)
    r.update(E(4, 5))
    r.update(E(4, 9))
    assert tuple(r.extract_min()) == (4, 5)


def test_delete_present_and_absent(pbh):
    r = engine(pbh, 2)
    r.update(E(3, 8))
    r.delete_value(3)
    assert r.live_size() == 0
    assert r.check_invariants() == []
    r2 = engine(pbh, 2)
    r2.update(E(3, 8))
    r2.delete_value(99)
    r2.delete_value(0x80000005)  # beyond the index: absent
    assert r2.live_size() == 1
    assert tuple(r2.extract_min()) == (3, 8)


def test_bulk_preconditions(pbh):
    r = engine(pbh, 4)
    r.bulk_update([E(1, 5), E(2, 3), E(9, 8)])
    assert r.live_size() == 3
    assert tuple(r.find_min()) == (2, 3)
    h = engine(pbh, 4)
    with pytest.raises(pbh.PreconditionError):
        h.bulk_update([E(1, 1), E(2, 2), E(3, 3), E(4, 4), E(5, 5)])
    with pytest.raises(pbh.PreconditionError):
        h.bulk_update([E(1, 1), E(1, 2)])
    with pytest.raises(pbh.PreconditionError):
        h.bulk_update([E(2, 1), E(1, 2)])
    with pytest.raises(pbh.PreconditionError):
        h.bulk_update([])


def test_overflow_and_refill_small_d(pbh):
    # d=1: level 0 overflows after cap0 inserts; everything must come back in order
    r = engine(pbh, 1)
    rng = np.random.default_rng(5)
    pr = rng.permutation(3000) + 1
    for v, p in enumerate(pr):
        r.update(E(v, int(p)))
    assert r.check_invariants() == []
    got = [r.extract_min().priority for _ in range(3000)]
    assert got == list(range(1, 3001))


# ---- test_engine.cpp ------------------------------------------------------
def test_engine_round_trip(pbh):
    eng = engine(pbh, 2)
    eng.update(E(5, 10))
    eng.update(E(6, 4))
    assert eng.live_size() == 2
    assert tuple(eng.extract_min()) == (6, 4)
    eng.delete_value(5)
    assert eng.live_size() == 0
    eng.drain()
    assert eng.check_invariants() == []


def test_engine_zero_workers(pbh):
    with pytest.raises(pbh.PreconditionError):
        pbh.Engine(pbh.EngineConfig(d=1, workers=0))


def test_fresh_metrics_zero(pbh):
    m = engine(pbh, 1).snapshot_metrics()
    assert m.ops == 0
    assert all(r == 0 for r in m.resolves_per_level)
    assert all(t == 0 for t in m.touches_per_level)


def test_metrics_json_keys(pbh, O):
    eng = engine(pbh, 2)
    run = eng.run_trace(O.gen_legal_trace(500, 2, 31))
    j = json.loads(run.metrics.to_json())
    assert j["schema"] == "pbh.metrics.v1"
    assert j["ops"] == 500
    assert isinstance(j["resolves_per_level"], list)
    assert isinstance(j["touches_per_level"], list)
    assert "wall_ms" in j


def test_empty_trace(pbh, O):
    eng = engine(pbh, 1)
    run = eng.run_trace(O.Trace([], [0], [], []))
    assert len(run.extracted_values) == 0
    assert run.metrics.ops == 0


def test_trace_error_op_index(pbh, O):
    eng = engine(pbh, 1)
    tr = O.Trace([ord("U"), ord("E"), ord("E")], [0, 1, 1, 1], [1], [5])
    with pytest.raises(pbh.TraceError) as ei:
        eng.run_trace(tr)
    assert ei.value.op_index == 2


def test_drain_leaves_engine_usable(pbh):
    eng = engine(pbh, 2)
    for v in range(100):
        eng.update(E(v, 1000 - v))
    eng.drain()
    assert eng.check_invariants() == []
    assert tuple(eng.extract_min()) == (99, 901)
    for v in range(100, 200):
        eng.update(E(v, 2000 + v))
    eng.drain()
    assert eng.check_invariants() == []
    assert eng.live_size() == 199


def test_bulk_through_engine(pbh):
    eng = engine(pbh, 4)
    eng.bulk_update([E(1, 50), E(2, 40), E(3, 60)])
    eng.bulk_update([E(10, 5)])
    assert tuple(eng.extract_min()) == (10, 5)
    assert tuple(eng.extract_min()) == (2, 40)
    eng.drain()
    assert eng.live_size() == 2


def test_resolve_counts_follow_4_to_1(pbh, O):
    # test_engine.cpp:87-105: resolves of level i ~ n / 4^i for n single updates
    n = 4096
    tr = O.Trace([ord("U")] * n, np.arange(n + 1), np.arange(n),
                 [1 + (i * 40503) % 99991 for i in range(n)])
    eng = engine(pbh, 1)
    eng.run_trace(tr)
    m = eng.snapshot_metrics()
    assert m.ops == n
    assert m.resolves_per_level[0] == n


# ---- oracle equivalence (test_bucket_heap.cpp:213-235, test_engine.cpp:107-119)
def _check_trace(pbh, O, tr, d, debug=True):
    want_v, want_p = O.run_oracle(tr)
    eng = engine(pbh, d, debug=debug)
    got = eng.run_trace(tr)
    assert len(got.extracted_values) == len(want_v)
    bad = np.nonzero((got.extracted_values != want_v) | (got.extracted_priorities != want_p))[0]
    assert len(bad) == 0, f"first mismatch at extraction {bad[0]}"
    assert got.metrics.ops == tr.n_ops
    assert eng.check_invariants() == []


@pytest.mark.parametrize("d", [1, 3, 8])
@pytest.mark.parametrize("seed", range(1, 13))
def test_legal_traces_match_oracle(pbh, O, d, seed):
    _check_trace(pbh, O, O.gen_legal_trace(3000, d, seed * 977), d)


@pytest.mark.parametrize("d", [4, 64, 1000])
def test_long_legal_traces(pbh, O, d):
    _check_trace(pbh, O, O.gen_legal_trace(30000, d, 321 + d), d)


@pytest.mark.parametrize("kmax,d", [(16, 16), (300, 300), (1024, 1024), (4096, 4096)])
def test_mixed_bulk_traces(pbh, O, kmax, d):
    # BASELINE C1 generator at reduced size
    _check_trace(pbh, O, O.gen_mixed_trace(3000, 1 << 16, kmax, 7 + kmax), d, debug=False)


def test_golden_trace_fixtures(pbh):
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "traces.npz")
    z = np.load(path)
    for name in [k[:-6] for k in z.files if k.endswith("_kinds")]:
        d = int(z[name + "_d"])

        class T:
            pass
        t = T()
        t.kinds, t.offsets, t.vals, t.prios = (z[name + "_kinds"], z[name + "_offsets"],
                                               z[name + "_vals"], z[name + "_prios"])
        got = engine(pbh, d).run_trace(t)
        assert np.array_equal(got.extracted_values, z[name + "_out_v"]), name
        assert np.array_equal(got.extracted_priorities, z[name + "_out_p"]), name


@pytest.mark.parametrize("d", [1, 8, 64])
def test_run_ops_matches_run_trace(pbh, O, d):
    # run_ops = the same single-client calls without the closing drain: the
    # extraction sequence is the oracle's, and a later drain + extraction of
    # everything left agrees with run_trace's final state
    tr = O.gen_legal_trace(4000, d, 31 + d)
    want_v, want_p = O.run_oracle(tr)
    eng = pbh.Engine(pbh.EngineConfig(d=d))
    try:
        got = eng.run_ops(tr)
        assert np.array_equal(got.extracted_values, want_v)
        assert np.array_equal(got.extracted_priorities, want_p)
        n_left = eng.live_size()
        eng.drain()
        assert eng.check_invariants() == []
        assert eng.live_size() == n_left
    finally:
        eng.close()


def _decrease_storm(n_keys, d, rounds, seed):
    """Fresh keys, then `rounds` passes of strict decreases over all keys in
    batches of d, then extract everything: most stored entries go stale."""
    rng = np.random.default_rng(seed)
    p = rng.integers(1 << 30, 1 << 31, n_keys).astype(np.uint64)
    kinds, offs, vals, prios = [], [0], [], []

    def bulk(ks):
        kinds.append(ord("B"))
        vals.append(ks.astype(np.uint32))
        prios.append(p[ks].copy())
        offs.append(offs[-1] + len(ks))
    for b in range(0, n_keys, d):
        bulk(np.arange(b, min(n_keys, b + d)))
    for _ in range(rounds):
        for b in range(0, n_keys, d):
            ks = np.arange(b, min(n_keys, b + d))
            p[ks] -= rng.integers(1, 1000, len(ks)).astype(np.uint64)
            bulk(ks)
    for _ in range(n_keys):
        kinds.append(ord("E"))
        offs.append(offs[-1])
    from oracle import oracle as O
    return O.Trace(np.array(kinds, np.uint8), np.array(offs, np.uint64),
                   np.concatenate(vals), np.concatenate(prios))


@pytest.mark.parametrize("n_keys,d,rounds", [(1 << 14, 1024, 12), (1 << 16, 16384, 8)])
def test_filtered_deep_merges_drop_stale(pbh, O, n_keys, d, rounds):
    # repeated decreases of every key make most deep entries stale: the
    # streamed (d=1024) and grid (d=16384) merges then drop them through the
    # position index, and the extraction sequence stays the oracle's
    tr = _decrease_storm(n_keys, d, rounds, 7)
    want_v, want_p = O.run_oracle(tr)
    eng = pbh.Engine(pbh.EngineConfig(d=d, debug_assertions=False, key_universe=n_keys))
    try:
        k = int(np.nonzero(tr.kinds == ord("E"))[0][0])
        head = O.Trace(tr.kinds[:k], tr.offsets[:k + 1], tr.vals, tr.prios)
        eng.run_ops(head)
        st = eng.stats()
        assert st["stale_dropped"] > 0, st
        tail = O.Trace(tr.kinds[k:], tr.offsets[k:] - tr.offsets[k], tr.vals[:0], tr.prios[:0])
        got = eng.run_trace(tail)
        assert np.array_equal(got.extracted_values, want_v)
        assert np.array_equal(got.extracted_priorities, want_p)
        assert eng.check_invariants() == []
    finally:
        eng.close()
