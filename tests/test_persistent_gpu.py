"""Single-op Engine API in persistent mode (pbh_heap_set_persistent): a
resident k_trace_bank serves update / bulk_update / extract_min / find_min /
delete_value posted through mapped host memory.

Traces are replayed op by op through the per-call API (engine.cpp:90-109)
and the extraction sequence is checked bit-exactly against the oracle
(run_oracle, tests/oracle.hpp:55-75) with the kernel kept resident (idle
200 us), exiting between almost every call (idle 1 us: the relaunch race),
and off (one launch per op). Calls that stop the resident kernel (live_size,
metrics, run_trace) are interleaved.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def replay(P, tr, d, idle_us, universe=1 << 16, probe_every=0, debug=False):
    eng = P.Engine(P.EngineConfig(d=d, debug_assertions=debug, key_universe=universe))
    eng.set_persistent(idle_us)
    out_v, out_p = [], []
    kinds = bytes(np.asarray(tr.kinds, dtype=np.uint8))
    off = np.asarray(tr.offsets)
    vals = np.asarray(tr.vals, dtype=np.uint32)
    prios = np.asarray(tr.prios, dtype=np.uint64)
    for i, k in enumerate(kinds):
        b, e = int(off[i]), int(off[i + 1])
        if k == ord("U"):
            eng.update((int(vals[b]), int(prios[b])))
        elif k == ord("B"):
            eng.bulk_update(values=vals[b:e], priorities=prios[b:e])
        elif k == ord("E"):
            v, p = tuple(eng.extract_min())
            out_v.append(v)
            out_p.append(p)
        elif k == ord("D"):
            eng.delete_value(int(vals[b]))
        if probe_every and i % probe_every == probe_every - 1:
            eng.live_size()
            if i % (2 * probe_every) == 2 * probe_every - 1:
                eng.snapshot_metrics()
    return eng, np.array(out_v, dtype=np.uint32), np.array(out_p, dtype=np.uint64)


def check(P, O, tr, d, idle_us, **kw):
    want_v, want_p = O.run_oracle(tr)
    eng, got_v, got_p = replay(P, tr, d, idle_us, **kw)
    n = len(got_v)
    assert n == len(want_v)
    bad = np.nonzero((got_v != want_v) | (got_p != want_p))[0]
    assert len(bad) == 0, f"first mismatch at extraction {bad[0]} of {n}"
    # what is left comes out in the oracle's order too: the trace extended by
    # one extract per live value
    live = eng.live_size()
    ext = O.Trace(np.concatenate([tr.kinds, np.full(live, ord("E"), np.uint8)]),
                  np.concatenate([tr.offsets, np.full(live, tr.offsets[-1], np.uint64)]),
                  tr.vals, tr.prios)
    all_v, all_p = O.run_oracle(ext)
    rest_v, rest_p = [], []
    for _ in range(live):
        v, p = tuple(eng.extract_min())
        rest_v.append(v)
        rest_p.append(p)
    assert eng.live_size() == 0
    assert np.array_equal(np.array(rest_v, dtype=np.uint32), all_v[n:])
    assert np.array_equal(np.array(rest_p, dtype=np.uint64), all_p[n:])
    assert eng.check_invariants() == []
    eng.close()


@pytest.mark.parametrize("idle_us", [200, 1, 0])
@pytest.mark.parametrize("d", [1, 8, 64])
def test_legal_trace_single_calls(pbh, O, d, idle_us):
    check(pbh, O, O.gen_legal_trace(3000, d, 4242 + d), d, idle_us, debug=True)


@pytest.mark.parametrize("idle_us", [200, 1])
def test_mixed_trace_single_calls(pbh, O, idle_us):
    # C1-shaped batches up to 1024 (those above 256 take the one-shot path
    # and stop the resident kernel); ~150k inserts cross the one-CTA limit
    # (2^16), so the resident kernel is relaunched on the grid
    check(pbh, O, O.gen_mixed_trace(2000, 1 << 16, 1024, 99), 1024, idle_us, probe_every=97)


def test_growth_and_errors_in_persistent_mode(pbh, O):
    # a small key universe: updates beyond it fail inside the resident
    # kernel (KEY_RANGE), which exits; the op is re-run after index growth
    check(pbh, O, O.gen_mixed_trace(600, 1 << 16, 64, 5), 64, 200, universe=1 << 8)
    eng = pbh.Engine(pbh.EngineConfig(d=8, debug_assertions=True))
    eng.set_persistent(200)
    with pytest.raises(pbh.EmptyHeapError):
        eng.extract_min()
    eng.update((5, 50))
    eng.update((3, 30))
    assert tuple(eng.find_min()) == (3, 30)
    eng.update((5, 10))  # decrease
    with pytest.raises(pbh.PreconditionError):
        eng.update((5, 20))  # increase with debug checks
    with pytest.raises(pbh.PreconditionError):
        eng.bulk_update(values=np.array([9, 7], np.uint32), priorities=np.array([1, 1], np.uint64))
    assert tuple(eng.extract_min()) == (5, 10)
    eng.delete_value(3)
    with pytest.raises(pbh.PreconditionError):
        eng.update((3, 1))  # re-insert of a deleted value
    assert eng.live_size() == 0
    eng.update((77, 7))
    assert tuple(eng.extract_min()) == (77, 7)
    eng.close()


def test_set_persistent_rejects_huge_idle(pbh):
    eng = pbh.Engine(pbh.EngineConfig(d=8))
    with pytest.raises(pbh.PreconditionError):
        eng.set_persistent(10 ** 8)
    eng.close()


@pytest.mark.timeout(300)
def test_two_resident_engines_and_sssp_interleaved(pbh, O):
    # two heaps alternate call by call (each call waits for the other heap's
    # resident kernel to go idle), with an SSSP solve on the same device in
    # between: every result still matches the oracle
    from paper_1908_09378_b200 import gen
    tr_a = O.gen_legal_trace(400, 8, 11)
    tr_b = O.gen_legal_trace(400, 8, 12)
    want_a, _ = O.run_oracle(tr_a)
    want_b, _ = O.run_oracle(tr_b)
    engs = [pbh.Engine(pbh.EngineConfig(d=8, debug_assertions=True)) for _ in range(2)]
    outs = [[], []]
    g = gen.grid(32, 32, 3)
    want_dist = O.dijkstra(O.Graph(g.vertex_count, g.offsets, g.targets, g.weights), 0)["dist"]
    for i in range(max(tr_a.n_ops, tr_b.n_ops)):
        for which, tr in enumerate((tr_a, tr_b)):
            if i >= tr.n_ops:
                continue
            k, b = int(tr.kinds[i]), int(tr.offsets[i])
            e = int(tr.offsets[i + 1])
            eng = engs[which]
            if k == ord("U"):
                eng.update((int(tr.vals[b]), int(tr.prios[b])))
            elif k == ord("B"):
                eng.bulk_update(values=tr.vals[b:e], priorities=tr.prios[b:e])
            elif k == ord("E"):
                outs[which].append(tuple(eng.extract_min())[0])
            elif k == ord("D"):
                eng.delete_value(int(tr.vals[b]))
        if i == 200:
            r = pbh.par_dijkstra(g, 0)
            assert np.array_equal(np.asarray(r.dist), want_dist)
    assert np.array_equal(np.array(outs[0], np.uint32), want_a)
    assert np.array_equal(np.array(outs[1], np.uint32), want_b)
    for eng in engs:
        eng.close()


def test_resident_kernel_idle_exit_and_modes(pbh):
    import time
    eng = pbh.Engine(pbh.EngineConfig(d=8, debug_assertions=True))
    eng.set_persistent(1000000)  # 1 s: two quick calls share one resident kernel
    eng.update((1, 10))
    eng.update((2, 20))
    assert eng.persist_profile()["launches"] == 1
    eng.set_persistent(50)  # stops the resident kernel; 50 us idle from now on
    eng.update((3, 30))
    time.sleep(0.02)  # the kernel exits after 50 us without a request
    eng.update((4, 40))
    pp = eng.persist_profile()
    assert pp["launches"] == 3 and pp["requests"] == 4
    eng.set_persistent(0)  # one launch per call: no resident kernel
    assert tuple(eng.extract_min()) == (1, 10)
    assert eng.persist_profile()["launches"] == 3
    assert eng.live_size() == 3
    eng.close()


def test_close_while_resident_then_reuse_device(pbh, O):
    # destroy with the resident kernel still running (it is stopped and its
    # state saved first), then a new heap on the same device works
    for _ in range(3):
        eng = pbh.Engine(pbh.EngineConfig(d=4, debug_assertions=True))
        eng.set_persistent(1000000)
        for v in range(50):
            eng.update((v, 1000 - v))
        assert tuple(eng.extract_min()) == (49, 951)
        eng.close()  # no other call in between: the kernel is resident here
    tr = O.gen_legal_trace(500, 4, 77)
    check(pbh, O, tr, 4, 200, debug=True)
