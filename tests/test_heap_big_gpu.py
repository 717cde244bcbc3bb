"""Large bulk_update batches (d >= 8192) take the grid path of the op-trace
interpreter: grid validation and classification, grid sort (CTA-sorted chunks
plus merge passes) and one push into S_1. Extraction sequences must stay
bit-exact vs the oracle (run_oracle, tests/oracle.hpp:19-81), and the
preconditions must fail before any mutation (bucket_heap.cpp:127-136)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def engine(P, d, debug=True, **kw):
    return P.Engine(P.EngineConfig(d=d, workers=1, debug_assertions=debug, **kw))


def check(pbh, O, tr, d, debug=True, universe=0):
    want_v, want_p = O.run_oracle(tr)
    eng = engine(pbh, d, debug=debug, key_universe=universe)
    got = eng.run_trace(tr)
    assert len(got.extracted_values) == len(want_v)
    bad = np.nonzero((got.extracted_values != want_v) | (got.extracted_priorities != want_p))[0]
    assert len(bad) == 0, f"first mismatch at extraction {bad[0]}"
    assert eng.check_invariants() == []
    return eng


@pytest.mark.parametrize("seed", [1, 2])
def test_mixed_trace_big_batches(pbh, O, seed):
    # C1-shaped trace with batches of up to 16384 (most take the grid path)
    tr = O.gen_mixed_trace(400, 1 << 18, 16384, seed)
    check(pbh, O, tr, 16384, debug=False, universe=1 << 18)


def test_prefill_then_decrease_sweep_then_drain(pbh, O):
    # C4 shape at small scale: fresh keys in big batches, then big batches of
    # strict decreases, then extract everything
    rng = np.random.default_rng(4)
    n, d = 1 << 16, 12000
    kinds, offs, vals, prios = [], [0], [], []
    p_now = rng.integers(1 << 39, 1 << 40, n, dtype=np.uint64)
    for b in range(0, n, d):
        ks = np.arange(b, min(n, b + d), dtype=np.uint32)
        kinds.append(ord("B"))
        vals.append(ks)
        prios.append(p_now[ks])
        offs.append(offs[-1] + len(ks))
    for _ in range(6):
        ks = np.sort(rng.choice(n, d, replace=False)).astype(np.uint32)
        p_now[ks] -= rng.integers(1, 1025, d).astype(np.uint64)
        kinds.append(ord("B"))
        vals.append(ks)
        prios.append(p_now[ks].copy())
        offs.append(offs[-1] + d)
    for _ in range(n):
        kinds.append(ord("E"))
        offs.append(offs[-1])
    tr = O.Trace(np.array(kinds, np.uint8), np.array(offs, np.uint64),
                 np.concatenate(vals).astype(np.uint32), np.concatenate(prios).astype(np.uint64))
    check(pbh, O, tr, d, debug=True, universe=n)


def test_big_batch_preconditions_do_not_mutate(pbh, O):
    d = 10000
    eng = engine(pbh, d, key_universe=1 << 15)
    good = [pbh.Element(v, 1000 + v) for v in range(d)]
    eng.bulk_update(good)
    bad = [pbh.Element(v, 5) for v in range(d, 2 * d)]
    bad[7000], bad[7001] = bad[7001], bad[7000]  # unsorted in the middle
    with pytest.raises(pbh.PreconditionError):
        eng.bulk_update(bad)
    assert eng.live_size() == d
    inc = [pbh.Element(v, 10 ** 9) for v in range(0, d)]  # priority increase (debug)
    with pytest.raises(pbh.PreconditionError):
        eng.bulk_update(inc)
    assert eng.live_size() == d
    assert tuple(eng.extract_min()) == (0, 1000)
    assert eng.check_invariants() == []
