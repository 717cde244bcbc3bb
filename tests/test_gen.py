"""The product's workload generators (include/pbh_gen.h, C++) must agree draw
for draw with the oracle's independent restatement (oracle/pbh_oracle.c)."""
import numpy as np


def test_grid_matches_oracle(O):
    from paper_1908_09378_b200 import gen
    a = gen.grid(33, 47, 1)
    b = O.gen_grid(33, 47, 1)
    assert np.array_equal(a.offsets, b.off)
    assert np.array_equal(a.targets, b.tgt)
    assert np.array_equal(a.weights, b.w)


def test_band_matches_oracle(O):
    from paper_1908_09378_b200 import gen
    a = gen.band(5000, 64, 2)
    b = O.gen_band(5000, 64, 2)
    assert np.array_equal(a.offsets, b.off)
    assert np.array_equal(a.targets, b.tgt)
    assert np.array_equal(a.weights, b.w)


def test_mixed_trace_matches_oracle(O):
    from paper_1908_09378_b200 import gen
    for n, u, k, s in [(3000, 1 << 12, 64, 1), (2000, 1 << 16, 1024, 3), (500, 64, 8, 9)]:
        a = gen.mixed_trace(n, u, k, s)
        b = O.gen_mixed_trace(n, u, k, s)
        assert np.array_equal(a.kinds, b.kinds)
        assert np.array_equal(a.offsets, b.offsets)
        assert np.array_equal(a.vals, b.vals)
        assert np.array_equal(a.prios, b.prios)


def test_sweep_batches_are_strict_decreases():
    from paper_1908_09378_b200 import gen
    n = 1 << 12
    pr = gen.sweep_prefill(n, 4)
    assert np.all((pr >= 1 << 39) & (pr < 1 << 40))
    before = pr.copy()
    v, p = gen.sweep_batches(n, 32, 10, 5, pr)
    for b in range(10):
        vb = v[b * 32:(b + 1) * 32]
        assert np.all(np.diff(vb.astype(np.int64)) > 0)
    assert np.all(pr <= before)
