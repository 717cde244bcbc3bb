"""The product's workload generators (include/pbh_gen.h, C++) must agree draw
for draw with the oracle's independent restatement (oracle/pbh_oracle.c)."""
import numpy as np
import pytest


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


# ---- device generators: bit-identical to the host ones
@pytest.mark.gpu
@pytest.mark.parametrize("v,deg", [(4096, 64), (1 << 16, 256), (300, 1), (1000, 999)])
def test_band_device_matches_host(v, deg):
    from paper_1908_09378_b200 import gen
    want = gen.band(v, deg, 2)
    got = gen.band_device(v, deg, 2).to_host()
    assert np.array_equal(got.offsets, want.offsets)
    assert np.array_equal(got.targets, want.targets)
    assert np.array_equal(got.weights, want.weights)


@pytest.mark.gpu
@pytest.mark.parametrize("r,c", [(64, 64), (1, 50), (37, 1), (333, 517)])
def test_grid_device_matches_host(r, c):
    from paper_1908_09378_b200 import gen
    want = gen.grid(r, c, 1)
    got = gen.grid_device(r, c, 1).to_host()
    assert np.array_equal(got.offsets, want.offsets)
    assert np.array_equal(got.targets, want.targets)
    assert np.array_equal(got.weights, want.weights)


@pytest.mark.gpu
def test_sssp_on_device_generated_graph():
    import paper_1908_09378_b200 as P
    from paper_1908_09378_b200 import gen
    gd = gen.band_device(8192, 64, 2)
    ctx = P.SsspContext(gd, max_sources=1)
    ctx.run([0])
    r = ctx.fetch(0, settled=False)
    ctx.close()
    host = P.par_dijkstra(gen.band(8192, 64, 2), 0)
    assert np.array_equal(r.dist, host.dist)
