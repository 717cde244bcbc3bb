"""Multi-source SSSP with the results gathered on the first device over
NVLink (pbh_sssp_multi_device). On a one-GPU box the gather is a device-local
copy; the sharding, the peer-copy path and the result layout are the same."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_device_gather_matches_host_path(pbh, O):
    import torch
    g = O.gen_band(4096, 64, 2)
    srcs = [0, 17, 1024, 4095]
    dist_h, parent_h = pbh.par_dijkstra_multi(g, srcs)
    V = g.V
    dist_d = torch.empty(len(srcs) * V, dtype=torch.int64, device="cuda:0")
    parent_d = torch.empty(len(srcs) * V, dtype=torch.int32, device="cuda:0")
    ms = pbh.par_dijkstra_multi_device(g, srcs, dist_d.data_ptr(), parent_d.data_ptr(),
                                       devices=(0,))
    assert ms > 0
    got_d = dist_d.cpu().numpy().view(np.uint64).reshape(len(srcs), V)
    got_p = parent_d.cpu().numpy().view(np.uint32).reshape(len(srcs), V)
    assert np.array_equal(got_d, dist_h)
    assert np.array_equal(got_p, parent_h)
    for i, s in enumerate(srcs):
        assert np.array_equal(got_d[i], O.dijkstra(g, s)["dist"])


def test_device_gather_sharded_over_device_list(pbh, O):
    # the same device listed twice: two shards, two contexts, one gather target
    import torch
    g = O.gen_random(2000, 16000, 100, 3)
    srcs = list(range(0, 2000, 250))
    V = g.V
    dist_d = torch.empty(len(srcs) * V, dtype=torch.int64, device="cuda:0")
    pbh.par_dijkstra_multi_device(g, srcs, dist_d.data_ptr(), 0, devices=(0, 0))
    got = dist_d.cpu().numpy().view(np.uint64).reshape(len(srcs), V)
    for i, s in enumerate(srcs):
        assert np.array_equal(got[i], O.dijkstra(g, s)["dist"])
