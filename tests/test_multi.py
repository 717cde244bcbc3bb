"""Multi-GPU plumbing on CPU: world_size-2 gloo runs of the bench's sharding and
max-over-ranks timing logic (no device work). The data path has no collective;
the only cross-rank operation is the MAX reduction of the timed region."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch

    import bench
    srcs = bench.sources_for(rank, 64, 1 << 20)
    mine = torch.tensor([float(100 + 50 * rank)])
    dist.all_reduce(mine, op=dist.ReduceOp.MAX)
    gathered = [None] * world
    dist.all_gather_object(gathered, srcs)
    q.put((rank, float(mine.item()), gathered))
    dist.destroy_process_group()


def test_two_rank_sharding_and_max():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, mx, gathered in out:
        assert mx == 150.0  # max over ranks, as bench.py reports
        a, b = gathered
        assert len(a) == len(b) == 64
        assert not set(a) & set(b)  # disjoint shards: no duplicated work
        assert a == [(i * 16384) % (1 << 20) for i in range(64)]  # rank 0 == BASELINE C5


def test_sssp_bytes_accounting():
    import bench
    # C3 algorithmic bytes
    assert bench.sssp_bytes(1 << 20, 268435456, 1 << 20) == 2168455176
    # C2 grid: E=67,092,480, V=16,777,216
    assert bench.sssp_bytes(16777216, 67092480, 16777216) == 872284168


@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(__file__), "..", "oracle",
                                                    "_ref", "libpbhref.so")),
                    reason="oracle/_ref not built")
def test_reference_multi_source_matches_oracle():
    # the reference arm's multi-threaded C5 sample computes the same distances
    import numpy as np

    from oracle import oracle as O
    g = O.gen_band(2048, 64, 2)
    srcs = [0, 512, 1024, 1536]
    d = O.ref_sssp_multi(g, srcs, algo="par", threads=2)
    for i, s in enumerate(srcs):
        assert np.array_equal(d[i], O.dijkstra(g, s)["dist"])
