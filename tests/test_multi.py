"""Multi-GPU plumbing on CPU: world_size-2 gloo runs of the bench's real
shard / gather bookkeeping (bench.Dist, paper_1908_09378_b200.multi.shard and
GatherPlan). The GPU-0 gather buffer is stood in for by a shared-memory block
whose name travels like the CUDA IPC handle does (broadcast from rank 0);
each rank writes its shard's rows at the offsets the plan gives, exactly as
pbh_sssp_ctx_gather does into the IPC-mapped buffer. The data path has no
collective; the only cross-rank reductions are the MAX of the timed region
and the small per-source parity records."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


V_TEST = 1000


def _fake_solve(src):
    """Deterministic stand-in for one source's (dist, parent) rows."""
    dist = np.arange(V_TEST, dtype=np.uint64) * np.uint64(3) + np.uint64(src) * np.uint64(1 << 20)
    parent = (np.arange(V_TEST, dtype=np.uint32) + np.uint32(src % 7)) % np.uint32(V_TEST)
    return dist, parent


def _check_assembled(buf, plan, srcs_all):
    dist = buf[:plan.dist_bytes].view(np.uint64).reshape(len(srcs_all), V_TEST)
    par = buf[plan.dist_bytes:plan.nbytes].view(np.uint32).reshape(len(srcs_all), V_TEST)
    return all(np.array_equal(dist[i], _fake_solve(s)[0]) and
               np.array_equal(par[i], _fake_solve(s)[1]) for i, s in enumerate(srcs_all))


def _worker(rank, world, port, q):
    from multiprocessing import shared_memory
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world),
                      RANK=str(rank), LOCAL_RANK=str(rank))
    import bench
    from paper_1908_09378_b200.multi import GatherPlan, shard
    D = bench.Dist()
    assert D.backend == "gloo" and D.world == world
    srcs_all = bench.c5_sources(64)
    b, e = shard(len(srcs_all), D.world, D.rank)
    srcs = srcs_all[b:e]
    plan = GatherPlan(len(srcs_all), V_TEST, D.world)
    shm = shared_memory.SharedMemory(create=True, size=plan.nbytes) if D.rank == 0 else None
    name = D.bcast(shm.name if shm else None)  # like the 64-byte IPC handle
    if D.rank != 0:
        shm = shared_memory.SharedMemory(name=name)
    buf = np.frombuffer(shm.buf, dtype=np.uint8)
    # "gather": this rank's rows at the plan's offsets (source-major)
    for i, s in enumerate(srcs):
        d, p = _fake_solve(s)
        o = plan.dist_offset(D.rank) + i * V_TEST * 8
        buf[o:o + d.nbytes] = d.view(np.uint8)
        o = plan.parent_offset(D.rank) + i * V_TEST * 4
        buf[o:o + p.nbytes] = p.view(np.uint8)
    D.barrier()
    mx = D.max(100.0 + 50 * D.rank)  # max over ranks, as bench.py reports
    recs = D.gather_objs([{"src": s} for s in srcs])
    ok = _check_assembled(buf, plan, srcs_all) if D.rank == 0 else None
    q.put((D.rank, srcs, mx, [r["src"] for part in recs for r in part], ok))
    D.barrier()
    del buf
    shm.close()
    if D.rank == 0:
        shm.unlink()
    D.close()


@pytest.mark.parametrize("world", [2, 3])
def test_multi_rank_shard_and_gather(world):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=180) for _ in range(world)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    all_srcs = [i * 16384 for i in range(64)]
    assert [s for _, srcs, _, _, _ in out for s in srcs] == all_srcs  # contiguous, disjoint
    for rank, srcs, mx, gathered, ok in out:
        assert mx == 100.0 + 50 * (world - 1)
        assert gathered == all_srcs
        if rank == 0:
            assert ok is True  # the assembled buffer is the source-major result


def test_shard_covers_contiguously():
    from paper_1908_09378_b200.multi import shard
    for n in (1, 7, 63, 64, 65, 1000):
        for world in (1, 2, 3, 4, 8, 100):
            rs = [shard(n, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            sizes = [e - b for b, e in rs]
            assert max(sizes) - min(sizes) <= 1


def test_gather_plan_offsets():
    from paper_1908_09378_b200.multi import GatherPlan
    p = GatherPlan(64, 1 << 20, 8)
    assert p.nbytes == 64 * (1 << 20) * 12
    assert p.dist_offset(3) == 24 * (1 << 20) * 8
    assert p.parent_offset(0) == p.dist_bytes
    assert p.parent_offset(7) == p.dist_bytes + 56 * (1 << 20) * 4


def test_sssp_bytes_accounting():
    import bench
    # C3 algorithmic bytes
    assert bench.sssp_bytes(1 << 20, 268435456, 1 << 20) == 2168455176
    # C2 grid: E=67,092,480, V=16,777,216
    assert bench.sssp_bytes(16777216, 67092480, 16777216) == 872284168


@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(__file__), "..", "oracle",
                                                    "_ref", "libpbhref.so")),
                    reason="oracle/_ref not built")
def test_reference_batch_matches_oracle():
    # the reference arm's multi-threaded batch (graph imported once) computes
    # the same distances and settle orders as the C restatement
    from oracle import oracle as O
    g = O.gen_band(2048, 64, 2)
    srcs = [0, 512, 1024, 1536]
    rg = O.RefGraph(g)
    r = rg.sssp_batch(srcs, "par", threads=2, want_dist=True)
    t = rg.sssp_batch(srcs, "ref", threads=2)
    rg.close()
    for i, s in enumerate(srcs):
        want = O.dijkstra(g, s)
        assert np.array_equal(r["dist"][i], want["dist"])
        assert int(r["settled_ck"][i]) == O.fnv1a(want["settled_order"]) == int(t["settled_ck"][i])
        assert int(r["ops"][i]) == want["ops"]
