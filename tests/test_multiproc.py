"""Multi-rank host logic of bench.py (world_size 2, gloo on CPU): frame sharding,
max-over-ranks timing, whole-job sums, and the one collective (broadcast of the packed
prediction table from the adapting rank)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import bench

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        r, local, w = bench.dist_env()
        assert (r, w) == (rank, world)
        mine = bench.shard(101, rank, world)
        allv = [None] * world
        dist.all_gather_object(allv, mine)
        flat = sorted(i for part in allv for i in part)
        assert flat == list(range(101))  # every frame exactly once
        t = bench.max_over_ranks(10.0 + rank, dist)
        n = bench.sum_over_ranks(float(len(mine)), dist)
        # broadcast of the prediction table (CPU stand-in for the NCCL device buffer)
        buf = torch.arange(4096, dtype=torch.int32).to(torch.uint8) if rank == 0 else torch.zeros(4096, dtype=torch.uint8)
        dist.broadcast(buf, src=0)
        ok = bool(torch.equal(buf, torch.arange(4096, dtype=torch.int32).to(torch.uint8)))
        q.put((rank, t, n, ok, bench.frame_seed(1234, mine[0])))
    finally:
        dist.destroy_process_group()


def test_two_rank_sharding_and_aggregation():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    res = sorted(q.get() for _ in range(world))
    for rank, t, n, ok, seed in res:
        assert t == 11.0  # max over ranks
        assert n == 101.0  # whole-job frame count
        assert ok
    assert res[0][4] != res[1][4]  # per-frame seeds differ across shards


def test_frame_seeds_are_independent_of_sharding():
    import bench

    assert [bench.frame_seed(1, i) for i in bench.shard(10, 1, 2)] == [bench.frame_seed(1, i) for i in (1, 3, 5, 7, 9)]
