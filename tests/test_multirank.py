"""Multi-GPU host logic on CPU (gloo, world size 2): subsets are sharded round-robin with no data-path
collective, every subset is solved exactly once, and the step time is the max over ranks."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, K, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = bench.shard_subsets(K, rank, world)
    ms = 10.0 * (rank + 1)                        # rank-dependent "device time"
    t = bench.max_over_ranks(ms, dist)
    gathered = [None] * world
    dist.all_gather_object(gathered, mine)
    if rank == 0:
        out.put((t, gathered))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("K", [1, 4, 10])
def test_two_rank_sharding_and_max_timing(K):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, K, q)) for r in range(world)]
    for p in procs:
        p.start()
    t, gathered = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert t == 20.0                               # max over ranks
    flat = sorted(k for g in gathered for k in g)
    if K >= world:
        assert flat == list(range(K))              # each subset exactly once
    else:
        assert set(flat) == set(range(K))          # fewer subsets than ranks: every rank still works
    assert all(len(g) >= 1 for g in gathered)


def test_single_rank_identity():
    assert bench.max_over_ranks(3.5, None) == 3.5
    assert bench.shard_subsets(10, 0, 1) == list(range(10))
