"""Multi-GPU host logic on CPU (gloo, world size 2): subsets are independent given the
operator, so bench.py shards them round-robin over ranks with no data-path
collective; every subset is solved exactly once, the step time is the max over ranks, and rank 0
alone prints the JSON line.  The rank path of bench.run_distributed runs unchanged; only the GPU leg
(the solves themselves) is a stub with a rank-dependent device time."""
import json
import os
import socket
import subprocess
import sys
import types

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import bench

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class StubLeg:
    """Stands in for bench.GpuLeg: same interface, no GPU."""

    def __init__(self, rank, K, N):
        self.rank = rank
        self.cfg = types.SimpleNamespace(K=K, n_iter=N)
        self.solved = []

    def prepare(self, subsets):
        self.subsets = subsets

    def warmup(self, w):
        pass

    def steps(self, nsteps, host):
        infos = []
        for i in range(nsteps):
            self.solved.append(self.subsets[i % len(self.subsets)])
            infos.append({"rel_residual": 1e-8, "rank": 3})
        return 10.0 * (self.rank + 1) * nsteps, infos, 7 * nsteps    # rank-dependent device ms

    def clock_start(self):
        pass

    def clock_stop(self):
        return {"sm_mhz": None, "sm_max_mhz": None, "reasons": []}

    def h2d_bytes(self):
        return 80

    def d2h_bytes(self):
        return 64

    def config(self):
        return {"workload": "stub"}

    def extras(self, value, rank, world):
        return {"stub_world": world}


def _worker(rank, world, port, K, steps, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    args = types.SimpleNamespace(steps=steps, warmup=3)
    leg = StubLeg(rank, K, N=5)
    lines = []
    bench.run_distributed(args, leg, rank, world, dist, None, emit=lines.append)
    gathered = [None] * world
    dist.all_gather_object(gathered, (leg.subsets, leg.solved))
    if rank == 0:
        out.put((lines, gathered))
    else:
        out.put((lines, None))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("K,steps", [(1, 2), (4, 2), (10, 5)])
def test_two_rank_run_distributed(K, steps):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, K, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    lines = [l for l, _ in got]
    gathered = [g for _, g in got if g is not None][0]
    assert sum(len(l) for l in lines) == 1                  # rank 0 alone prints
    res = json.loads([l for l in lines if l][0][0])
    assert res["n_gpus"] == world and res["scaling"] == "weak"
    ms = 10.0 * world * steps                               # max over ranks of the device time
    assert res["ms_per_step"] == pytest.approx(ms / steps)
    assert res["value"] == pytest.approx(steps * 5 * world / (ms / 1e3))
    assert res["stub_world"] == world and res["config"]["subsets_per_rank"] >= 1
    owned = sorted(k for subs, _ in gathered for k in subs)
    if K >= world:
        assert owned == list(range(K))                      # each subset owned by exactly one rank
    else:
        assert set(owned) == set(range(K))                  # fewer subsets than ranks: every rank still works
    assert all(len(solved) == 2 * steps for _, solved in gathered)   # timed + e2e pass, K steps each


def test_single_rank_identity():
    assert bench.max_over_ranks(3.5, None) == 3.5
    assert bench.shard_subsets(10, 0, 1) == list(range(10))
    assert bench.shard_subsets(10, 1, 4) == [1, 5, 9]


def test_gpus_flag_relaunches_under_torchrun(monkeypatch):
    """`bench.py --gpus N` outside torchrun re-executes itself under torch.distributed.run with N
    processes (the contract's one-process-per-GPU launch) instead of silently running one rank."""
    calls = []
    monkeypatch.setattr(subprocess, "call", lambda cmd: calls.append(cmd) or 0)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2"])
    with pytest.raises(SystemExit) as e:
        bench.main()
    assert e.value.code == 0
    cmd = calls[0]
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd
    assert "127.0.0.1" in cmd and cmd[-4:] == ["--gpus", "4", "--steps", "2"]
