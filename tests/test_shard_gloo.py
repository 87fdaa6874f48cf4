"""Multi-process permutation sharding (world_size 2, gloo on CPU): the shard
ranges partition [0, L) and the all-gather reassembles the per-rank maxima
in global permutation order, as NCCL does on the GPU path."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1703_01506_b200.shard import gather_maxima, shard_bounds


@pytest.mark.parametrize("L,world", [(1000, 2), (100000, 8), (129, 4), (5, 8), (128, 2)])
def test_shard_bounds_partition(L, world):
    seen = []
    pers = set()
    for r in range(world):
        lo, hi, per = shard_bounds(L, r, world)
        pers.add(per)
        assert per % 128 == 0 and 0 <= lo <= hi <= L
        seen.extend(range(lo, hi))
    assert seen == list(range(L)) and len(pers) == 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, L, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi, per = shard_bounds(L, rank, world)
    # stand-in for the device kernel: a deterministic function of the global index
    idx = torch.arange(lo, hi, dtype=torch.float64)
    m, a = gather_maxima((idx * 37 % 1009) / 8.0, (idx * 7 % 997).to(torch.int32), L, per)
    q.put((rank, m.numpy(), a.numpy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("L", [1000, 130, 3])
def test_gather_reassembles_global_order(L):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, L, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    idx = np.arange(L, dtype=np.float64)
    for _, m, a in res:
        assert np.array_equal(m, (idx * 37 % 1009) / 8.0)
        assert np.array_equal(a, (idx * 7 % 997).astype(np.int32))
