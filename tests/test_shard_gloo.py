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


def _engine_worker(rank, world, port, L, q):
    """run_naive_distributed at world 2 on CPU: the real shard bounds, the
    shared-upload replica (replicate_rows: each rank's row slice + one
    all-gather), the per-rank label range and the packed (max, argmax)
    all-gather; only the device engine call is replaced by the CPU oracle
    on the same replica and the same label rows."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1703_01506_b200 as rmx
    from oracle import oracle
    from paper_1703_01506_b200 import shard
    from paper_1703_01506_b200.labels import generate_orders

    seen = {}

    def oracle_compute(x_dev, n1, plan, lo, hi, two_sided):
        xv = x_dev.numpy()
        seen["replica"] = xv.copy()
        orders = generate_orders(plan.master_seed, lo, hi, xv.shape[1]).astype(np.int64)
        mx, am, _ = oracle.naive_maxnull(xv, n1, orders, two_sided)
        return torch.from_numpy(mx), torch.from_numpy(am.astype(np.int32))

    shard._device = lambda: torch.device("cpu")
    shard._shard_compute = oracle_compute
    g = np.random.default_rng(11)
    vals = g.standard_normal((301, 12)).astype(np.float32)
    x = rmx.DataMatrix(vals, 5, 7)
    plan = rmx.PermutationPlan(9, L, 12)
    null, am = shard.run_naive_distributed(x, plan, two_sided=True)
    q.put((rank, null.maxima, am, seen.get("replica")))
    dist.destroy_process_group()


@pytest.mark.parametrize("L", [300, 129])
def test_distributed_entry_matches_single_process_oracle(L):
    from oracle import oracle
    from paper_1703_01506_b200.labels import generate_orders

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_engine_worker, args=(r, world, port, L, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = np.random.default_rng(11)
    vals = g.standard_normal((301, 12)).astype(np.float32).astype(np.float64)
    mx, am, _ = oracle.naive_maxnull(vals, 5, generate_orders(9, 0, L, 12).astype(np.int64), True)
    for rank, m, a, replica in res:
        assert np.array_equal(m, mx) and np.array_equal(a, am)
        if replica is not None:  # every computing rank saw all of X, bit for bit
            assert np.array_equal(replica, vals)


def test_pack_roundtrip():
    from paper_1703_01506_b200.shard import pack_maxima, unpack_maxima

    m = torch.tensor([1.5, -0.0, 3e300, -7.25], dtype=torch.float64)
    a = torch.tensor([3, 0, 2**31 - 1, 17], dtype=torch.int32)
    p = pack_maxima(m, a, 6)
    assert p.shape == (6, 3) and p.dtype == torch.int32
    mm, aa = unpack_maxima(p)
    assert torch.equal(mm[:4], m) and torch.equal(aa[:4], a)
    assert torch.isnan(mm[4:]).all() and (aa[4:] == -1).all()
