"""Permutation sharding across GPUs (one process per GPU, torch.distributed).

Permutations are independent units (reference naive.py:70-73: every index
owns its stream and its output slot), so GPU g of G evaluates the contiguous
range [g*per, (g+1)*per) of the plan (per rounded up to the 128-permutation
M tile) with no data-path communication; the only exchange is one
all-gather of the per-permutation max (fp64) and argmax (int32) at the end,
ordered by rank, which reproduces the reference's index order
(naive.py:88-101).  The tensor-core arithmetic does not depend on the shard,
so maxima and argmax are bit-identical for every G.
"""

from __future__ import annotations

from typing import Optional

import numpy as np

from .exceptions import UsageError


def shard_bounds(L: int, rank: int, world: int, align: int = 128) -> tuple[int, int, int]:
    """(lo, hi, per): this rank's permutation range and the padded shard size."""
    if world < 1 or not 0 <= rank < world:
        raise UsageError(f"bad rank {rank} / world {world}")
    per = -(-L // world)
    per = -(-per // align) * align
    lo = min(L, rank * per)
    hi = min(L, lo + per)
    return lo, hi, per


def dist_info(group=None) -> tuple[int, int]:
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def gather_maxima(local_max, local_arg, L: int, per: int, group=None):
    """All-gather padded per-rank (max, argmax) shards; returns the first L
    entries in global permutation order (same tensors on every rank)."""
    import torch
    import torch.distributed as dist

    rank, world = dist_info(group)
    dev = local_max.device
    pm = torch.full((per,), float("nan"), dtype=torch.float64, device=dev)
    pa = torch.full((per,), -1, dtype=torch.int32, device=dev)
    k = int(local_max.numel())
    if k:
        pm[:k] = local_max
        pa[:k] = local_arg
    if world == 1:
        return pm[:L], pa[:L]
    gm = [torch.empty_like(pm) for _ in range(world)]
    ga = [torch.empty_like(pa) for _ in range(world)]
    dist.all_gather(gm, pm, group=group)
    dist.all_gather(ga, pa, group=group)
    return torch.cat(gm)[:L], torch.cat(ga)[:L]


class ShardedNaive:
    """NaivePT over this rank's permutation shard with device-resident inputs.

    x_dev: (v, n) float64 replica on this rank's GPU; the shard's label rows
    are generated on the GPU from the plan (labels.device_orders), or
    uploaded from ``orders_host`` when given.
    """

    def __init__(self, x_dev, n1: int, plan, two_sided: bool, group=None,
                 orders_host: Optional[np.ndarray] = None):
        import torch

        from .labels import device_orders
        from .naive_engine import NaiveJob

        self.group = group
        self.rank, self.world = dist_info(group)
        self.L = int(plan.count)
        self.lo, self.hi, self.per = shard_bounds(self.L, self.rank, self.world)
        self.orders_host = orders_host
        self.job = None
        if self.hi > self.lo:
            if orders_host is None:
                od = device_orders(plan.master_seed, self.lo, self.hi, int(x_dev.shape[1]),
                                   x_dev.device)
            else:
                od = torch.from_numpy(np.ascontiguousarray(orders_host)).to(x_dev.device)
            self.job = NaiveJob(x_dev, n1, od, two_sided)
        self.device = x_dev.device

    @property
    def local_count(self) -> int:
        return self.hi - self.lo

    def compute(self):
        import torch

        if self.job is None:
            e = torch.empty(0, dtype=torch.float64, device=self.device)
            return e, torch.empty(0, dtype=torch.int32, device=self.device)
        self.job.prepare()
        self.job.tfill()
        self.job.finish()
        return self.job.max_out, self.job.argmax_out

    def step(self):
        m, a = self.compute()
        return gather_maxima(m, a, self.L, self.per, self.group)


def run_naive_distributed(x, plan, two_sided: bool = False, group=None):
    """Public multi-GPU entry: every rank passes the same host (x, plan) and
    gets the full (MaxNull, argmax).  Each rank runs its permutation shard
    through the host-input engine (rmx_naive_maxnull_host_plan_range*: X
    uploaded chunk by chunk under K0/K1, the shard's labels generated on its
    GPU), then one all-gather of (max, argmax).  Single-process when
    torch.distributed is not initialised."""
    import torch

    from .domain import MaxNull, as_data_matrix, as_plan
    from .naive_engine import _run_from_host, cuda_device

    x = as_data_matrix(x)
    plan = as_plan(plan)
    if plan.subjects != x.subjects:
        raise UsageError("plan and data matrix disagree on subject count")
    dev = cuda_device()
    rank, world = dist_info(group)
    L = int(plan.count)
    lo, hi, per = shard_bounds(L, rank, world)
    if hi > lo:
        _, _, job = _run_from_host(x, plan, two_sided, dev, lo, hi)
        lm, la = job.max_out, job.argmax_out
    else:
        lm = torch.empty(0, dtype=torch.float64, device=dev)
        la = torch.empty(0, dtype=torch.int32, device=dev)
    m, a = gather_maxima(lm, la, L, per, group)
    return MaxNull(m.cpu().numpy()), a.cpu().numpy().astype(np.int64)
