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


def pack_maxima(local_max, local_arg, per: int):
    """(per, 3) int32 rows [max as two int32 words | argmax]: one buffer, so
    the exchange is one collective of 12 B per permutation.  Padding rows
    carry NaN / -1."""
    import torch

    dev = local_max.device
    pm = torch.full((per,), float("nan"), dtype=torch.float64, device=dev)
    pa = torch.full((per,), -1, dtype=torch.int32, device=dev)
    k = int(local_max.numel())
    if k:
        pm[:k] = local_max
        pa[:k] = local_arg
    return torch.cat([pm.view(torch.int32).view(per, 2), pa.view(per, 1)], dim=1).contiguous()


def unpack_maxima(packed):
    """Inverse of pack_maxima over any number of rows: (max fp64, argmax int32)."""
    import torch

    m = packed[:, :2].contiguous().view(torch.float64).reshape(-1)
    return m, packed[:, 2].contiguous()


def gather_maxima(local_max, local_arg, L: int, per: int, group=None):
    """All-gather padded per-rank (max, argmax) shards in ONE collective of
    12 B per permutation (all_gather_into_tensor over NCCL; the list form on
    backends without it, e.g. gloo); returns the first L entries in global
    permutation order (same tensors on every rank)."""
    import torch
    import torch.distributed as dist

    rank, world = dist_info(group)
    packed = pack_maxima(local_max, local_arg, per)
    if world == 1:
        m, a = unpack_maxima(packed)
        return m[:L], a[:L]
    out = torch.empty((world * per, 3), dtype=torch.int32, device=packed.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, packed, group=group)
    else:
        dist.all_gather(list(out.chunk(world)), packed, group=group)
    m, a = unpack_maxima(out)
    return m[:L], a[:L]


def row_bounds(v: int, rank: int, world: int) -> tuple[int, int, int]:
    """(lo, hi, per): this rank's voxel-row slice of X for the shared upload."""
    per = -(-v // world)
    lo = min(v, rank * per)
    return lo, min(v, lo + per), per


def replicate_rows(x_host, device, group=None):
    """Every rank gets all of X (v x n, the host array's dtype) on `device`
    while uploading only its own 1/world slice of the rows over PCIe: each
    rank copies rows [lo, hi) from its (page-locked) host array, then one
    all-gather over NVLink assembles the replica.  At world 1 this is a plain
    upload.  Bit-exact (a copy)."""
    import torch
    import torch.distributed as dist

    from .hostmem import to_device

    def upload(a):
        a = np.ascontiguousarray(a)
        if torch.device(device).type == "cpu":  # gloo tests
            return torch.from_numpy(a.copy())
        return to_device(a, device)

    rank, world = dist_info(group)
    v, n = x_host.shape
    if world == 1:
        return upload(x_host)
    lo, hi, per = row_bounds(v, rank, world)
    local = torch.zeros((per, n), dtype=_torch_dtype(x_host.dtype), device=device)
    if hi > lo:
        local[: hi - lo] = upload(x_host[lo:hi])
    full = torch.empty((world * per, n), dtype=local.dtype, device=device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(full, local, group=group)
    else:
        dist.all_gather(list(full.chunk(world)), local, group=group)
    return full[:v]


def _torch_dtype(dt):
    import torch

    return {np.dtype(np.float64): torch.float64, np.dtype(np.float32): torch.float32}[np.dtype(dt)]


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


def _shard_compute(x_dev, n1: int, plan, lo: int, hi: int, two_sided: bool):
    """This rank's permutations [lo, hi) over the device replica of X: the
    shard's labels generated on its GPU from the plan seed, then the engine
    (K0 / K1 / K2 through rmx_naive_maxnull).  Returns device (max, argmax)."""
    from .labels import device_orders
    from .naive_engine import NaiveJob

    od = device_orders(plan.master_seed, lo, hi, int(x_dev.shape[1]), x_dev.device)
    job = NaiveJob(x_dev, n1, od, two_sided)
    return job.run()


def run_naive_distributed(x, plan, two_sided: bool = False, group=None):
    """Public multi-GPU entry: every rank passes the same host (x, plan) and
    gets the full (MaxNull, argmax).

    world 1: the single-GPU host engine (rmx_naive_maxnull_host_plan*: X
    uploaded chunk by chunk under K0/K1).  world N > 1: each rank uploads
    only its 1/N row slice of X (the float32 source when the DataMatrix
    keeps one) and one NCCL all-gather over NVLink assembles the replica
    (replicate_rows: ~1/N of the PCIe time instead of every rank moving all
    of X), then the rank runs its permutation shard and one all-gather of
    12 B per permutation returns the maxima in global order."""
    import torch

    from .domain import MaxNull, as_data_matrix, as_plan
    from .naive_engine import _run_from_host, cuda_device

    x = as_data_matrix(x)
    plan = as_plan(plan)
    if plan.subjects != x.subjects:
        raise UsageError("plan and data matrix disagree on subject count")
    dev = _device()
    rank, world = dist_info(group)
    L = int(plan.count)
    lo, hi, per = shard_bounds(L, rank, world)
    if world == 1:
        _, _, job = _run_from_host(x, plan, two_sided, cuda_device(), lo, hi)
        lm, la = job.max_out, job.argmax_out
    else:
        src = x.float32_values if x.float32_values is not None else x.values
        xd = replicate_rows(src, dev, group)
        if xd.dtype != torch.float64:
            xd = xd.to(torch.float64)  # exact upcast of the float32 source
        if hi > lo:
            lm, la = _shard_compute(xd, x.n1, plan, lo, hi, two_sided)
        else:
            lm = torch.empty(0, dtype=torch.float64, device=dev)
            la = torch.empty(0, dtype=torch.int32, device=dev)
    m, a = gather_maxima(lm, la, L, per, group)
    return MaxNull(m.cpu().numpy()), a.cpu().numpy().astype(np.int64)


def _device():
    from .naive_engine import cuda_device

    return cuda_device()
