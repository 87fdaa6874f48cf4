"""Permutation label matrices: PermutationPlan -> L x n subject orders.

The engine consumes the plan as a dense int16 matrix ``orders[p, :]`` =
``plan.shuffle(p)`` (group 1 = the first n1 entries, in shuffle order -- the
order matters for the bit-exact refinement, which sums in that order, as the
reference's fancy-indexed blocks do; reference model.py:65-69).

Generating a shuffle costs ~26-30 us of host time per permutation (numpy
SeedSequence + SFC64), i.e. ~3 s for L = 1e5 on one core.  The
engine therefore generates the rows on the GPU (``device_orders``: the same
streams restated bit for bit in rng_kernels.cu, ~ms for 1e5 rows); the host
path (``plan_orders``: forked workers, cached) serves the CPU-side users
(the oracle, materialised-T bookkeeping, the reference arm).
"""

from __future__ import annotations

import os
import threading
from collections import OrderedDict

import numpy as np

from .exceptions import UsageError
from .hostpar import fill_rows
from .rng import shuffle_order

_CACHE: "OrderedDict[tuple, np.ndarray]" = OrderedDict()
_CACHE_BYTES = 0
_CACHE_LIMIT = int(os.environ.get("RMX_LABEL_CACHE_BYTES", str(2 << 30)))
_LOCK = threading.Lock()


def generate_orders(seed: int, lo: int, hi: int, n: int, workers: int | None = None) -> np.ndarray:
    """Rows [lo, hi) of the plan's order matrix (uncached), drawn by forked
    workers into shared memory (identical to a serial loop)."""
    if n > 32767:
        raise UsageError(f"subject count {n} exceeds the int16 label format")
    if hi - lo < 4096:
        workers = 1
    return fill_rows((n,), np.int16, lambda i: shuffle_order(seed, lo + i, n), hi - lo, workers)


def plan_orders(plan, lo: int = 0, hi: int | None = None) -> np.ndarray:
    """Cached order matrix for ``plan`` rows [lo, hi) (int16, read-only)."""
    global _CACHE_BYTES
    hi = plan.count if hi is None else hi
    key = (int(plan.master_seed), int(plan.count), int(plan.subjects))
    with _LOCK:
        full = _CACHE.get(key)
        if full is not None:
            _CACHE.move_to_end(key)
            return full[lo:hi]
    if (hi - lo) != plan.count:
        # a shard: generate only the requested rows, do not cache
        return generate_orders(key[0], lo, hi, key[2])
    full = generate_orders(key[0], 0, plan.count, key[2])
    full.setflags(write=False)
    with _LOCK:
        _CACHE[key] = full
        _CACHE_BYTES += full.nbytes
        while _CACHE_BYTES > _CACHE_LIMIT and len(_CACHE) > 1:
            _, old = _CACHE.popitem(last=False)
            _CACHE_BYTES -= old.nbytes
    return full[lo:hi]


def device_orders(seed: int, lo: int, hi: int, n: int, device, stream=None):
    """Rows [lo, hi) of the plan's order matrix generated on the GPU
    (rmx_plan_orders: numpy's SeedSequence -> SFC64 -> permutation restated
    bit for bit), as an (hi - lo, n) int16 CUDA tensor."""
    import ctypes

    import torch

    from . import _native as nat

    if n > 32767:
        raise UsageError(f"subject count {n} exceeds the int16 label format")
    out = torch.empty((max(hi - lo, 0), n), dtype=torch.int16, device=device)
    if hi > lo:
        s = stream if stream is not None else torch.cuda.current_stream(device)
        st = nat.Status()
        rc = nat.load().rmx_plan_orders(ctypes.c_uint64(int(seed) & ((1 << 64) - 1)), int(lo),
                                        int(hi - lo), int(n), nat.ptr(out), nat.stream_handle(s),
                                        ctypes.byref(st))
        nat.raise_for(rc, st)
    return out


def clear_cache() -> None:
    global _CACHE_BYTES
    with _LOCK:
        _CACHE.clear()
        _CACHE_BYTES = 0
