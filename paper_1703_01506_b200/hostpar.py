"""Parallel host-side draws from the reference's RNG streams.

numpy's Generator holds the GIL while it fills arrays, so threads do not
scale; a process pool scales but pickling hundreds of MB back costs more
than the draws.  Here forked workers write their rows straight into an
anonymous shared mapping created before the fork.  Each row comes from its
own ``stream(seed, *path)``, so the result is identical to a serial loop.
"""

from __future__ import annotations

import mmap
import os

import numpy as np

_MIN_PARALLEL_ROWS = 64


def fill_rows(shape, dtype, row_fn, nrows: int, workers: int | None = None) -> np.ndarray:
    """out[i] = row_fn(i) for i < nrows, computed by forked workers into
    shared memory (serial below a size threshold or without fork)."""
    out_shape = (nrows,) + tuple(shape)
    nbytes = int(np.prod(out_shape)) * np.dtype(dtype).itemsize
    workers = workers or min(os.cpu_count() or 1, 32)
    if workers <= 1 or nrows < _MIN_PARALLEL_ROWS or not hasattr(os, "fork") or nbytes == 0:
        out = np.empty(out_shape, dtype=dtype)
        for i in range(nrows):
            out[i] = row_fn(i)
        return out
    buf = mmap.mmap(-1, nbytes, flags=mmap.MAP_SHARED | mmap.MAP_ANONYMOUS)
    out = np.frombuffer(buf, dtype=dtype).reshape(out_shape)
    bounds = np.linspace(0, nrows, workers + 1).astype(np.int64)
    pids = []
    for w in range(workers):
        lo, hi = int(bounds[w]), int(bounds[w + 1])
        if hi <= lo:
            continue
        pid = os.fork()
        if pid == 0:  # child: fill rows, exit without running parent cleanups
            code = 0
            try:
                for i in range(lo, hi):
                    out[i] = row_fn(i)
            except BaseException:
                code = 1
            os._exit(code)
        pids.append(pid)
    failed = False
    for pid in pids:
        _, status = os.waitpid(pid, 0)
        failed |= status != 0
    if failed:
        raise RuntimeError("parallel host draw failed in a worker process")
    return out  # backed by the shared mapping (kept alive by the array)
