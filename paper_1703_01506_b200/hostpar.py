"""Parallel host-side draws from the reference's RNG streams.

Each row comes from its own ``stream(seed, *path)``, so any parallel order
gives the result of a serial loop.  Long rows (e.g. v normals per row) go to
a thread pool: numpy releases the GIL while it fills an array, and threads
need no fork -- forking a process that holds page-locked (cudaHostRegister)
buffers makes the kernel copy those pages eagerly into every child.  Short
rows (a permutation of n subjects: the per-row cost is Python-level stream
construction under the GIL) go to forked workers writing into an anonymous
shared mapping created before the fork.
"""

from __future__ import annotations

import mmap
import os
import threading

import numpy as np

_MIN_PARALLEL_ROWS = 64
_THREAD_ROW_ELEMS = 1 << 16


def fill_rows(shape, dtype, row_fn, nrows: int, workers: int | None = None) -> np.ndarray:
    """out[i] = row_fn(i) for i < nrows, computed by forked workers into
    shared memory (serial below a size threshold or without fork)."""
    out_shape = (nrows,) + tuple(shape)
    nbytes = int(np.prod(out_shape)) * np.dtype(dtype).itemsize
    workers = workers or min(os.cpu_count() or 1, 32)
    row_elems = int(np.prod(shape)) if len(shape) else 1
    if workers > 1 and nrows > 1 and row_elems >= _THREAD_ROW_ELEMS:
        from concurrent.futures import ThreadPoolExecutor

        out = np.empty(out_shape, dtype=dtype)

        def one(i):
            out[i] = row_fn(i)

        with ThreadPoolExecutor(max_workers=workers) as ex:
            list(ex.map(one, range(nrows)))
        return out
    # no fork while other threads run (run_rapid's host draws): a child
    # could inherit a lock one of them holds
    if (workers <= 1 or nrows < _MIN_PARALLEL_ROWS or not hasattr(os, "fork") or nbytes == 0
            or threading.active_count() > 1):
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
