"""NaivePT on the B200: drop-in ``run_naive``.

Reference: naive.py:60-109 ``run_naive(x, plan, materialize, two_sided,
threads, mem_cap_bytes) -> (MaxNull, StatMatrix | None, counters)``.

Device pipeline (librmx.so):
  K0 prepare  fp64 standardisation + int8 digit planes (balanced, n >= 192)
              or fp16 hi/lo split planes of Z (and Z^2)
  K1 tfill    tcgen05 contraction G.[Z|Z^2] + fused t / top-4 epilogue
  K2 finish   fp64 refinement of the band candidates -> maxima bit-identical
              to the reference (numpy arithmetic restated, np_exact.cuh)
``materialize=True`` additionally fills the dense statistic matrix with the
exact fp64 kernel (bit-identical to the reference's ``store[:, i] = col``).
From host arrays (``run_naive``), one ``rmx_naive_maxnull_host`` call uploads
X chunk by chunk and overlaps the copy with K0/K1.

Threads: the reference parallelises over permutation blocks on a thread pool
and guarantees thread-count-independent results (naive.py:86-101).  Here the
parallelism is the GPU's; ``threads`` is validated for API parity and has no
effect on the (deterministic) result.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _native as nat
from .domain import MaxNull, StatMatrix, as_data_matrix, as_plan
from .exceptions import EngineUnavailableError, UsageError

DEFAULT_MEM_CAP_BYTES = 2 << 30

_CHECKED_DEVICES: set = set()


def resolve_threads(threads: Optional[int]) -> int:
    """Same precedence as the reference (naive.py:37-46): argument, then
    RAPIDMAXNULL_THREADS, then os.cpu_count()."""
    if threads is None:
        env = os.environ.get("RAPIDMAXNULL_THREADS")
        if env:
            threads = int(env)
    if threads is None:
        threads = os.cpu_count() or 1
    if threads < 1:
        raise UsageError(f"thread count must be >= 1, got {threads}")
    return threads


def cuda_device():
    """The current CUDA device, checked to be sm_100 (B200).  Raises
    EngineUnavailableError otherwise -- there is no CPU path."""
    import torch

    if not torch.cuda.is_available():
        raise EngineUnavailableError("no CUDA device visible; the engine has no CPU fallback")
    dev = torch.cuda.current_device()
    if dev not in _CHECKED_DEVICES:
        nat.device_check(dev)
        _CHECKED_DEVICES.add(dev)
    return torch.device("cuda", dev)


@dataclass
class NaiveResult:
    maxima: np.ndarray
    argmax: np.ndarray
    stats: dict = field(default_factory=dict)
    T: Optional[np.ndarray] = None


class NaiveJob:
    """A NaivePT evaluation over device-resident inputs.

    x:      (v, n) float64 CUDA tensor (DataMatrix.values layout)
    orders: (L, n) int16 CUDA tensor (row p = plan.shuffle(p))
    The three phases are exposed separately so callers can time the
    tensor-core contraction alone (bench.py); ``run`` chains them.
    """

    def __init__(self, x, n1: int, orders, two_sided: bool, stream=None):
        import torch

        if x.dtype != torch.float64 or x.dim() != 2 or not x.is_contiguous():
            raise UsageError("x must be a contiguous (v, n) float64 CUDA tensor")
        if orders.dtype != torch.int16 or orders.dim() != 2 or not orders.is_contiguous():
            raise UsageError("orders must be a contiguous (L, n) int16 CUDA tensor")
        if orders.shape[1] != x.shape[1]:
            raise UsageError("orders and x disagree on the subject count")
        self.lib = nat.load()
        self.x, self.orders = x, orders
        self.v, self.n = int(x.shape[0]), int(x.shape[1])
        self.L = int(orders.shape[0])
        self.n1 = int(n1)
        self.two_sided = int(bool(two_sided))
        self.stream = stream if stream is not None else torch.cuda.current_stream(x.device)
        self.ws_bytes = int(self.lib.rmx_naive_workspace_bytes(self.v, self.n, self.L))
        self.workspace = torch.empty(self.ws_bytes, dtype=torch.uint8, device=x.device)
        self.max_out = torch.empty(self.L, dtype=torch.float64, device=x.device)
        self.argmax_out = torch.empty(self.L, dtype=torch.int32, device=x.device)
        self._st = nat.Status()
        self.stats = nat.NaiveStats()

    def _s(self):
        return nat.stream_handle(self.stream)

    def prepare(self) -> None:
        rc = self.lib.rmx_naive_prepare(
            nat.ptr(self.x), self.v, self.n, self.n1, self.L, nat.ptr(self.workspace),
            self.ws_bytes, self._s(), ctypes.byref(self._st))
        nat.raise_for(rc, self._st)

    def tfill(self) -> None:
        rc = self.lib.rmx_naive_tfill(
            self.v, self.n, self.n1, nat.ptr(self.orders), self.L, self.two_sided,
            nat.ptr(self.workspace), self.ws_bytes, self._s(), ctypes.byref(self._st),
            ctypes.byref(self.stats))
        nat.raise_for(rc, self._st)

    def finish(self) -> None:
        rc = self.lib.rmx_naive_finish(
            nat.ptr(self.x), self.v, self.n, self.n1, nat.ptr(self.orders), self.L,
            self.two_sided, nat.ptr(self.max_out), nat.ptr(self.argmax_out),
            nat.ptr(self.workspace), self.ws_bytes, self._s(), ctypes.byref(self._st),
            ctypes.byref(self.stats))
        nat.raise_for(rc, self._st)

    def run(self):
        """All phases in one ABI call (rmx_naive_maxnull)."""
        rc = self.lib.rmx_naive_maxnull(
            nat.ptr(self.x), self.v, self.n, self.n1, nat.ptr(self.orders), self.L,
            self.two_sided, nat.ptr(self.max_out), nat.ptr(self.argmax_out),
            nat.ptr(self.workspace), self.ws_bytes, self._s(), ctypes.byref(self._st),
            ctypes.byref(self.stats))
        nat.raise_for(rc, self._st)
        return self.max_out, self.argmax_out

    def tfill_debug(self):
        """t~ for every (perm, voxel) from the tensor-core epilogue (float32,
        (L, v)); validation only."""
        import torch

        t = torch.full((self.L, self.v), float("nan"), dtype=torch.float32, device=self.x.device)
        self.prepare()
        rc = self.lib.rmx_naive_tfill_debug(
            self.v, self.n, self.n1, nat.ptr(self.orders), self.L, self.two_sided, nat.ptr(t),
            nat.ptr(self.workspace), self.ws_bytes, self._s(), ctypes.byref(self._st))
        nat.raise_for(rc, self._st)
        return t


def tstat_exact_device(x, n1: int, orders, stream=None):
    """(L, v) float64 statistics, bit-identical to the reference, on device."""
    import torch

    lib = nat.load()
    v, n = int(x.shape[0]), int(x.shape[1])
    L = int(orders.shape[0])
    out = torch.empty((L, v), dtype=torch.float64, device=x.device)
    stream = stream if stream is not None else torch.cuda.current_stream(x.device)
    st = nat.Status()
    rc = lib.rmx_tstat_exact(nat.ptr(x), v, n, int(n1), nat.ptr(orders), L, nat.ptr(out), v,
                             nat.stream_handle(stream), ctypes.byref(st))
    nat.raise_for(rc, st)
    return out


def upload(x_values: np.ndarray, orders: np.ndarray, device):
    """Host -> device copies of the data matrix and the label matrix
    (page-locked in place, see hostmem.py)."""
    from .hostmem import to_device

    xd = to_device(np.ascontiguousarray(x_values, dtype=np.float64), device)
    od = to_device(np.ascontiguousarray(orders, dtype=np.int16), device)
    return xd, od


def data_to_device(x, device, one_shot: bool = False):
    """(v, n) float64 device copy of a DataMatrix, uploaded from its float32
    source when it keeps one (half the bytes; the upcast is exact).
    one_shot: through a page-locked staging ring instead of page-locking the
    array in place (cheaper for an array uploaded once, hostmem.upload_staged)."""
    import torch

    from .hostmem import to_device, upload_staged

    up = upload_staged if one_shot else to_device
    x = as_data_matrix(x)
    if x.float32_values is not None:
        return up(x.float32_values, device).to(dtype=torch.float64)
    return up(x.values, device)


def run_naive_ex(x, plan, materialize: bool = False, two_sided: bool = False,
                 threads: Optional[int] = None,
                 mem_cap_bytes: int = DEFAULT_MEM_CAP_BYTES) -> NaiveResult:
    """``run_naive`` with the argmax voxel and engine diagnostics."""
    x = as_data_matrix(x)
    plan = as_plan(plan)
    if plan.subjects != x.subjects:
        raise UsageError("plan and data matrix disagree on subject count")
    v, L = x.voxels, plan.count
    if materialize:
        needed = v * L * 8
        if needed > mem_cap_bytes:
            raise UsageError(
                f"materializing the statistic matrix needs {needed} bytes "
                f"({v} voxels x {L} permutations x 8), above the cap {mem_cap_bytes}; "
                f"raise the cap or drop --dump-T"
            )
    resolve_threads(threads)
    device = cuda_device()
    mx, am, job = _run_from_host(x, plan, two_sided, device)
    T = None
    if materialize:
        T = tstat_exact_device(job.x, x.n1, job.orders).t().contiguous().cpu().numpy()
    return NaiveResult(mx, am.astype(np.int64), job.stats.as_dict(), T)


def _run_from_host(x, plan, two_sided: bool, device, lo: int = 0, hi: Optional[int] = None):
    """One rmx_naive_maxnull_host_plan(_f32) call: host X in (page-locked in
    place; the float32 source when the DataMatrix keeps one),
    the plan's labels generated on the device from its seed (rmx_plan_orders'
    streams, bit-identical to numpy) while X's first chunk uploads, the X
    upload overlapped with the engine chunk by chunk, host max/argmax out.
    Returns (max, argmax, job) -- the job keeps the device copies for
    follow-up work (materialisation).  [lo, hi): a permutation range of the
    plan (one rank's shard, rmx_naive_maxnull_host_plan_range*)."""
    import torch

    from .hostmem import pinned, pinned_empty

    n1 = x.n1
    f32 = x.float32_values
    xh = pinned(f32 if f32 is not None else x.values)
    v, n = xh.shape
    hi = int(plan.count) if hi is None else int(hi)
    L = hi - int(lo)
    ranged = lo != 0 or hi != int(plan.count)
    if n > 32767:
        raise UsageError(f"subject count {n} exceeds the int16 label format")
    xd = torch.empty((v, n), dtype=torch.float64, device=device)
    od = torch.empty((L, n), dtype=torch.int16, device=device)
    job = NaiveJob(xd, n1, od, two_sided)
    mx = pinned_empty((L,), np.float64)
    am = pinned_empty((L,), np.int32)
    seed = ctypes.c_uint64(int(plan.master_seed) & ((1 << 64) - 1))
    tail = (L, job.two_sided, mx.ctypes.data, am.ctypes.data)
    bufs = (nat.ptr(xd), nat.ptr(od), nat.ptr(job.max_out), nat.ptr(job.argmax_out),
            nat.ptr(job.workspace), job.ws_bytes, job._s(), ctypes.byref(job._st),
            ctypes.byref(job.stats))
    head = (xh.ctypes.data, v, n, int(n1), seed) + ((int(lo),) if ranged else ())
    if f32 is not None:
        x32 = torch.empty((v, n), dtype=torch.float32, device=device)
        fn = (job.lib.rmx_naive_maxnull_host_plan_range_f32 if ranged
              else job.lib.rmx_naive_maxnull_host_plan_f32)
        rc = fn(*head, *tail, nat.ptr(x32), *bufs)
        del x32  # the call is synchronous
    else:
        fn = (job.lib.rmx_naive_maxnull_host_plan_range if ranged
              else job.lib.rmx_naive_maxnull_host_plan)
        rc = fn(*head, *tail, *bufs)
    nat.raise_for(rc, job._st)
    return mx.copy(), am.copy(), job


def run_naive(x, plan, materialize: bool = False, two_sided: bool = False,
              threads: Optional[int] = None, mem_cap_bytes: int = DEFAULT_MEM_CAP_BYTES):
    """Drop-in for the reference ``run_naive`` (naive.py:60-109)."""
    res = run_naive_ex(x, plan, materialize, two_sided, threads, mem_cap_bytes)
    plan = as_plan(plan)
    v, L = as_data_matrix(x).voxels, plan.count
    counters = {
        "full_statistic_evaluations": v * L,
        "subsampled_statistic_evaluations": 0,
        "statistic_evaluations": v * L,
    }
    mat = StatMatrix(res.T, plan) if res.T is not None else None
    return MaxNull(res.maxima), mat, counters


# ---------------------------------------------------------------------------
# .mat0 file in, streamed: the reference CLI's naive run
# (cli.py:70-116: read_matrix -> run_naive(materialize=dump_t) -> write_array)
# without ever holding X or T on the host.

_RING: dict = {}


def _staging_ring(nbytes: int) -> np.ndarray:
    """A cached page-locked float64 staging ring of at least `nbytes`."""
    from .hostmem import pinned_empty

    have = _RING.get("ring")
    if have is None or have.nbytes < nbytes:
        have = pinned_empty((-(-nbytes // 8),), np.float64)
        _RING["ring"] = have
    return have


def _mat0_data_header(path):
    """(v, n, n1, n2) of a .mat0 data file, with the reference read_matrix's
    DataFormatError for a bare matrix or an invalid group split
    (matio.py:83-91 + DataMatrix validation, model.py)."""
    from .exceptions import DataFormatError
    from .matfiles import mat0_info

    v, n, n1, n2 = mat0_info(path)
    if n1 == 0 and n2 == 0:
        raise DataFormatError(
            f"{path}: header carries no group split (n1=n2=0); "
            f"this file stores a bare matrix, not subject data")
    if min(n1, n2) < 2:
        raise DataFormatError(
            f"{path}: need at least two subjects per group for variance estimates, "
            f"got n1={n1}, n2={n2}")
    if n1 + n2 != n:
        raise DataFormatError(
            f"{path}: group sizes n1+n2={n1 + n2} do not match column count {n}")
    return v, n, n1, n2


def run_naive_mat0(path, plan, two_sided: bool = False, dump_t=None,
                   threads: Optional[int] = None, staging_bytes: int = 192 << 20,
                   lo: int = 0, hi: Optional[int] = None) -> NaiveResult:
    """NaivePT over the data matrix stored in the .mat0 file `path`.

    The float64 payload is streamed file -> page-locked ring -> device by
    ``rmx_naive_maxnull_mat0`` (parallel positional reads of the next piece
    while the copy engine moves this one and K0/K1 work on the chunks that
    have landed), so the read overlaps the engine instead of preceding it.
    With ``dump_t`` the (v, L) statistic matrix is then written to that path
    as a bare .mat0 straight from the device (``rmx_tstat_dump_mat0``,
    slab by slab), bit-identical to the reference's ``write_array(mat.values,
    dump_t)`` and with no memory cap.  ``[lo, hi)``: a permutation range of
    the plan (one rank's shard); ``maxima`` then holds those entries.
    Results equal ``run_naive_ex(read_matrix(path), plan, ...)`` bit for bit.
    """
    import torch

    from .exceptions import DataFormatError
    from .hostmem import pinned_empty
    from .matfiles import _bpath, nonfinite_error

    plan = as_plan(plan)
    v, n, n1, n2 = _mat0_data_header(path)
    if plan.subjects != n:
        raise UsageError("plan and data matrix disagree on subject count")
    nthreads = resolve_threads(threads)
    device = cuda_device()
    hi = int(plan.count) if hi is None else int(hi)
    L = hi - int(lo)
    if not 0 <= lo < hi <= plan.count:
        raise UsageError(f"permutation range [{lo}, {hi}) outside the plan of {plan.count}")
    if n > 32767:
        raise UsageError(f"subject count {n} exceeds the int16 label format")
    xd = torch.empty((v, n), dtype=torch.float64, device=device)
    od = torch.empty((L, n), dtype=torch.int16, device=device)
    job = NaiveJob(xd, n1, od, two_sided)
    mx = pinned_empty((L,), np.float64)
    am = pinned_empty((L,), np.int32)
    ring_bytes = max(int(staging_bytes), 3 * n * 8)
    ring = _staging_ring(ring_bytes)
    bad = ctypes.c_int64(-1)
    seed = ctypes.c_uint64(int(plan.master_seed) & ((1 << 64) - 1))
    rc = job.lib.rmx_naive_maxnull_mat0(
        _bpath(path), v, n, n1, seed, int(lo), L, job.two_sided, mx.ctypes.data, am.ctypes.data,
        ring.ctypes.data, ring_bytes, nthreads, ctypes.byref(bad), nat.ptr(xd), nat.ptr(od),
        nat.ptr(job.max_out), nat.ptr(job.argmax_out), nat.ptr(job.workspace), job.ws_bytes,
        job._s(), ctypes.byref(job._st), ctypes.byref(job.stats))
    if rc == nat.RMX_E_FORMAT and bad.value >= 0:
        raise nonfinite_error(path, bad.value, n)
    if rc == nat.RMX_E_FORMAT:
        raise DataFormatError(job._st.msg.decode(errors="replace"))
    nat.raise_for(rc, job._st)
    res = NaiveResult(mx.copy(), am.astype(np.int64), job.stats.as_dict(), None)
    if dump_t is not None:
        dump_statistic_matrix_device(job.x, n1, job.orders, dump_t, threads=nthreads,
                                     stream=job.stream)
    return res


def dump_statistic_matrix_device(x, n1: int, orders, path, threads: Optional[int] = None,
                                 staging_bytes: int = 256 << 20, stream=None) -> None:
    """Write the (v, L) statistic matrix of device-resident X (v x n float64)
    and labels (L x n int16) to `path` as a bare .mat0, streamed slab by slab
    (rmx_tstat_dump_mat0)."""
    import torch

    from .matfiles import _bpath

    lib = nat.load()
    v, n = int(x.shape[0]), int(x.shape[1])
    L = int(orders.shape[0])
    ring_bytes = max(int(staging_bytes), 2 * L * 8)
    ring = _staging_ring(ring_bytes)
    stream = stream if stream is not None else torch.cuda.current_stream(x.device)
    st = nat.Status()
    rc = lib.rmx_tstat_dump_mat0(nat.ptr(x), v, n, int(n1), nat.ptr(orders), L, _bpath(path),
                                 ring.ctypes.data, ring_bytes, resolve_threads(threads),
                                 nat.stream_handle(stream), ctypes.byref(st))
    nat.raise_for(rc, st)


def dump_statistic_matrix(x, plan, path, threads: Optional[int] = None) -> None:
    """The reference's ``--dump-T`` output for an in-memory DataMatrix:
    ``write_array(run_naive(x, plan, materialize=True)[1].values, path)``,
    streamed from the device instead of materialised on the host."""
    from .labels import device_orders

    x = as_data_matrix(x)
    plan = as_plan(plan)
    if plan.subjects != x.subjects:
        raise UsageError("plan and data matrix disagree on subject count")
    device = cuda_device()
    xd = data_to_device(x, device)
    od = device_orders(plan.master_seed, 0, plan.count, x.subjects, device)
    dump_statistic_matrix_device(xd, x.n1, od, path, threads=threads)
