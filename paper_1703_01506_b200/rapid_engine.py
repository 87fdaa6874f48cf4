"""RapidPT on the B200: drop-in ``train`` / ``recover`` / ``run_rapid`` and the
low-rank entry points of the reference's lrmc module.

Reference: rapid.py:72-275 and lrmc.py:85-268.  What runs where:

  host (numpy, the reference's own streams -> bit-identical inputs)
      permutation labels, Omega draws (RECOVER_OMEGA, TRAIN_OMEGA), the basis
      initialisation draw (BASIS_INIT), the max-gap normals (SHIFT_GAP)
  device (librmx.so)
      training columns       exact fp64 statistic kernel (bit-identical)
      GROUSE                 native update loop: gathered Gram + Cholesky
                             solve, residual, prediction, rank-one rotation,
                             CholeskyQR2 re-orthonormalisation
      sigma, mu, maxima      batched LS fits, residual mean/variance,
                             completion + max kernels
      recovery               K2 exact Omega statistics -> K3 batched gathered
                             Gram + Cholesky -> K4 completion W.U^T fused with
                             Philox residual noise and the row max

Deliberate deviations:
  * the recovery residual noise is a counter-based Philox N(0,1) keyed by
    (seed, permutation, voxel), not numpy's SFC64 stream (v doubles per
    permutation cannot be shipped) -- parity is distributional
    for sigma > 0 and exact-to-tolerance for sigma = 0;
  * the restricted-basis condition test uses Cholesky pivots (rank-deficient
    restrictions are detected; the reference's 1e12 eigenvalue threshold is
    approximated by a lower bound, see solve_block);
  * GROUSE runs in a different summation order than OpenBLAS, so the trained
    basis agrees with the reference's up to rounding, not bit for bit.
"""

from __future__ import annotations

import ctypes
import math
import os
import time
from typing import Optional

import numpy as np

from . import _native as nat
from .domain import (
    Basis,
    MaxNull,
    ObservedColumn,
    PendingBasis,
    SubspaceModel,
    as_data_matrix,
    as_plan,
    observed_rows,
)
from .hostpar import fill_rows
from .exceptions import (
    DegenerateVoxelError,
    IllConditionedBasisError,
    NumericalError,
    UsageError,
)
from .labels import device_orders, plan_orders
from .naive_engine import cuda_device, data_to_device, resolve_threads, tstat_exact_device
from .rng import BASIS_INIT, RECOVER_OMEGA, SHIFT_GAP, TRAIN_OMEGA, omega_draw, stream

COND_LIMIT = 1e12
_BLOCK = 256            # reference recovery span (rapid.py:36), used for error parity
_RESAMPLE_ATTEMPTS = 5
_LSQ_BATCH_BYTES = 1 << 30


# ---------------------------------------------------------------- host draws
def draw_omegas(seed: int, domain: int, lo: int, hi: int, v: int, k: int,
                extra: Optional[int] = None, workers: Optional[int] = None) -> np.ndarray:
    """Sorted observation sets of indices [lo, hi) of a stream domain (first
    draw of each stream): rapid.py:158-160 / lrmc.py:237-241."""

    def row(i):
        path = (domain, lo + i) if extra is None else (domain, lo + i, extra)
        return omega_draw(stream(seed, *path), v, k)

    return fill_rows((k,), np.int32, row, hi - lo, workers)


def device_omegas(seed: int, domain: int, lo: int, hi: int, v: int, k: int, dev,
                  extra: Optional[int] = None):
    """draw_omegas on the GPU (rmx_omega_draws: numpy's Generator.choice
    restated bit for bit), as an (hi - lo, k) int32 CUDA tensor; numpy's
    tail-shuffle branch (v > 10000 and k > v / 50) is drawn on the host."""
    torch = _torch()
    out = torch.empty((max(hi - lo, 0), k), dtype=torch.int32, device=dev)
    if hi <= lo:
        return out
    if v > 10000 and k > v // 50:
        return _to_dev(draw_omegas(seed, domain, lo, hi, v, k, extra=extra), dev)
    st = nat.Status()
    rc = nat.load().rmx_omega_draws(ctypes.c_uint64(int(seed) & ((1 << 64) - 1)), int(domain),
                                    int(lo), int(hi - lo), -1 if extra is None else int(extra),
                                    int(v), int(k), nat.ptr(out), _stream(dev), ctypes.byref(st))
    nat.raise_for(rc, st)
    return out


def draw_normals(seed: int, domain: int, lo: int, hi: int, v: int) -> np.ndarray:
    """stream(seed, domain, i).standard_normal(v) for i in [lo, hi), fp32
    (numpy's float64 values, cast), by the native generator on all host
    threads (normals.py)."""
    from .normals import standard_normal_rows

    return standard_normal_rows(seed, domain, lo, hi, v, dtype=np.float32)


def _resample(seed: int, path: tuple, attempt: int, v: int, k: int) -> np.ndarray:
    """The attempt-th redraw of a stream whose first draw was already used
    (the reference draws again from the same generator, lrmc.py:240-250,
    rapid.py:180)."""
    g = stream(seed, *path)
    for _ in range(attempt):
        g.choice(v, size=k, replace=False)
    return np.sort(g.choice(v, size=k, replace=False)).astype(np.int32)


# ---------------------------------------------------------------- device helpers
def _torch():
    import torch

    return torch


def _stream(dev):
    return nat.stream_handle(_torch().cuda.current_stream(dev))


def _to_dev(a, dev, dtype=None):
    torch = _torch()
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.to(dev)


def _lsq(u_dev, r: int, idx_dev, k: int, vals_dev, B: int):
    """Batched solve_block on device -> (W (B x r), flags (B), norms (B x 4))."""
    torch = _torch()
    dev = u_dev.device
    W = torch.empty((B, r), dtype=torch.float64, device=dev)
    flags = torch.empty(B, dtype=torch.int32, device=dev)
    norms = torch.empty((B, 4), dtype=torch.float64, device=dev)
    per = (r + 1) * (r + 1) * 8 + 32
    batch = max(1, min(B, _LSQ_BATCH_BYTES // per))
    ws_bytes = int(nat.load().rmx_lsq_workspace_bytes(r, batch))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    nat.call("rmx_lsq_solve", nat.ptr(u_dev), r, r, nat.ptr(idx_dev), k, nat.ptr(vals_dev), B,
             nat.ptr(W), nat.ptr(flags), nat.ptr(norms), nat.ptr(ws), ws_bytes, _stream(dev))
    return W, flags, norms


_RECOVER_SETTLE = 1e-4


def _lsq_tc(u_dev, r: int, idx_dev, k: int, vals_dev, B: int, settle: float = 0.0):
    """Batched solve_block with the tensor-core Gram + fp64 refinement
    (rmx_lsq_solve_tc_settle; settle = 0: two refinement steps on every
    system, else the second only where the first correction exceeds
    settle |w|) -> (W (B x r), flags (B), stats [tc used, fp64 redos])."""
    torch = _torch()
    dev = u_dev.device
    W = torch.empty((B, r), dtype=torch.float64, device=dev)
    flags = torch.empty(B, dtype=torch.int32, device=dev)
    per = (r + 1) * (r + 1) * 8 + 32
    batch = max(1, min(B, _LSQ_BATCH_BYTES // per))
    ws_bytes = int(nat.load().rmx_lsq_workspace_bytes(r, batch))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    stats = (ctypes.c_int32 * 2)()
    nat.call("rmx_lsq_solve_tc_settle", nat.ptr(u_dev), r, int(u_dev.shape[0]), r,
             nat.ptr(idx_dev), k, nat.ptr(vals_dev), B, nat.ptr(W), nat.ptr(flags), nat.ptr(ws),
             ws_bytes, stats, float(settle), _stream(dev))
    return W, flags, (int(stats[0]), int(stats[1]))


def _orthonormalize(u_dev, force: bool) -> float:
    drift = ctypes.c_double(0.0)
    v, r = u_dev.shape
    nat.call("rmx_orthonormalize", nat.ptr(u_dev), v, r, int(force), ctypes.byref(drift),
             _stream(u_dev.device))
    return float(drift.value)


def _complete_max(u32, w32, perm_base: int, sigma: float, mu: float, seed: int, two_sided: bool,
                  znoise=None, base=None):
    torch = _torch()
    v, r = u32.shape
    B = w32.shape[0]
    out = torch.empty(B, dtype=torch.float64, device=u32.device)
    nat.call("rmx_complete_max", nat.ptr(u32), v, r, nat.ptr(w32), B, int(perm_base),
             float(sigma), float(mu), ctypes.c_uint64(int(seed) & ((1 << 64) - 1)),
             int(bool(two_sided)), nat.ptr(znoise), nat.ptr(base), nat.ptr(out),
             _stream(u32.device))
    return out


def _basis_device(model: SubspaceModel, dev):
    """fp64 basis on device, cached on the (frozen) model object."""
    cache = getattr(model, "_rmx_dev", None)
    if cache is not None and cache[0] == dev:
        return cache[1], cache[2]
    u = _to_dev(model.basis.matrix, dev)
    u32 = u.to(_torch().float32)
    object.__setattr__(model, "_rmx_dev", (dev, u, u32))
    return u, u32


# ---------------------------------------------------------------- lrmc API
def init_basis(v: int, r: int, seed: int) -> Basis:
    """Orthonormal basis of a seeded Gaussian draw (reference lrmc.py:85-93):
    the draw is the reference's BASIS_INIT stream; the orthonormalisation is
    CholeskyQR2 on the device (same span; column signs may differ from
    numpy's Householder QR, which GROUSE is invariant to)."""
    if r > v:
        raise UsageError(f"rank {r} exceeds dimension {v}")
    if r < 1:
        raise UsageError("rank must be >= 1")
    dev = cuda_device()
    u = _basis_init_async(seed, v, r, dev)()
    _orthonormalize(u, force=True)
    return Basis(u.cpu().numpy(), copy=False)


def _lsq_exact(u_dev, r: int, idx_dev, k: int, vals_dev, B: int):
    """rmx_lsq_solve_exact: reference-semantics fits -> (W (B x r) on the
    device, flags (B,) host, conds (B,) host)."""
    torch = _torch()
    dev = u_dev.device
    W = torch.empty((B, r), dtype=torch.float64, device=dev)
    flags = np.zeros(B, dtype=np.int32)
    conds = np.zeros(B, dtype=np.float64)
    nat.call("rmx_lsq_solve_exact", nat.ptr(u_dev), r, r, nat.ptr(idx_dev), k, nat.ptr(vals_dev),
             B, nat.ptr(W), flags.ctypes.data, conds.ctypes.data, _stream(dev))
    return W, flags, conds


def solve_block(u_stack: np.ndarray, values: np.ndarray):
    """Batched LS fits (reference lrmc.py:127-149) -> (w (B, r), conds (B,)).

    conds = sqrt(lambda_max / lambda_min) of each normal matrix (inf when
    lambda_min <= 0), from the device's Householder tridiagonalisation +
    bisection; systems with cond > 1e12 get w = U_Omega^T values (the
    reference's solve against the identity)."""
    u_stack = np.ascontiguousarray(u_stack, dtype=np.float64)
    values = np.ascontiguousarray(values, dtype=np.float64)
    B, k, r = u_stack.shape
    dev = cuda_device()
    torch = _torch()
    U = _to_dev(u_stack.reshape(B * k, r), dev)
    idx = torch.arange(B * k, dtype=torch.int32, device=dev).reshape(B, k)
    W, _, conds = _lsq_exact(U, r, idx, k, _to_dev(values, dev), B)
    return W.cpu().numpy(), conds


def fit_coefficients(b: Basis, col: ObservedColumn) -> np.ndarray:
    """LS coefficients on the observed rows (reference lrmc.py:107-124)."""
    if col.size < b.rank:
        raise UsageError(f"{col.size} observed rows cannot determine {b.rank} coefficients")
    if col.indices[-1] >= b.voxels:
        raise UsageError("observed row index outside the basis")
    w, conds = solve_block(b.matrix[col.indices][None], col.values[None])
    if not np.isfinite(conds[0]) or conds[0] > COND_LIMIT:
        raise IllConditionedBasisError(float(conds[0]))
    return w[0]


def track_update(b: Basis, col: ObservedColumn, step: float):
    """One GROUSE update (reference lrmc.py:160-193) on the device: mutates and
    returns `b`, plus the pre-update fit residual norm on the observed rows.
    Raises IllConditionedBasisError(cond) like the reference's _gram_fit."""
    if col.size < b.rank:
        raise UsageError(f"{col.size} observed rows cannot determine {b.rank} coefficients")
    if col.indices[-1] >= b.voxels:
        raise UsageError("observed row index outside the basis")
    dev = cuda_device()
    u = _to_dev(b.matrix, dev)
    idx = _to_dev(np.asarray(col.indices, dtype=np.int32), dev)
    vals = _to_dev(np.asarray(col.values, dtype=np.float64), dev)
    rn = ctypes.c_double(0.0)
    nat.call("rmx_track_update", nat.ptr(u), b.voxels, b.rank, nat.ptr(idx), col.size,
             nat.ptr(vals), float(step), ctypes.byref(rn), _stream(dev))
    b.matrix[...] = u.cpu().numpy()
    return b, float(rn.value)


def complete_column(b: Basis, w: np.ndarray) -> np.ndarray:
    """U w (reference lrmc.py:152-157)."""
    w = np.asarray(w, dtype=np.float64)
    if w.shape != (b.rank,):
        raise UsageError(f"coefficients must have shape ({b.rank},), got {w.shape}")
    dev = cuda_device()
    torch = _torch()
    u = _to_dev(b.matrix, dev)
    out = torch.empty(b.voxels, dtype=torch.float64, device=dev)
    nat.call("rmx_gemv", nat.ptr(u), b.voxels, b.rank, nat.ptr(_to_dev(w, dev)), nat.ptr(out),
             _stream(dev))
    return out.cpu().numpy()


class TrainingResult:
    def __init__(self, basis, passes, updates, pass_residuals, final_omegas, converged):
        self.basis = basis
        self.passes = passes
        self.updates = updates
        self.pass_residuals = pass_residuals
        self.final_omegas = final_omegas
        self.converged = converged


def _basis_init_async(seed: int, v: int, rank: int, dev):
    """init_basis's normals (lrmc.py:85-93: ONE sequential stream(seed,
    BASIS_INIT) of v x rank doubles, 2.1e8 at config 5) drawn by the native
    generator (normals.py, bit-identical to numpy) on a host thread while the
    X upload, the training columns, the Omega draws and the recovery
    statistics run on the GPU: 8 MB blocks into two page-locked buffers,
    each block's upload (side stream) overlapping the next block's draw.
    Returns a joiner giving the (v, rank) fp64 device tensor."""
    torch = _torch()
    from .hostmem import pinned_empty
    from .normals import NormalStream

    side = torch.cuda.Stream(dev)
    out = torch.empty((v, rank), dtype=torch.float64, device=dev)
    ring = pinned_empty((1 << 21,), np.float64)  # two 8 MB halves
    import threading

    drawn = threading.Event()  # set when the stream is drawn (other host draws wait for it)
    trace = os.environ.get("RMX_TRACE_BASIS")

    def work():
        t_start = time.perf_counter()
        torch.cuda.set_device(dev)
        gen = NormalStream(seed, (BASIS_INIT,))
        try:
            # one native call: draw into a ring half while the other half's
            # upload is in flight (no per-block Python, no GIL)
            gen.fill_device(out, ring, side)
        finally:
            gen.close()
            drawn.set()
        if trace:
            print(f"[basis-init] draw + upload {time.perf_counter() - t_start:.3f}s", flush=True)
        return out

    join = _host_async(work)

    def joined():
        t = join()
        cur = torch.cuda.current_stream(dev)
        cur.wait_stream(side)
        t.record_stream(cur)
        return t

    joined.drawn = drawn
    return joined


def _to_dev_async(draw, dev):
    """draw() on a host thread, then its upload on a side stream from the
    same thread (the GPU meanwhile runs GROUSE); the joiner orders the
    current stream after the copy."""
    torch = _torch()
    side = torch.cuda.Stream(dev)

    def work():
        a = draw()
        # through the page-locked staging ring: a pageable copy of this size
        # (1.7 GB of SHIFT_GAP normals at config 5) holds the CUDA context lock
        # while the driver stages it, stalling the GROUSE launch thread
        from .hostmem import upload_staged

        with torch.cuda.stream(side):
            return upload_staged(np.ascontiguousarray(a), dev, side)

    join = _host_async(work)

    def joined():
        t = join()
        cur = torch.cuda.current_stream(dev)
        cur.wait_stream(side)
        t.record_stream(cur)  # allocated on the side stream, consumed on this one
        return t

    return joined


def _host_array_async(shape):
    """A float64 host array with every page already touched, prepared on a
    host thread while the GPU runs GROUSE (the host is otherwise idle)."""

    def work():
        a = np.empty(shape, dtype=np.float64)
        a.fill(0.0)
        return a

    return _host_async(work)


def _d2h_async(t, dest):
    """Copy the device tensor `t` into the host array dest() on a side stream
    from a host thread, overlapping later GPU work: 32 MB row blocks through
    two page-locked buffers, block c + 1 in flight while block c is copied
    out on the host.  Returns the joiner."""
    torch = _torch()
    side = torch.cuda.Stream(t.device)
    side.wait_stream(torch.cuda.current_stream(t.device))

    def work():
        h = dest()
        v, width = t.shape
        rows = max(1, min(v, (32 << 20) // (8 * width)))
        bufs = [torch.empty((rows, width), dtype=t.dtype, pin_memory=True) for _ in range(2)]
        evs = [torch.cuda.Event(), torch.cuda.Event()]
        blocks = [(lo, min(v, lo + rows)) for lo in range(0, v, rows)]

        def issue(c):
            lo, hi = blocks[c]
            bufs[c & 1][: hi - lo].copy_(t[lo:hi], non_blocking=True)
            evs[c & 1].record(side)

        with torch.cuda.stream(side):
            issue(0)
            for c, (lo, hi) in enumerate(blocks):
                evs[c & 1].synchronize()
                if c + 1 < len(blocks):
                    issue(c + 1)
                h[lo:hi] = bufs[c & 1].numpy()[: hi - lo]
        return h

    return _host_async(work)


def _train_basis_device(t_dev, v: int, ell: int, k: int, rank: int, seed: int,
                        max_passes: int, tolerance: float, init=None, host_basis: bool = False,
                        before_grouse=None):
    """GROUSE on device.  t_dev: (ell, v) fp64 training statistics; init: a
    joiner from _basis_init_async (else the normals are drawn here)."""
    torch = _torch()
    dev = t_dev.device
    if init is None:
        init = _basis_init_async(seed, v, rank, dev)
    # the observation sets of every pass (stream(seed, TRAIN_OMEGA, i, p), drawn
    # on the GPU) while the host still draws the BASIS_INIT normals
    om_dev = torch.empty((max_passes, ell, k), dtype=torch.int32, device=dev)
    for p in range(max_passes):
        om_dev[p] = device_omegas(seed, TRAIN_OMEGA, 0, ell, v, k, dev, extra=p)
    _mark("train_omegas")
    u = init()
    host_u = _host_array_async((v, rank)) if host_basis else None
    _mark("basis_normals_ready")
    _orthonormalize(u, force=True)
    _mark("basis_upload+qr")
    final = torch.empty((ell, k), dtype=torch.int32, device=dev)
    pass_resid = (ctypes.c_double * max_passes)()
    passes, conv, updates = ctypes.c_int32(0), ctypes.c_int32(0), ctypes.c_int64(0)

    def cb(_user, col, pas, attempt, out):
        try:
            idx = _resample(seed, (TRAIN_OMEGA, col, pas), attempt, v, k)
            ctypes.memmove(out, idx.ctypes.data, idx.nbytes)
            return 0
        except Exception:
            return 1

    cbf = nat.OMEGA_CB(cb)
    if before_grouse is not None:
        before_grouse()
    nat.call("rmx_grouse_train", nat.ptr(t_dev), v, ell, rank, k, nat.ptr(om_dev), max_passes,
             float(tolerance), nat.ptr(u), cbf, None, pass_resid, ctypes.byref(passes),
             ctypes.byref(conv), ctypes.byref(updates), nat.ptr(final), _stream(dev))
    _mark("grouse")
    res = [pass_resid[i] for i in range(passes.value)]
    return u, final, int(passes.value), bool(conv.value), int(updates.value), res, host_u


def train_basis(t_ex: np.ndarray, k: int, rank: int, seed: int, max_passes: int = 50,
                tolerance: float = 1e-3, resample_attempts: int = 5) -> TrainingResult:
    """GROUSE passes over the training columns (reference lrmc.py:208-268)."""
    t_ex = np.asarray(t_ex, dtype=np.float64)
    v, ell = t_ex.shape
    if k < rank:
        raise UsageError(f"{k} observed rows per update cannot identify rank {rank}")
    if k > v:
        raise UsageError(f"observed rows {k} exceed voxel count {v}")
    dev = cuda_device()
    t_dev = _to_dev(np.ascontiguousarray(t_ex.T), dev)
    u, final, passes, conv, updates, res, _ = _train_basis_device(t_dev, v, ell, k, rank, seed,
                                                               max_passes, tolerance)
    fo = final.cpu().numpy()
    return TrainingResult(Basis(u.cpu().numpy(), copy=False), passes, updates, res,
                          [fo[i].astype(np.int64) for i in range(ell)], conv)


# ---------------------------------------------------------------- train / recover
_PHASE_LOG = None  # tools/rapid_phases.py sets a list: (tag, seconds) marks, device-synchronised


_HOST_MARKS = os.environ.get("RMX_RAPID_HOSTMARKS")  # diagnostics: host-side marks, no device sync


def _mark(tag: str) -> None:
    if _PHASE_LOG is not None:
        _torch().cuda.synchronize()
        _PHASE_LOG.append((tag, time.perf_counter()))
    elif _HOST_MARKS:
        print(f"[host-mark] {time.perf_counter():.3f} {tag}", flush=True)


def _host_async(fn):
    """Run fn() on a background host thread; returns a joiner that re-raises."""
    import threading

    box = {}

    def work():
        try:
            box["a"] = fn()
        except BaseException as exc:  # re-raised by the joiner
            box["e"] = exc

    th = threading.Thread(target=work, name="rmx-host-draw", daemon=True)
    th.start()

    def join():
        th.join()
        if "e" in box:
            raise box["e"]
        return box.pop("a")

    return join


class _RecoverInputs:
    """Recovery inputs that do not depend on the trained basis (rapid.py:
    158-168: the shuffles, the Omega draws and the exact statistics at the
    Omega rows), computed by run_rapid while the host draws init_basis's
    normals.  A degenerate-voxel report is kept and raised when recovery
    starts, i.e. in the reference's order (after training)."""

    def __init__(self, x, xd, plan, seed: int, ell: int, k: int, dev):
        torch = _torch()
        L, v = plan.count, x.voxels
        self.key = (int(seed), ell, k, L, plan.master_seed)
        self.xd = xd
        self.od = device_orders(plan.master_seed, ell, L, x.subjects, dev)
        self.omd = device_omegas(seed, RECOVER_OMEGA, ell, L, v, k, dev)
        self.t = torch.empty((L - ell, k), dtype=torch.float64, device=dev)
        self.st = nat.Status()
        self.rc = nat.load().rmx_rapid_stats(nat.ptr(xd), v, x.subjects, x.n1, nat.ptr(self.od),
                                             nat.ptr(self.omd), L - ell, k, nat.ptr(self.t),
                                             _stream(dev), ctypes.byref(self.st))


def _train_device(x, cfg, prefetch_recovery: bool = False):
    """Shared by train() and run_rapid(): returns (model, training maxima,
    t_dev (ell x v, device), recovery inputs or None).  The GPU work that
    does not need the basis (X upload, training columns, Omega draws and --
    for run_rapid -- the recovery statistics) runs while a host thread draws
    init_basis's sequential normals (the max-gap normals on other host
    threads); the basis's host array is prepared during GROUSE."""
    torch = _torch()
    cfg = cfg.resolve(x)
    if cfg.engine != "rapid":
        raise UsageError("training is only meaningful for the rapid engine")
    ell, rank = cfg.training_columns, cfg.rank
    v = x.voxels
    k = observed_rows(cfg.sample_rate, v)
    plan = cfg.plan_for(x)
    dev = cuda_device()
    init = _basis_init_async(cfg.seed, v, rank, dev)    # host, overlapped with the GPU work below
    gap = None
    if cfg.shift_override is None and cfg.shift_estimator != "residual-sup":
        # the SHIFT_GAP streams (needed after GROUSE) start once the serial
        # BASIS_INIT stream (GROUSE's critical path) is drawn: no competition
        # for host cores with the one stream that cannot be parallelised
        def gap_draw():
            init.drawn.wait()
            return draw_normals(cfg.seed, SHIFT_GAP, 0, ell, v)

        gap = _to_dev_async(gap_draw, dev)
    xd = data_to_device(x, dev, one_shot=True)
    od = device_orders(plan.master_seed, 0, ell, x.subjects, dev)
    t_dev = tstat_exact_device(xd, x.n1, od)            # (ell, v), bit-exact columns
    _mark("x_upload+training_columns")
    pre, pre_join = None, None
    if prefetch_recovery and ell < plan.count:
        if os.environ.get("RMX_PREFETCH_SERIAL"):
            pre = _RecoverInputs(x, xd, plan, cfg.seed, ell, k, dev)
        else:
            # recovery's basis-independent inputs on a low-priority side
            # stream from a host thread, concurrently with GROUSE (latency-
            # bound: most SMs idle) instead of in front of it
            lo_prio = torch.cuda.Stream(dev, priority=0)  # the lowest priority
            # after the training columns (GROUSE's input): interleaved with
            # them the prefetch only delayed GROUSE's start
            lo_prio.wait_stream(torch.cuda.current_stream(dev))

            trace_pf = os.environ.get("RMX_TRACE_PREFETCH")
            pf_ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)] if trace_pf else None

            def prefetch():
                torch.cuda.set_device(dev)
                with torch.cuda.stream(lo_prio):
                    if pf_ev:
                        pf_ev[0].record(lo_prio)
                    r = _RecoverInputs(x, xd, plan, cfg.seed, ell, k, dev)
                    done = torch.cuda.Event()
                    done.record(lo_prio)
                    if pf_ev:
                        pf_ev[1].record(lo_prio)
                return r, done

            pre_join = _host_async(prefetch)
        _mark("recovery_prefetch")
    if os.environ.get("RMX_RAPID_SYNC_BEFORE_GROUSE"):  # diagnostics: no prefetch beside GROUSE
        torch.cuda.synchronize()
    hi_prio = torch.cuda.Stream(dev, priority=-100)  # mapped to the highest priority
    hi_prio.wait_stream(torch.cuda.current_stream(dev))
    pre_box = {}

    def prefetch_first():
        # GROUSE's three-stream chain is latency-bound end to end: resident
        # blocks of the prefetch's kernels beside it cost it more than their own
        # duration (config 5: +1.0 s for 0.6 s of prefetch), so the prefetch --
        # which has had the GPU to itself while the host drew the BASIS_INIT
        # normals -- finishes before the first update starts
        if pre_join is not None and not os.environ.get("RMX_PREFETCH_BESIDE_GROUSE"):
            pre_box["r"] = pre_join()
            torch.cuda.current_stream(dev).wait_event(pre_box["r"][1])

    with torch.cuda.stream(hi_prio):
        if pre_join is not None and pf_ev:
            pf_ev[2].record(hi_prio)
        u, final, passes, conv, _, _, host_u = _train_basis_device(
            t_dev, v, ell, k, rank, cfg.seed, cfg.max_passes, cfg.tolerance, init,
            host_basis=prefetch_recovery, before_grouse=prefetch_first)
    if pre_join is not None and pf_ev:
        pf_ev[3].record(hi_prio)
        torch.cuda.synchronize()
        print(f"[prefetch-trace] prefetch start -> end {pf_ev[0].elapsed_time(pf_ev[1]):.1f} ms; "
              f"prefetch start -> basis phase start {pf_ev[0].elapsed_time(pf_ev[2]):.1f} ms; "
              f"basis phase start -> GROUSE end {pf_ev[2].elapsed_time(pf_ev[3]):.1f} ms",
              flush=True)
    torch.cuda.current_stream(dev).wait_stream(hi_prio)
    for tnsr in (u, final):
        tnsr.record_stream(torch.cuda.current_stream(dev))
    if pre_join is not None:
        pre, done = pre_box["r"] if "r" in pre_box else pre_join()
        cur = torch.cuda.current_stream(dev)
        cur.wait_event(done)
        for tnsr in (pre.od, pre.omd, pre.t):
            tnsr.record_stream(cur)
    # fits of the frozen basis on the final pass's observed rows (rapid.py:90-97)
    vals = torch.empty((ell, k), dtype=torch.float64, device=dev)
    nat.call("rmx_gather_rows", nat.ptr(t_dev), v, nat.ptr(final), k, ell, nat.ptr(vals),
             _stream(dev))
    W, flags, norms = _lsq(u, rank, final, k, vals, ell)
    if int(flags.max().item()) != 0:
        raise IllConditionedBasisError(math.inf)
    _mark("final_fits")
    if cfg.sigma_override is not None:
        sigma = float(cfg.sigma_override)
        if sigma < 0:
            raise UsageError("sigma override must be >= 0")
    else:
        resid = torch.empty((ell, k), dtype=torch.float64, device=dev)
        nat.call("rmx_resid_batch", nat.ptr(u), rank, nat.ptr(final), k, nat.ptr(vals),
                 nat.ptr(W), ell, nat.ptr(resid), _stream(dev))
        mv = torch.empty(2, dtype=torch.float64, device=dev)
        nat.call("rmx_mean_var", nat.ptr(resid), ell * k, nat.ptr(mv), _stream(dev))
        sigma = float(math.sqrt(max(float(mv[1].item()), 0.0)))
    tmax = torch.empty(ell, dtype=torch.float64, device=dev)
    nat.call("rmx_row_max", nat.ptr(t_dev), ell, v, int(cfg.two_sided), nat.ptr(tmax),
             _stream(dev))
    training_maxima = tmax.cpu().numpy()
    _mark("sigma+training_maxima")
    u32 = u.to(torch.float32)
    w32 = W.to(torch.float32)
    if cfg.shift_override is not None:
        mu = float(cfg.shift_override)
    elif cfg.shift_estimator == "residual-sup":
        m = _complete_max(u32, w32, 0, 0.0, 0.0, cfg.seed, cfg.two_sided, base=t_dev)
        mu = float(m.max().item())
    else:  # max-gap: gaps to synthetic columns with the reference's SHIFT_GAP normals
        z = gap()
        synth = _complete_max(u32, w32, 0, sigma, 0.0, cfg.seed, cfg.two_sided, znoise=z)
        mu = float(np.mean(training_maxima - synth.cpu().numpy()))
    _mark("shift")
    if prefetch_recovery:  # run_rapid: the host copy overlaps recovery (joined before it returns)
        basis = PendingBasis(_d2h_async(u, host_u), tuple(u.shape))
    else:
        basis = Basis(u.cpu().numpy(), copy=False)
    model = SubspaceModel(
        basis=basis, residual_std=sigma, max_shift=mu,
        training_columns=ell, sample_rate=cfg.sample_rate, training_maxima=training_maxima,
        two_sided=cfg.two_sided, seed=cfg.seed, passes=passes, converged=conv)
    object.__setattr__(model, "_rmx_dev", (dev, u, u32))
    _mark("model_basis_d2h")
    return model, training_maxima, t_dev, pre


def train(x, cfg):
    """Training phase (reference rapid.py:72-135) -> (model, training maxima,
    training columns t_ex (v x ell))."""
    x = as_data_matrix(x)
    model, training_maxima, t_dev, _ = _train_device(x, cfg)
    return model, training_maxima, t_dev.t().contiguous().cpu().numpy()


def _degenerate_in_recovery(x, plan, ell, L, k, t_perm_idx, omega_idx, omegas, orders):
    """Raise like the reference: spans of 256 permutations from ell; the first
    failing span reports the flat index into its (count x k) block."""
    p = ell + t_perm_idx
    lo = ell + ((p - ell) // _BLOCK) * _BLOCK
    voxel = (p - lo) * k + omega_idx
    row = x.values[omegas[t_perm_idx, omega_idx]]
    o = orders[t_perm_idx]
    m = row[o[: x.n1]].mean() - row[o[x.n1:]].mean()
    raise DegenerateVoxelError(int(voxel), float(m))


def recover(x, model: SubspaceModel, plan, cfg, _pre: Optional[_RecoverInputs] = None):
    """Recovery phase (reference rapid.py:209-250) -> (MaxNull, counters).
    `_pre`: run_rapid's basis-independent inputs computed during training."""
    torch = _torch()
    x = as_data_matrix(x)
    plan = as_plan(plan)
    cfg = cfg.resolve(x)
    ell, L = model.training_columns, plan.count
    if ell >= L:
        raise UsageError(f"no columns to recover: training columns {ell} >= permutations {L}")
    resolve_threads(cfg.threads)
    v, n1 = x.voxels, x.n1
    k = observed_rows(model.sample_rate, v)
    dev = cuda_device()
    u, u32 = _basis_device(model, dev)
    r = model.basis.rank
    maxima = np.empty(L, dtype=np.float64)
    maxima[:ell] = model.training_maxima
    nrec = L - ell
    if _pre is not None and _pre.key == (int(model.seed), ell, k, L, plan.master_seed):
        xd, od, omd, t, st, rc = _pre.xd, _pre.od, _pre.omd, _pre.t, _pre.st, _pre.rc
    else:
        xd = data_to_device(x, dev, one_shot=True)
        od = device_orders(plan.master_seed, ell, L, x.subjects, dev)
        omd = device_omegas(model.seed, RECOVER_OMEGA, ell, L, v, k, dev)
        t = torch.empty((nrec, k), dtype=torch.float64, device=dev)
        st = nat.Status()
        rc = nat.load().rmx_rapid_stats(nat.ptr(xd), v, x.subjects, n1, nat.ptr(od), nat.ptr(omd),
                                        nrec, k, nat.ptr(t), _stream(dev), ctypes.byref(st))
    if rc == nat.RMX_E_DEGENERATE:
        _degenerate_in_recovery(x, plan, ell, L, k, int(st.perm), int(st.voxel),
                                omd.cpu().numpy(), od.cpu().numpy())
    nat.raise_for(rc, st)
    _mark("recover_inputs")
    # w feeds the completion as fp16 rows (|error| ~2^-12 sum |w_i u_i|), so
    # the second fp64 refinement step is kept only where the first one moved
    # w by more than 1e-4 |w| (settled systems: w within ~1e-8 |w|)
    W, flags, _ = _lsq_tc(u, r, omd, k, t, nrec, settle=_RECOVER_SETTLE)
    _mark("recover_lsq")
    evals = nrec * k
    bad = np.flatnonzero(flags.cpu().numpy() != 0)
    for j in bad:  # rapid.py:173-196: redraw from the same stream, up to 5 times
        i = ell + int(j)
        ok = False
        last_cond = float("inf")
        for attempt in range(1, _RESAMPLE_ATTEMPTS + 1):
            idx = _resample(model.seed, (RECOVER_OMEGA, i), attempt, v, k)
            idx_d = _to_dev(idx[None], dev)
            tj = torch.empty((1, k), dtype=torch.float64, device=dev)
            nat.call("rmx_rapid_stats", nat.ptr(xd), v, x.subjects, n1, nat.ptr(od[j:j + 1]),
                     nat.ptr(idx_d), 1, k, nat.ptr(tj), _stream(dev))
            evals += k
            wj, fj, cj = _lsq_exact(u, r, idx_d, k, tj, 1)
            last_cond = float(cj[0])
            if int(fj[0]) == 0:
                W[j] = wj[0]
                ok = True
                break
        if not ok:
            raise NumericalError(
                f"permutation {i}: restricted basis stayed ill-conditioned "
                f"(last condition number {last_cond:.3e}) after "
                f"{_RESAMPLE_ATTEMPTS} observation resamples")
    m = _complete_max(u32, W.to(torch.float32), ell, model.residual_std, model.max_shift,
                      model.seed, model.two_sided)
    maxima[ell:] = m.cpu().numpy()
    counters = {
        "subsampled_statistic_evaluations": int(evals),
        "recovery_columns": nrec,
        "observed_rows_per_column": k,
        "resampled_evaluations": int(evals - k * nrec),
    }
    return MaxNull(maxima), counters


def run_rapid(x, cfg):
    """Full accelerated run (reference rapid.py:253-275)."""
    x = as_data_matrix(x)
    cfg = cfg.resolve(x)
    plan = cfg.plan_for(x)
    t0 = time.perf_counter()
    _mark("run_rapid_start")
    model, _, _, pre = _train_device(x, cfg, prefetch_recovery=True)
    t1 = time.perf_counter()
    null, rec = recover(x, model, plan, cfg, _pre=pre)
    _mark("recover")
    model.basis.matrix  # the basis's host copy, overlapped with recovery
    _mark("basis_host_copy_join")
    t2 = time.perf_counter()
    v = x.voxels
    counters = {
        "full_statistic_evaluations": v * model.training_columns,
        **rec,
        "statistic_evaluations": v * model.training_columns + rec["subsampled_statistic_evaluations"],
        "training_passes": model.passes,
        "training_converged": model.converged,
        "train_seconds": t1 - t0,
        "recover_seconds": t2 - t1,
        "total_seconds": t2 - t0,
    }
    return null, model, counters
