"""numpy's ``Generator.standard_normal`` over the reference's streams, bit for
bit, on host cores (librmx: csrc/normals.cpp).

The reference draws its basis initialisation as ONE stream of v x r normals
(lrmc.py:85-93, ``stream(seed, BASIS_INIT).standard_normal((v, r))``: 2.1e8
at config 5) and its max-gap shift normals as ell streams of v
(rapid.py:115-121).  numpy's ziggurat consumes one 64-bit word per normal on
its fast path, so a stream is one serial SFC64 chain; the native generator
steps it and applies the ziggurat in compiled code (no Python / ufunc
overhead), and independent streams run on a thread pool.

numpy's ziggurat tables (k, w, f) are taken from numpy itself at first use:
a probing bit generator (a ``bitgen_t`` whose ``next_uint64`` /
``next_double`` we control, wrapped in the "BitGenerator" capsule numpy's
``Generator`` accepts) makes ``standard_normal`` reveal w[i] (one word with
rabs = 1 returns 1 * w[i]), k[i] (bisection on the smallest rabs that leaves
the fast path) and f[i] (wedge tests with a chosen U decide between the
doubles next to exp(-x_i^2 / 2)).  So the tables always match the installed
numpy, exactly.
"""

from __future__ import annotations

import ctypes
import math
import threading

import numpy as np

from . import _native as nat

_TABLES = None
_LOCK = threading.Lock()

_N64 = ctypes.CFUNCTYPE(ctypes.c_uint64, ctypes.c_void_p)
_N32 = ctypes.CFUNCTYPE(ctypes.c_uint32, ctypes.c_void_p)
_ND = ctypes.CFUNCTYPE(ctypes.c_double, ctypes.c_void_p)


class _BitGen(ctypes.Structure):  # numpy/random/bitgen.h bitgen_t
    _fields_ = [("state", ctypes.c_void_p), ("next_uint64", _N64), ("next_uint32", _N32),
                ("next_double", _ND), ("next_raw", _N64)]


class _Probe:
    """A bit generator numpy's Generator accepts, fed from Python."""

    def __init__(self):
        import threading as _t

        self.words = []
        self.u = 0.5
        self.n64 = 0
        self.ndbl = 0

        def n64(_):
            self.n64 += 1
            return self.words.pop(0) if self.words else 0

        def n32(_):
            return 0

        def nd(_):
            self.ndbl += 1
            return self.u

        self._cb = (_N64(n64), _N32(n32), _ND(nd), _N64(n64))
        self._bg = _BitGen(None, *self._cb)
        new = ctypes.pythonapi.PyCapsule_New
        new.restype = ctypes.py_object
        new.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_void_p]
        self.capsule = new(ctypes.addressof(self._bg), b"BitGenerator", None)
        self.lock = _t.Lock()
        self.gen = np.random.Generator(self)

    def draw(self, word: int, u: float = 0.5) -> tuple[float, bool]:
        """standard_normal() fed `word` first and `u` by next_double; (value,
        left the fast path).  A rejected wedge test draws a fresh word, which
        the empty queue answers with 0 (a fast-path 0.0)."""
        self.words = [word]
        self.u = u
        self.n64 = self.ndbl = 0
        x = float(self.gen.standard_normal())
        return x, (self.n64 > 1 or self.ndbl > 0)


def _wedge_accepts(f_prev: float, f_i: float, u: float, x: float) -> bool:
    # distributions.c: (f[idx-1] - f[idx]) * U + f[idx] < exp(-0.5 * x * x)
    return (f_prev - f_i) * u + f_i < math.exp(-0.5 * x * x)


def _probe_f(p: _Probe, i: int, k_i: int, w_i: float, f_prev: float) -> float:
    """f[i] exactly: candidates around exp(-x_i^2 / 2) are told apart by wedge
    tests whose U sits between the candidates' decision boundaries."""
    xi = w_i * 2.0 ** 52
    c0 = math.exp(-0.5 * xi * xi)
    cands = [c0]
    for _ in range(4):
        cands.insert(0, np.nextafter(cands[0], -np.inf))
        cands.append(np.nextafter(cands[-1], np.inf))
    # wedge points near the strip's outer edge x_i: there E = exp(-x^2/2) is
    # just above f[i], the separating U is small, and the candidates' left
    # sides differ by a whole ulp (near U = 1/2 the two roundings merge them)
    rabs_list = [(1 << 52) - (1 << j) for j in range(8, 46, 2)]
    lo, hi = 0, len(cands) - 1  # the answer is in cands[lo..hi]
    while lo < hi:
        mid = (lo + hi) // 2  # split {.. c_mid} | {c_mid+1 ..}
        a, b = float(cands[mid]), float(cands[mid + 1])
        u = rabs = None
        for rb in rabs_list:
            if rb < int(k_i):
                continue
            x = rb * w_i
            E = math.exp(-0.5 * x * x)
            ua = (E - a) / (f_prev - a)
            ub = (E - b) / (f_prev - b)
            if not (0.0 <= ub < ua < 1.0):
                continue
            for t in np.linspace(ub, ua, 17)[1:-1]:  # c_a accepts, c_b rejects
                t = float(t)
                if _wedge_accepts(f_prev, a, t, x) and not _wedge_accepts(f_prev, b, t, x):
                    u, rabs = t, rb
                    break
            if u is not None:
                break
        if u is None:
            raise RuntimeError(f"cannot separate ziggurat f[{i}] candidates")
        val, slow = p.draw((rabs << 9) | i, u)
        accepted = slow and val != 0.0 and p.n64 == 1
        # the true f accepts like c_a (<= mid) or rejects like c_b (> mid)
        if accepted:
            hi = mid
        else:
            lo = mid + 1
    return float(cands[lo])


def _probe_tables():
    p = _Probe()
    w = np.empty(256)
    k = np.zeros(256, dtype=np.uint64)
    for idx in range(256):
        w[idx] = abs(p.draw((1 << 9) | idx)[0])
        lo, hi = 0, 1 << 52  # fast path <=> rabs < k[idx]; find the smallest slow rabs
        while lo < hi:
            mid = (lo + hi) // 2
            if p.draw((mid << 9) | idx)[1]:
                hi = mid
            else:
                lo = mid + 1
        k[idx] = lo
    f = np.empty(256)
    f[0] = 1.0  # the base strip's top (exp(0)); idx 0 takes the tail, not the wedge
    for i in range(1, 256):
        f[i] = _probe_f(p, i, int(k[i]), float(w[i]), float(f[i - 1]))
    return k, w, f


def tables():
    """(k uint64[256], w float64[256], f float64[256]) of the installed numpy."""
    global _TABLES
    with _LOCK:
        if _TABLES is None:
            k, w, f = _probe_tables()
            lib = nat.load()
            lib.rmx_normal_tables_set(k.ctypes.data, w.ctypes.data, f.ctypes.data)
            _TABLES = (k, w, f)
        return _TABLES


def standard_normal(seed: int, path: tuple, count: int, out=None) -> np.ndarray:
    """``stream(seed, *path).standard_normal(count)`` (float64), natively."""
    tables()
    if out is None:
        out = np.empty(int(count), dtype=np.float64)
    p = (ctypes.c_uint32 * max(1, len(path)))(*[int(x) for x in path])
    nat.call("rmx_standard_normal", int(seed) & ((1 << 64) - 1), p, len(path), int(count),
             out.ctypes.data)
    return out


def standard_normal_rows(seed: int, domain: int, lo: int, hi: int, count: int,
                         dtype=np.float32, out=None, threads: int = 0) -> np.ndarray:
    """Row i - lo = ``stream(seed, domain, i).standard_normal(count)`` for i in
    [lo, hi), as `dtype` (float32: numpy's float64 values cast), on threads."""
    tables()
    dtype = np.dtype(dtype)
    if out is None:
        out = np.empty((hi - lo, int(count)), dtype=dtype)
    p32 = out.ctypes.data if dtype == np.float32 else None
    p64 = out.ctypes.data if dtype == np.float64 else None
    nat.call("rmx_standard_normal_rows", int(seed) & ((1 << 64) - 1), int(domain), int(lo),
             int(hi), int(count), p32, p64, int(threads))
    return out


class NormalStream:
    """``stream(seed, *path)``'s standard normals drawn piece by piece (the
    ctypes call releases the GIL: a host thread can draw while Python issues
    GPU work)."""

    def __init__(self, seed: int, path: tuple):
        tables()
        self._h = ctypes.c_void_p()
        p = (ctypes.c_uint32 * max(1, len(path)))(*[int(x) for x in path])
        nat.call("rmx_normal_stream_open", int(seed) & ((1 << 64) - 1), p, len(path),
                 ctypes.byref(self._h))

    def fill(self, out: np.ndarray) -> np.ndarray:
        assert out.dtype == np.float64 and out.flags["C_CONTIGUOUS"]
        rc = nat.load().rmx_normal_stream_fill(self._h, int(out.size), out.ctypes.data)
        if rc:
            raise RuntimeError(f"rmx_normal_stream_fill failed ({rc})")
        return out

    def fill_device(self, out, pinned: np.ndarray, stream) -> None:
        """Draw out.numel() normals straight into the contiguous fp64 CUDA
        tensor `out` through the page-locked ring `pinned` (one native call,
        the GIL released; returns when the last copy has landed)."""
        st = nat.Status()
        rc = nat.load().rmx_normal_stream_fill_device(
            self._h, int(out.numel()), out.data_ptr(), pinned.ctypes.data, int(pinned.size),
            nat.stream_handle(stream), ctypes.byref(st))
        nat.raise_for(rc, st)

    def close(self) -> None:
        if self._h:
            nat.load().rmx_normal_stream_close(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


__all__ = ["tables", "standard_normal", "standard_normal_rows", "NormalStream"]
