"""CPU oracle for the max-null hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import this module.  It is the checker, never the
thing measured or shipped: the product path in ``paper_1703_01506_b200``
never imports it and fails loudly without its CUDA library.

Two layers:
  * ``rmx_oracle.c`` (built by ``oracle/Makefile``) restates the NaivePT
    statistic path bit-exactly: numpy pairwise summation, ``_welch_rows``
    (reference teststat.py:28-50), ``group_blocks`` (model.py:65-69),
    ``column_max`` (teststat.py:88-90) and the ``_max_block`` loop
    (naive.py:49-57).
  * numpy restatements of the RapidPT recovery algebra (rapid.py:138-206,
    lrmc.py:127-157), used to check the GPU recovery kernels.

Pinned against vectors produced by the reference itself
(tests/golden/make_golden.py -> tests/golden/*.npz).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "librmx_oracle.so")
_lib = None


def build() -> str:
    """Compile the C restatement (gcc); returns the .so path."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(
            os.path.join(_HERE, "rmx_oracle.c")
        ):
            build()
        L = ctypes.CDLL(_SO)
        dp = ctypes.POINTER(ctypes.c_double)
        ip = ctypes.POINTER(ctypes.c_int64)
        L.rmx_oracle_welch.argtypes = [dp, ip, ctypes.c_int, ctypes.c_int, dp, dp]
        L.rmx_oracle_welch.restype = ctypes.c_int
        L.rmx_oracle_naive.argtypes = [
            dp, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ip, ctypes.c_int64,
            ctypes.c_int, dp, ip, dp, ip, ip, dp,
        ]
        L.rmx_oracle_naive.restype = ctypes.c_int
        L.rmx_oracle_np_sum.argtypes = [dp, ctypes.c_int64]
        L.rmx_oracle_np_sum.restype = ctypes.c_double
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _ip(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


class OracleDegenerate(Exception):
    def __init__(self, perm, voxel, mean_diff):
        self.perm, self.voxel, self.mean_diff = perm, voxel, mean_diff
        super().__init__(f"perm {perm} voxel {voxel} mean_diff {mean_diff}")


def np_sum(a: np.ndarray) -> float:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return float(lib().rmx_oracle_np_sum(_dp(a), a.size))


def welch(row: np.ndarray, order: np.ndarray, n1: int) -> tuple[float, float, bool]:
    """(t, mean_diff, degenerate) for one voxel row under `order`."""
    row = np.ascontiguousarray(row, dtype=np.float64)
    order = np.ascontiguousarray(order, dtype=np.int64)
    t = np.zeros(1)
    num = np.zeros(1)
    deg = lib().rmx_oracle_welch(_dp(row), _ip(order), n1, row.size - n1, _dp(t), _dp(num))
    return float(t[0]), float(num[0]), bool(deg)


def naive_maxnull(x: np.ndarray, n1: int, orders: np.ndarray, two_sided: bool,
                  materialize: bool = False, threads: int = 1):
    """(maxima[L], argmax[L], T[v,L] or None).  Threads split permutations
    (the C loop releases the GIL through ctypes)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    orders = np.ascontiguousarray(orders, dtype=np.int64)
    v, n = x.shape
    L = orders.shape[0]
    maxima = np.empty(L)
    argmax = np.empty(L, dtype=np.int64)
    T = np.empty((v, L)) if materialize else None
    if materialize and threads != 1:
        threads = 1                         # T column slices are strided
    bounds = np.linspace(0, L, max(1, threads) + 1).astype(np.int64)

    def work(lo, hi):
        if hi <= lo:
            return None
        dperm = np.zeros(1, dtype=np.int64)
        dvox = np.zeros(1, dtype=np.int64)
        dnum = np.zeros(1)
        sub = orders[lo:hi]
        mx = np.empty(hi - lo)
        am = np.empty(hi - lo, dtype=np.int64)
        rc = lib().rmx_oracle_naive(
            _dp(x), v, n, n1, _ip(sub), hi - lo, int(two_sided), _dp(mx), _ip(am),
            _dp(T) if T is not None else None, _ip(dperm), _ip(dvox), _dp(dnum),
        )
        if rc:
            return (int(dperm[0]) + lo, int(dvox[0]), float(dnum[0]))
        maxima[lo:hi] = mx
        argmax[lo:hi] = am
        return None

    if threads <= 1:
        errs = [work(0, L)]
    else:
        with ThreadPoolExecutor(threads) as pool:
            errs = list(pool.map(lambda i: work(bounds[i], bounds[i + 1]), range(threads)))
    errs = [e for e in errs if e is not None]
    if errs:
        raise OracleDegenerate(*min(errs))
    return maxima, argmax, T


# --------------------------------------------------------------------------
# RapidPT recovery algebra (numpy restatement; reference rapid.py:138-206)
# --------------------------------------------------------------------------

def solve_block(u_stack: np.ndarray, values: np.ndarray):
    """lrmc.py:127-149: normal equations with exact condition numbers."""
    gram = np.matmul(u_stack.transpose(0, 2, 1), u_stack)
    rhs = np.matmul(u_stack.transpose(0, 2, 1), values[..., None])
    lam = np.linalg.eigvalsh(gram)
    lo, hi = lam[:, 0], lam[:, -1]
    with np.errstate(divide="ignore", invalid="ignore"):
        conds = np.sqrt(np.where(lo > 0, hi / lo, np.inf))
    bad = ~np.isfinite(conds) | (conds > 1e12)
    g = gram.copy()
    g[bad] = np.eye(gram.shape[-1])
    return np.linalg.solve(g, rhs)[..., 0], conds


def welch_rows(block1: np.ndarray, block2: np.ndarray) -> np.ndarray:
    """Row-wise statistic via the bit-exact C restatement (teststat.py:28-50)."""
    n1 = block1.shape[1]
    rows = np.ascontiguousarray(np.concatenate([block1, block2], axis=1))
    order = np.arange(rows.shape[1], dtype=np.int64)
    return np.array([welch(r, order, n1)[0] for r in rows])


def recover_noise_free(x: np.ndarray, n1: int, u: np.ndarray, orders: np.ndarray,
                       omegas: np.ndarray, two_sided: bool, mu: float = 0.0):
    """Recovered maxima with sigma = 0 (rapid.py:156-205 without the residual
    draw): per permutation, Omega-row statistics -> LS fit -> U w -> max + mu.
    Returns (maxima, coefficients)."""
    L, k = omegas.shape
    stats = np.empty((L, k))
    for i in range(L):
        rows = x[omegas[i]]
        o = orders[i]
        stats[i] = welch_rows(rows[:, o[:n1]], rows[:, o[n1:]])
    w, _ = solve_block(u[omegas], stats)
    cols = w @ u.T
    vals = np.abs(cols).max(axis=1) if two_sided else cols.max(axis=1)
    return vals + mu, w, stats


# --------------------------------------------------------------------------
# GROUSE training (numpy restatement; reference lrmc.py:85-104,160-193,208-268)
# --------------------------------------------------------------------------

def _stream(seed: int, *path: int) -> np.random.Generator:
    """streams.py:31-38: SeedSequence(seed mod 2^64, spawn_key=path) -> SFC64."""
    key = np.random.SeedSequence(entropy=int(seed) & ((1 << 64) - 1),
                                 spawn_key=tuple(int(p) for p in path))
    return np.random.Generator(np.random.SFC64(key))


def init_basis(v: int, r: int, seed: int) -> np.ndarray:
    """lrmc.py:85-93: Q of the QR of a BASIS_INIT (domain 5) Gaussian draw."""
    return np.ascontiguousarray(np.linalg.qr(_stream(seed, 5).standard_normal((v, r)))[0])


def grouse(t_ex: np.ndarray, k: int, rank: int, seed: int, max_passes: int = 50,
           tolerance: float = 1e-3, force_halt=(), basis0=None):
    """train_basis (lrmc.py:208-268) with track_update (lrmc.py:160-193) and
    _gram_fit (lrmc.py:96-104) restated in numpy fp64.

    force_halt: global update indices whose FIRST observation draw is treated
    as ill-conditioned (the reference then redraws from the same generator,
    lrmc.py:240-250) -- the test hook matching RMX_GROUSE_TEST_HALT.
    Returns (U, passes, pass_residuals, final_omegas, converged)."""
    v, ell = t_ex.shape
    u = init_basis(v, rank, seed) if basis0 is None else np.array(basis0, dtype=np.float64)
    tau = ell * max_passes / 2.0
    t = 0
    res = []
    omegas = []
    passes, converged = 0, False
    for p in range(max_passes):
        rel_sum = 0.0
        omegas = []
        for i in range(ell):
            g = _stream(seed, 2, i, p)
            step = 1.0 / (1.0 + t / tau)
            for attempt in range(5):
                idx = np.sort(g.choice(v, size=k, replace=False))
                if attempt == 0 and t in force_halt:
                    continue
                vals = t_ex[idx, i]
                uo = u[idx]
                gram = uo.T @ uo
                lam = np.linalg.eigvalsh(gram)
                cond = np.inf if lam[0] <= 0.0 else float(np.sqrt(lam[-1] / lam[0]))
                if cond > 1e12:
                    continue
                w = np.linalg.solve(gram, uo.T @ vals)
                break
            else:
                raise ArithmeticError("restricted basis stayed ill-conditioned")
            resid = vals - uo @ w
            rn = float(np.linalg.norm(resid))
            if step != 0.0 and rn != 0.0:
                pred = u @ w
                pn = float(np.linalg.norm(pred))
                wn = float(np.linalg.norm(w))
                if pn != 0.0 and wn != 0.0 and rn > 1e-14 * max(1.0, pn):
                    theta = step * np.arctan(rn / pn)
                    d = (np.cos(theta) - 1.0) / pn * pred
                    d[idx] += np.sin(theta) / rn * resid
                    u += np.outer(d, w / wn)
            t += 1
            nb = float(np.linalg.norm(vals))
            rel_sum += rn / nb if nb > 0 else 0.0
            omegas.append(idx)
            if t % 64 == 0 and np.abs(u.T @ u - np.eye(rank)).max() > 1e-8:
                u = np.ascontiguousarray(np.linalg.qr(u)[0])
        rel = rel_sum / ell
        res.append(rel)
        passes = p + 1
        if rel < tolerance:
            converged = True
            break
    if np.abs(u.T @ u - np.eye(rank)).max() > 1e-8:
        u = np.ascontiguousarray(np.linalg.qr(u)[0])
    return u, passes, res, omegas, converged


def principal_cosines(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Cosines of the principal angles between span(a) and span(b) (columns)."""
    qa = np.linalg.qr(a)[0]
    qb = np.linalg.qr(b)[0]
    return np.clip(np.linalg.svd(qa.T @ qb, compute_uv=False), 0.0, 1.0)
