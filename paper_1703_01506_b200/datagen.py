"""Seeded synthetic inputs for BASELINE.json's five configurations.

The reference's own generator (simgen.py:54-60) makes i.i.d. data with a
scattered group-2 signal and cannot produce BASELINE.json's inputs (SURVEY
F8), so this module builds them: per subject an i.i.d. N(0,1) volume on the
config's 3-D grid, isotropic Gaussian smoothing, then a constant effect added
to a centred cube in the group-1 subjects; voxels are the C-order flattening
of the grid, values are rounded to float32 (the GPU and the reference see the
same float64-exact numbers).  No public dataset is involved; the paper's real
data (ADNI2) is not available and is not imitated.

Two backends with the same distribution:
  numpy  -- noise from stream(seed, SIM_NOISE, subject) (SFC64), smoothing by
            scipy.ndimage.gaussian_filter(mode='reflect', truncate=4);
            deterministic across machines; used by tests and golden files.
  torch  -- noise from a seeded torch generator on the GPU, separable
            Gaussian convolution; used by bench.py to build 0.8 GB inputs in
            milliseconds.  Values differ from the numpy backend, statistics
            do not.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

from .rng import SIM_NOISE, stream


@dataclass(frozen=True)
class Config:
    name: str
    grid: tuple
    n1: int
    n2: int
    sigma: float
    effect: float
    cube: tuple
    permutations: int
    seed: int             # data seed
    plan_seed: int        # permutation plan seed
    two_sided: bool
    engine: str = "naive"
    sample_rate: Optional[float] = None
    rank: Optional[int] = None
    training_columns: Optional[int] = None

    @property
    def voxels(self) -> int:
        return int(np.prod(self.grid))

    @property
    def subjects(self) -> int:
        return self.n1 + self.n2


CONFIGS = {
    "c1": Config("c1", (32, 32, 16), 10, 10, 1.0, 0.8, (8, 8, 4), 1_000, 1703015061, 1703015061,
                 True),
    "c2": Config("c2", (64, 64, 64), 50, 50, 2.0, 0.5, (16, 16, 16), 10_000, 1703015062,
                 1703015062, False),
    "c3": Config("c3", (64, 64, 64), 50, 50, 2.0, 0.5, (16, 16, 16), 10_000, 1703015062,
                 1703015062, False, engine="rapid", sample_rate=0.005, rank=100,
                 training_columns=100),
    "c4": Config("c4", (128, 64, 64), 200, 200, 2.0, 0.3, (24, 24, 24), 100_000, 1703015064,
                 1703015064, False),
    "c5": Config("c5", (128, 64, 64), 120, 280, 2.0, 0.3, (24, 24, 24), 100_000, 1703015064,
                 1703015065, False, engine="rapid", sample_rate=0.0035, rank=400,
                 training_columns=400),
}


def scaled(cfg: Config, grid: tuple, permutations: int) -> Config:
    """Same statistical design on a smaller grid / plan (parity tests)."""
    cube = tuple(max(1, (c * g) // og) for c, g, og in zip(cfg.cube, grid, cfg.grid))
    return Config(cfg.name + "-small", tuple(grid), cfg.n1, cfg.n2, cfg.sigma, cfg.effect, cube,
                  permutations, cfg.seed, cfg.plan_seed, cfg.two_sided, cfg.engine,
                  cfg.sample_rate, cfg.rank, cfg.training_columns)


def _cube_slices(cfg: Config):
    return tuple(slice((g - c) // 2, (g - c) // 2 + c) for g, c in zip(cfg.grid, cfg.cube))


def _subject_numpy(args):
    cfg, j = args
    from scipy.ndimage import gaussian_filter

    vol = stream(cfg.seed, SIM_NOISE, j).standard_normal(cfg.grid)
    vol = gaussian_filter(vol, sigma=cfg.sigma, mode="reflect", truncate=4.0)
    if j < cfg.n1:
        vol[_cube_slices(cfg)] += cfg.effect
    return vol.astype(np.float32).ravel()


def make_data_numpy(cfg: Config, workers: Optional[int] = None) -> np.ndarray:
    """(v, n) float64 matrix (float32-exact values), deterministic."""
    jobs = [(cfg, j) for j in range(cfg.subjects)]
    workers = workers or min(os.cpu_count() or 1, 16)
    if workers > 1 and cfg.voxels * cfg.subjects > 4_000_000:
        import multiprocessing as mp
        from concurrent.futures import ProcessPoolExecutor

        # forkserver: the workers fork from a clean server process, never from
        # this one (which may hold CUDA contexts and host threads: forking it
        # can deadlock the child)
        with ProcessPoolExecutor(workers, mp_context=mp.get_context("forkserver")) as pool:
            cols = list(pool.map(_subject_numpy, jobs, chunksize=4))
    else:
        cols = [_subject_numpy(a) for a in jobs]
    return np.stack(cols, axis=1).astype(np.float64)


def _gauss_kernel(sigma: float):
    r = int(4.0 * sigma + 0.5)
    xs = np.arange(-r, r + 1, dtype=np.float64)
    w = np.exp(-0.5 * (xs / sigma) ** 2)
    return w / w.sum(), r


def make_data_torch(cfg: Config, device, seed_offset: int = 0):
    """(v, n) float64 CUDA tensor (float32-exact values), same design."""
    import torch
    import torch.nn.functional as F

    g = torch.Generator(device=device)
    g.manual_seed(cfg.seed + seed_offset)
    n = cfg.subjects
    vol = torch.randn((n, 1) + tuple(cfg.grid), generator=g, device=device, dtype=torch.float32)
    w, r = _gauss_kernel(cfg.sigma)
    wt = torch.tensor(w, dtype=torch.float32, device=device)
    for axis in range(3):
        shape = [1, 1, 1, 1, 1]
        shape[2 + axis] = w.size
        pad = [0, 0, 0, 0, 0, 0]
        pad[2 * (2 - axis)] = r
        pad[2 * (2 - axis) + 1] = r
        vol = F.conv3d(F.pad(vol, pad, mode="replicate"), wt.view(shape))
    cs = _cube_slices(cfg)
    vol[: cfg.n1, 0, cs[0], cs[1], cs[2]] += cfg.effect
    return vol.reshape(n, -1).t().contiguous().to(torch.float64)


def grid_effect_mask(cfg: Config) -> np.ndarray:
    m = np.zeros(cfg.grid, dtype=bool)
    m[_cube_slices(cfg)] = True
    return m.ravel()


__all__ = ["Config", "CONFIGS", "scaled", "make_data_numpy", "make_data_torch",
           "grid_effect_mask", "math"]
