"""Seeded per-purpose random streams (host side).

Same contract as the reference (streams.py:31-38): the generator for
``(seed, *path)`` is ``Generator(SFC64(SeedSequence(seed mod 2**64,
spawn_key=path)))``, so permutations and observation sets generated here are
bit-identical to the reference's.  Domain ids are fixed by the reference
(streams.py:19-26) and must never be renumbered.

Only *inputs* come from here (labels, Omega sets, basis init).  The RapidPT
residual noise is drawn on the device from a counter-based Philox stream
instead ("RapidPT noise").
"""

from __future__ import annotations

import numpy as np

SHUFFLE = 1
TRAIN_OMEGA = 2
RECOVER_OMEGA = 3
RESIDUAL = 4
BASIS_INIT = 5
SIM_NOISE = 6
SIM_SIGNAL = 7
SHIFT_GAP = 8

_U64 = (1 << 64) - 1


def stream(seed: int, *path: int) -> np.random.Generator:
    seq = np.random.SeedSequence(entropy=int(seed) & _U64,
                                 spawn_key=tuple(int(p) for p in path))
    return np.random.Generator(np.random.SFC64(seq))


def shuffle_order(seed: int, index: int, subjects: int) -> np.ndarray:
    """Permutation ``index`` of a plan: identity at 0, else an SFC64 shuffle."""
    if index == 0:
        return np.arange(subjects)
    return stream(seed, SHUFFLE, index).permutation(subjects)


def omega_draw(rng: np.random.Generator, v: int, k: int) -> np.ndarray:
    """Sorted k-subset of range(v) -- the reference's Omega draw
    (rapid.py:160, lrmc.py:241): ``sort(rng.choice(v, k, replace=False))``."""
    return np.sort(rng.choice(v, size=k, replace=False))
