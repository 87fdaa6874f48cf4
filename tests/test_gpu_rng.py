"""The reference's random streams generated on the GPU (rng_kernels.cu)
against numpy itself: PermutationPlan shuffles and Omega draws must be
bit-identical (the labels feed the bit-exact statistic path)."""
import os

import numpy as np
import pytest

from paper_1703_01506_b200.rng import RECOVER_OMEGA, TRAIN_OMEGA, omega_draw, shuffle_order, stream

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.mark.parametrize("seed,lo,count,n", [(1703015061, 0, 300, 20), (2 ** 63 + 11, 5, 64, 400),
                                             (0, 1, 50, 3), (1703015064, 99_000, 40, 400),
                                             (7, 0, 20, 4097)])
def test_device_shuffles_match_numpy(seed, lo, count, n):
    import torch

    from paper_1703_01506_b200.labels import device_orders

    got = device_orders(seed, lo, lo + count, n, torch.device("cuda", 0)).cpu().numpy()
    want = np.stack([shuffle_order(seed, lo + i, n) for i in range(count)]).astype(np.int16)
    assert np.array_equal(got, want)


def test_device_shuffles_match_golden_file():
    import torch

    from paper_1703_01506_b200.labels import device_orders

    d = np.load(os.path.join(GOLD, "shuffles.npz"))  # s{seed}_n{n}: plan rows 0..63
    checked = 0
    for key in d.files:
        if not (key.startswith("s") and "_n" in key):
            continue
        seed, n = (int(t) for t in key[1:].split("_n"))
        ref = d[key]
        got = device_orders(seed, 0, ref.shape[0], n, torch.device("cuda", 0)).cpu().numpy()
        assert np.array_equal(got, ref.astype(np.int16)), key
        checked += 1
    assert checked >= 10


@pytest.mark.parametrize("v,k,extra", [(524288, 1836, None), (262144, 1311, 7), (5000, 30, None),
                                       (300, 60, 0), (9000, 4000, None)])
def test_device_omegas_match_numpy(v, k, extra):
    import torch

    from paper_1703_01506_b200.rapid_engine import device_omegas

    seed, lo, count = 1703015065, 400, 37
    dom = TRAIN_OMEGA if extra is not None else RECOVER_OMEGA
    got = device_omegas(seed, dom, lo, lo + count, v, k, torch.device("cuda", 0),
                        extra=extra).cpu().numpy()
    path = (lambda i: (dom, lo + i, extra)) if extra is not None else (lambda i: (dom, lo + i))
    want = np.stack([omega_draw(stream(seed, *path(i)), v, k) for i in range(count)])
    assert np.array_equal(got, want.astype(np.int32))


def test_tail_shuffle_branch_falls_back_to_host():
    import torch

    from paper_1703_01506_b200.rapid_engine import device_omegas

    got = device_omegas(5, RECOVER_OMEGA, 0, 3, 20000, 900, torch.device("cuda", 0)).cpu().numpy()
    want = np.stack([omega_draw(stream(5, RECOVER_OMEGA, i), 20000, 900) for i in range(3)])
    assert np.array_equal(got, want.astype(np.int32))


def test_device_omegas_match_reference_golden_draws():
    """Omega draws the reference itself produced (tests/golden/make_golden.py)."""
    import torch

    from paper_1703_01506_b200.rapid_engine import device_omegas

    d = np.load(os.path.join(GOLD, "shuffles.npz"))
    dev = torch.device("cuda", 0)
    checked = 0
    for key in d.files:
        if not key.startswith("omega_"):
            continue
        kind, seed, v, k = key.split("_")[1], *(int(t) for t in key.split("_")[2:])
        ref = d[key]
        if kind == "recover":
            got = device_omegas(seed, RECOVER_OMEGA, 0, ref.shape[0], v, k, dev)
        else:
            got = device_omegas(seed, TRAIN_OMEGA, 0, ref.shape[0], v, k, dev, extra=1)
        assert np.array_equal(got.cpu().numpy(), ref), key
        checked += 1
    assert checked == 6
