"""Host-side logic of the drop-in boundary (no GPU): domain types, RNG
streams, label generation, RunConfig defaults and the reference's error
messages, max-null queries."""
import os

import numpy as np
import pytest

import paper_1703_01506_b200 as rmx
from paper_1703_01506_b200.domain import observed_rows
from paper_1703_01506_b200.labels import generate_orders, plan_orders
from paper_1703_01506_b200.rng import RECOVER_OMEGA, TRAIN_OMEGA, omega_draw, stream

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_shuffles_bit_identical_to_reference_plan():
    g = np.load(os.path.join(GOLD, "shuffles.npz"))
    for key in g.files:
        if not key.startswith("s"):
            continue
        seed, n = key[1:].split("_n")
        got = generate_orders(int(seed), 0, 64, int(n))
        assert np.array_equal(got, g[key]), key
        plan = rmx.PermutationPlan(int(seed), 64, int(n))
        assert np.array_equal(plan.shuffle(5), g[key][5])


def test_omega_draws_bit_identical_to_reference():
    g = np.load(os.path.join(GOLD, "shuffles.npz"))
    for key in g.files:
        if not key.startswith("omega_"):
            continue
        kind, _, seed, v, k = key.split("_")
        seed, v, k = int(seed), int(v), int(k)
        for i, row in enumerate(g[key]):
            rng = stream(seed, RECOVER_OMEGA, i) if kind == "omega" and "recover" in key \
                else stream(seed, TRAIN_OMEGA, i, 1)
            assert np.array_equal(omega_draw(rng, v, k), row), key


def test_plan_index_zero_is_identity_and_regenerates():
    plan = rmx.PermutationPlan(99, 10, 6)
    assert np.array_equal(plan.shuffle(0), np.arange(6))
    assert np.array_equal(rmx.PermutationPlan(7, 100, 12).shuffle(33),
                          rmx.PermutationPlan(7, 500, 12).shuffle(33))
    with pytest.raises(rmx.UsageError):
        plan.shuffle(10)


def test_parallel_label_generation_matches_serial():
    a = generate_orders(1703015064, 0, 6000, 400, workers=4)
    b = generate_orders(1703015064, 0, 6000, 400, workers=1)
    assert np.array_equal(a, b)
    plan = rmx.PermutationPlan(1703015064, 6000, 400)
    assert np.array_equal(plan_orders(plan, 100, 300), a[100:300])


def test_data_matrix_validation_messages():
    with pytest.raises(rmx.UsageError, match="at least two subjects"):
        rmx.DataMatrix(np.zeros((3, 3)), 1, 2)
    with pytest.raises(rmx.UsageError, match="do not match"):
        rmx.DataMatrix(np.zeros((3, 5)), 2, 2)
    bad = np.zeros((3, 4))
    bad[1, 2] = np.nan
    with pytest.raises(rmx.UsageError, match="voxel 1, subject 2"):
        rmx.DataMatrix(bad, 2, 2)
    x = rmx.DataMatrix(np.arange(12.0).reshape(3, 4), 2, 2)
    assert not x.values.flags.writeable
    assert x.float32_values is None


def test_data_matrix_keeps_float32_source():
    """float32 input: values is the exact float64 upcast; the float32 copy is
    private (caller mutation does not leak) and read-only."""
    src = np.random.default_rng(0).standard_normal((5, 4)).astype(np.float32)
    x = rmx.DataMatrix(src, 2, 2)
    assert x.values.dtype == np.float64 and x.float32_values.dtype == np.float32
    assert np.array_equal(x.float32_values.astype(np.float64), x.values)
    src[0, 0] = 99.0
    assert x.float32_values[0, 0] != 99.0 and x.values[0, 0] != 99.0
    assert not x.float32_values.flags.writeable


def test_runconfig_resolve_defaults_and_errors():
    x = rmx.DataMatrix(np.random.default_rng(1).standard_normal((500, 10)), 5, 5)
    cfg = rmx.RunConfig(permutations=100, seed=0, engine="rapid").resolve(x)
    assert cfg.training_columns == 10 and cfg.rank == 10
    assert cfg.sample_rate == pytest.approx(2 * 10 * np.log(500) / 500)
    x = rmx.DataMatrix(np.random.default_rng(1).standard_normal((100, 6)), 3, 3)
    with pytest.raises(rmx.UsageError, match="rank"):
        rmx.RunConfig(permutations=50, seed=0, engine="rapid", rank=7).resolve(x)
    with pytest.raises(rmx.UsageError, match="identify rank"):
        rmx.RunConfig(permutations=50, seed=0, engine="rapid", training_columns=4,
                      rank=6).resolve(x)
    with pytest.raises(rmx.UsageError, match="exceed permutation count"):
        rmx.RunConfig(permutations=5, seed=0, engine="rapid", training_columns=6).resolve(x)
    with pytest.raises(rmx.UsageError, match="underdetermined"):
        rmx.RunConfig(permutations=50, seed=0, engine="rapid", sample_rate=0.01,
                      rank=4).resolve(x)
    assert observed_rows(0.005, 262144) == 1311 and observed_rows(0.0035, 524288) == 1836


def test_maxnull_and_queries():
    null = rmx.MaxNull(np.array([1.0, 2.0, 3.0, 4.0]))
    assert rmx.pvalue(null, 3.5) == 0.25 and rmx.pvalue(null, 10.0) == 0.25
    assert rmx.pvalue(rmx.MaxNull(np.array([1.0, 2.0, 2.0, 4.0])), 2.0) == 0.75
    big = rmx.MaxNull(np.arange(1.0, 101.0))
    assert rmx.threshold_at(big, 0.05) == 96.0 and rmx.threshold_at(big, 0.049) == 97.0
    with pytest.raises(rmx.UsageError, match="resolution"):
        rmx.threshold_at(big, 0.009)
    assert np.array_equal(rmx.reject_set(np.array([1.0, 5.0, 2.0, 5.0]), 4.0), [1, 3])
    with pytest.raises(rmx.UsageError):
        rmx.MaxNull(np.array([1.0, np.inf]))


def test_engine_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    x = rmx.DataMatrix(np.random.default_rng(0).standard_normal((10, 6)), 3, 3)
    with pytest.raises(rmx.EngineUnavailableError):
        rmx.run_naive(x, rmx.PermutationPlan(1, 5, 6))


def test_memory_cap_message_names_required_bytes():
    x = rmx.DataMatrix(np.random.default_rng(6).standard_normal((100, 6)), 3, 3)
    with pytest.raises(rmx.UsageError, match=str(100 * 100 * 8)):
        rmx.run_naive(x, rmx.PermutationPlan(1, 100, 6), materialize=True, mem_cap_bytes=1000)


def test_accepts_reference_objects_duck_typed():
    from paper_1703_01506_b200.domain import as_data_matrix, as_plan

    class RefDM:
        values = np.ones((4, 4))
        n1 = 2
        n2 = 2

    class RefPlan:
        master_seed, count, subjects = 3, 7, 4

    assert as_data_matrix(RefDM()).voxels == 4
    assert as_plan(RefPlan()).count == 7


def test_inflight_prune_releases_sources_without_self_deadlock():
    """hostmem._prune_inflight drops the last reference to a copied source
    array; that array's weakref callback (cudaHostUnregister bookkeeping)
    takes hostmem's lock again.  It must not deadlock (it did with a plain
    Lock: the C5 RapidPT test hung in data_to_device)."""
    import threading
    import weakref

    from paper_1703_01506_b200 import hostmem

    class Done:
        def query(self):
            return True

    fired = []

    def cb(_ref):
        with hostmem._LOCK:
            fired.append(1)

    a = np.ones(8)
    ref = weakref.ref(a, cb)
    hostmem._INFLIGHT.append((a, Done()))
    del a
    th = threading.Thread(target=hostmem._prune_inflight, daemon=True)
    th.start()
    th.join(timeout=10)
    assert not th.is_alive() and fired == [1] and ref() is None
