"""NaivePT parity on the GPU: librmx (through the C ABI) vs the CPU oracle.

The oracle is the bit-exact C restatement of the reference statistic path
(oracle/rmx_oracle.c, pinned to the reference by tests/test_oracle_golden.py).
The bar: maxima bit-identical, argmax identical (lowest index on exact ties).
"""
import numpy as np
import pytest

import paper_1703_01506_b200 as rmx
from paper_1703_01506_b200.labels import plan_orders

pytestmark = pytest.mark.gpu


def _data(v, n1, n2, seed, scale=1.0):
    g = np.random.default_rng(seed)
    vals = (g.standard_normal((v, n1 + n2)) * scale).astype(np.float32).astype(np.float64)
    return rmx.DataMatrix(vals, n1, n2)


CASES = [
    # v, n1, n2, L, two_sided, seed
    (20, 2, 2, 50, False, 42),
    (1, 3, 3, 30, False, 1),
    (300, 10, 10, 200, True, 3),
    (1000, 10, 10, 300, False, 4),
    (777, 3, 9, 129, False, 5),
    (2500, 50, 50, 257, False, 6),
    (1300, 120, 280, 140, False, 7),
    (4099, 200, 200, 130, True, 8),
]


@pytest.fixture(params=["i8", "f16"])
def k1_mode(request, monkeypatch):
    """Balanced designs run the int8 tensor-core path by default; RMX_I8=0
    selects the fp16 hi/lo path.  Both must give bit-identical maxima."""
    monkeypatch.setenv("RMX_I8", "1" if request.param == "i8" else "0")
    return request.param


@pytest.mark.parametrize("v,n1,n2,L,two_sided,seed", CASES)
def test_maxima_bit_exact_vs_oracle(oracle_mod, k1_mode, v, n1, n2, L, two_sided, seed):
    if k1_mode == "f16" and n1 != n2:
        pytest.skip("unbalanced designs have one path")
    x = _data(v, n1, n2, seed)
    plan = rmx.PermutationPlan(seed + 100, L, n1 + n2)
    res = rmx.run_naive_ex(x, plan, two_sided=two_sided)
    orders = plan_orders(plan).astype(np.int64)
    mx, am, _ = oracle_mod.naive_maxnull(x.values, n1, orders, two_sided, threads=8)
    assert np.array_equal(res.maxima, mx), np.abs(res.maxima - mx).max()
    assert np.array_equal(res.argmax, am)


def test_tensor_core_error_bound(oracle_mod, k1_mode):
    """|t~ - t| of the fused tcgen05 epilogue, before fp64 refinement.  fp16
    hi/lo: < 1e-5 relative; int8 on 16-bit fixed-point z: bounded by the
    quantisation (the refinement band is derived from the measured bound)."""
    import torch

    from paper_1703_01506_b200.naive_engine import NaiveJob, cuda_device, upload

    for (v, n1, n2, L, seed) in [(3000, 10, 10, 256, 11), (2000, 50, 50, 200, 12),
                                 (1500, 200, 200, 130, 13), (1200, 120, 280, 128, 14)]:
        x = _data(v, n1, n2, seed, scale=3.0)
        plan = rmx.PermutationPlan(seed, L, n1 + n2)
        orders = plan_orders(plan)
        xd, od = upload(x.values, orders, cuda_device())
        job = NaiveJob(xd, n1, od, False)
        t_dbg = job.tfill_debug().cpu().numpy().astype(np.float64)
        _, _, T = oracle_mod.naive_maxnull(x.values, n1, orders.astype(np.int64), False,
                                           materialize=True)
        err = np.abs(t_dbg - T.T) / np.maximum(np.abs(T.T), 1.0)
        assert np.isfinite(t_dbg).all()
        bound = 1e-3 if (k1_mode == "i8" and n1 == n2) else 1e-5
        assert err.max() < bound, (v, n1, n2, err.max())
        torch.cuda.synchronize()


def test_materialized_matrix_bit_exact(oracle_mod):
    x = _data(120, 3, 4, 21)
    plan = rmx.PermutationPlan(13, 40, 7)
    null, mat, counters = rmx.run_naive(x, plan, materialize=True)
    _, _, T = oracle_mod.naive_maxnull(x.values, 3, plan_orders(plan).astype(np.int64), False,
                                       materialize=True)
    assert mat.values.shape == (120, 40)
    assert np.array_equal(mat.values, T)
    assert np.array_equal(null.maxima, T.max(axis=0))
    assert counters["statistic_evaluations"] == 120 * 40


def test_constant_matrix_gives_all_zero_null():
    x = rmx.DataMatrix(np.full((10, 6), 3.5), 3, 3)
    null, _, _ = rmx.run_naive(x, rmx.PermutationPlan(5, 20, 6))
    assert np.all(null.maxima == 0.0)


def test_constant_voxel_with_inexact_means_matches_reference(oracle_mod):
    # 0.1 repeated: numpy's rounding of the group means gives t != 0
    vals = np.random.default_rng(3).standard_normal((50, 7)) * 1e-3
    vals[17] = 0.1
    x = rmx.DataMatrix(vals, 3, 4)
    plan = rmx.PermutationPlan(9, 33, 7)
    res = rmx.run_naive_ex(x, plan)
    mx, am, _ = oracle_mod.naive_maxnull(x.values, 3, plan_orders(plan).astype(np.int64), False)
    assert np.array_equal(res.maxima, mx)
    assert np.array_equal(res.argmax, am)


def test_degenerate_voxel_raises_first_in_permutation_order(oracle_mod):
    g = np.random.default_rng(4)
    vals = g.standard_normal((40, 6))
    vals[23] = [1.0, 1.0, 1.0, 2.0, 2.0, 2.0]      # degenerate under the identity
    vals[31] = [5.0, 5.0, 5.0, 7.0, 7.0, 7.0]
    x = rmx.DataMatrix(vals, 3, 3)
    plan = rmx.PermutationPlan(2, 10, 6)
    with pytest.raises(rmx.DegenerateVoxelError) as err:
        rmx.run_naive(x, plan)
    with pytest.raises(oracle_mod.OracleDegenerate) as ref:
        oracle_mod.naive_maxnull(x.values, 3, plan_orders(plan).astype(np.int64), False)
    assert err.value.voxel == ref.value.voxel == 23
    assert err.value.mean_diff == ref.value.mean_diff


def test_column_zero_is_the_true_labelling(oracle_mod):
    x = _data(500, 4, 4, 2)
    plan = rmx.PermutationPlan(9, 10, 8)
    null, _, _ = rmx.run_naive(x, plan)
    t0 = rmx.tstat_full(x.values[:, :4], x.values[:, 4:])
    assert null.maxima[0] == t0.max()


def test_two_sided_dominates_signed():
    x = _data(300, 3, 3, 7)
    plan = rmx.PermutationPlan(3, 25, 6)
    signed, _, _ = rmx.run_naive(x, plan)
    absolute, _, _ = rmx.run_naive(x, plan, two_sided=True)
    assert np.all(absolute.maxima >= signed.maxima)


def test_c1_full_config_bit_exact(oracle_mod):
    from paper_1703_01506_b200.datagen import CONFIGS, make_data_numpy

    cfg = CONFIGS["c1"]
    x = rmx.DataMatrix(make_data_numpy(cfg), cfg.n1, cfg.n2)
    plan = rmx.PermutationPlan(cfg.plan_seed, cfg.permutations, cfg.subjects)
    res = rmx.run_naive_ex(x, plan, two_sided=cfg.two_sided)
    mx, am, _ = oracle_mod.naive_maxnull(x.values, cfg.n1, plan_orders(plan).astype(np.int64),
                                         cfg.two_sided, threads=8)
    assert np.array_equal(res.maxima, mx)
    assert np.array_equal(res.argmax, am)


def test_i8_near_ties_and_outliers_bit_exact(oracle_mod, k1_mode):
    """Coarse quantisation (one huge subject per voxel) and clusters of
    near-identical voxels: many candidates inside the band, overflow to the
    exhaustive path; maxima must stay bit-identical."""
    g = np.random.default_rng(77)
    base = g.standard_normal((64, 60))
    vals = np.repeat(base, 40, axis=0) + g.standard_normal((64 * 40, 60)) * 1e-7
    vals[::7, 5] += 40.0  # outliers: large zmax -> coarse fixed point
    x = rmx.DataMatrix(vals, 30, 30)
    # 300 permutations: exhaustive fallback through X^T; 40: straight from X
    for plan, two_sided in ((rmx.PermutationPlan(5, 300, 60), False),
                            (rmx.PermutationPlan(6, 40, 60), True)):
        res = rmx.run_naive_ex(x, plan, two_sided=two_sided)
        mx, am, _ = oracle_mod.naive_maxnull(x.values, 30, plan_orders(plan).astype(np.int64),
                                             two_sided, threads=8)
        assert res.stats["overflow_perms"] > 0
        assert np.array_equal(res.maxima, mx)
        assert np.array_equal(res.argmax, am)


def test_subjects_beyond_the_tensor_tile_use_the_exact_path(oracle_mod):
    """n > ~640: the A tile no longer fits next to the TMA ring; the engine
    runs the exhaustive fp64 path (still on the GPU) with the same bits."""
    x = _data(300, 350, 350, 31)
    plan = rmx.PermutationPlan(41, 24, 700)
    res = rmx.run_naive_ex(x, plan, two_sided=True)
    mx, am, _ = oracle_mod.naive_maxnull(x.values, 350, plan_orders(plan).astype(np.int64), True,
                                         threads=8)
    assert res.stats["overflow_perms"] == 24
    assert np.array_equal(res.maxima, mx)
    assert np.array_equal(res.argmax, am)


def test_thread_count_has_no_effect():
    """Reference contract (tests/test_naive.py:78-83): results are identical
    for any thread count; here the parallelism is the GPU's."""
    x = _data(2000, 12, 12, 5)
    plan = rmx.PermutationPlan(8, 300, 24)
    a, _, _ = rmx.run_naive(x, plan, threads=1)
    b, _, _ = rmx.run_naive(x, plan, threads=7)
    assert np.array_equal(a.maxima, b.maxima)


def test_int8_pairs_many_tiles_and_chunks_bit_exact(oracle_mod):
    """int8 CTA-pair tiles over several permutation tiles and voxel chunks,
    uploaded and processed chunk by chunk from host memory."""
    x = _data(20000, 128, 128, 9)
    plan = rmx.PermutationPlan(12, 700, 256)
    res = rmx.run_naive_ex(x, plan, two_sided=True)
    assert res.stats["i8"] == 1 and res.stats["cg"] == 2 and res.stats["chunks"] > 1
    mx, am, _ = oracle_mod.naive_maxnull(x.values, 128, plan_orders(plan).astype(np.int64), True,
                                         threads=16)
    assert np.array_equal(res.maxima, mx)
    assert np.array_equal(res.argmax, am)


@pytest.mark.parametrize("v,n1,n2,L,seed", [(4099, 200, 200, 300, 21), (3001, 10, 11, 257, 22),
                                            (1, 3, 3, 30, 23)])
def test_float32_host_upload_bit_exact(oracle_mod, v, n1, n2, L, seed):
    """A DataMatrix built from float32 data uploads the float32 source
    (rmx_naive_maxnull_host_plan_f32; odd n makes the chunk offsets
    misaligned for the vector upcast); results equal the float64 upload's and
    the oracle's bit for bit."""
    g = np.random.default_rng(seed)
    f32 = g.standard_normal((v, n1 + n2)).astype(np.float32)
    x32 = rmx.DataMatrix(f32, n1, n2)
    assert x32.float32_values is not None
    x64 = rmx.DataMatrix(f32.astype(np.float64), n1, n2)
    assert x64.float32_values is None
    plan = rmx.PermutationPlan(seed + 100, L, n1 + n2)
    r32 = rmx.run_naive_ex(x32, plan)
    r64 = rmx.run_naive_ex(x64, plan)
    mx, am, _ = oracle_mod.naive_maxnull(x64.values, n1, plan_orders(plan).astype(np.int64),
                                         False, threads=8)
    assert np.array_equal(r32.maxima, r64.maxima) and np.array_equal(r32.maxima, mx)
    assert np.array_equal(r32.argmax, r64.argmax) and np.array_equal(r32.argmax, am)


@pytest.mark.parametrize("n1,n2", [(100, 100), (30, 50)])
def test_permutation_shards_bit_identical_to_single_gpu(n1, n2):
    """What each rank of an N-GPU run computes (shard.py: contiguous
    permutation ranges, labels generated on the device from the global
    index) reassembles to the single-GPU result bit for bit, for any N."""
    import torch

    from paper_1703_01506_b200.labels import device_orders
    from paper_1703_01506_b200.naive_engine import NaiveJob
    from paper_1703_01506_b200.shard import shard_bounds

    dev = torch.device("cuda", 0)
    x = _data(5000, n1, n2, 31)
    L = 1000
    plan = rmx.PermutationPlan(77, L, n1 + n2)
    full = rmx.run_naive_ex(x, plan)
    xd = torch.from_numpy(np.ascontiguousarray(x.values)).to(dev)
    for world in (2, 3, 8):
        mx, am = [], []
        for rank in range(world):
            lo, hi, _ = shard_bounds(L, rank, world)
            if hi <= lo:
                continue
            job = NaiveJob(xd, n1, device_orders(77, lo, hi, n1 + n2, dev), False)
            m, a = job.run()
            mx.append(m.cpu().numpy())
            am.append(a.cpu().numpy())
        assert np.array_equal(np.concatenate(mx), full.maxima), world
        assert np.array_equal(np.concatenate(am).astype(np.int64), full.argmax), world


@pytest.mark.parametrize("f32", [False, True])
def test_host_range_shards_bit_identical_to_single_gpu(f32):
    """rmx_naive_maxnull_host_plan_range(_f32), the host-input path each rank
    of run_naive_distributed runs: every permutation range reproduces its
    slice of the single-GPU result bit for bit (labels of the global indices
    generated on the device, X uploaded chunk by chunk), and the public
    multi-GPU entry at world size 1 equals run_naive_ex."""
    import torch

    from paper_1703_01506_b200.naive_engine import _run_from_host
    from paper_1703_01506_b200.shard import run_naive_distributed, shard_bounds

    dev = torch.device("cuda", 0)
    vals = np.random.default_rng(41).standard_normal((6000, 24)).astype(np.float32)
    x = rmx.DataMatrix(vals if f32 else vals.astype(np.float64), 12, 12)
    assert (x.float32_values is not None) == f32
    L = 900
    plan = rmx.PermutationPlan(1234, L, 24)
    full = rmx.run_naive_ex(x, plan)
    for world in (2, 3, 8):
        mx, am = [], []
        for rank in range(world):
            lo, hi, _ = shard_bounds(L, rank, world)
            if hi <= lo:
                continue
            m, a, _ = _run_from_host(x, plan, False, dev, lo, hi)
            mx.append(m)
            am.append(a)
        assert np.array_equal(np.concatenate(mx), full.maxima), world
        assert np.array_equal(np.concatenate(am).astype(np.int64), full.argmax), world
    null, arg = run_naive_distributed(x, plan)
    assert np.array_equal(null.maxima, full.maxima)
    assert np.array_equal(arg, full.argmax)


def _near_identity_orders(n, n1, L, seed):
    """Identity, then labellings that swap 1..3 subjects across the groups:
    the highest-kappa statistics a strong effect can produce (the group-1
    mean offset stays almost whole, the within-group variance tiny)."""
    g = np.random.default_rng(seed)
    rows = [np.arange(n)]
    while len(rows) < L:
        o = np.arange(n)
        k = int(g.integers(1, 4))
        a = g.choice(n1, k, replace=False)
        b = n1 + g.choice(n - n1, k, replace=False)
        o[a], o[b] = b, a
        g.shuffle(o[:n1])
        g.shuffle(o[n1:])
        rows.append(o)
    return np.stack(rows).astype(np.int16)


def _high_kappa_data(v, n1, n2, seed, effect=3.0, noise=0.02):
    g = np.random.default_rng(seed)
    vals = g.standard_normal((v, n1 + n2)) * noise
    vals[: v // 2, :n1] += effect          # kappa ~ 1 + (effect / 2 / noise)^2 ~ 5600
    vals[v // 2:, :] += g.standard_normal((v - v // 2, 1)) * 5.0  # large voxel offsets
    return rmx.DataMatrix(vals.astype(np.float32).astype(np.float64), n1, n2)


@pytest.mark.parametrize("n1,n2,mode", [(10, 10, "f16"), (50, 50, "f16"), (200, 200, "i8"),
                                        (200, 200, "f16"), (30, 70, "f16"), (120, 280, "f16")])
def test_high_kappa_stress_bit_exact(oracle_mod, monkeypatch, n1, n2, mode):
    """the refinement band must hold where cancellation in
    Q - S^2/n1 is worst (strong effect, tiny within-group variance, labellings
    one to three swaps from the truth).  Maxima and argmax must still equal
    the oracle's bit for bit."""
    from paper_1703_01506_b200.naive_engine import NaiveJob, cuda_device, upload

    monkeypatch.setenv("RMX_I8", "1" if mode == "i8" else "0")
    v, L = 3000, 384
    x = _high_kappa_data(v, n1, n2, seed=n1 + n2)
    orders = _near_identity_orders(n1 + n2, n1, L, seed=7)
    xd, od = upload(x.values, orders, cuda_device())
    mx, am = NaiveJob(xd, n1, od, False).run()
    ref_mx, ref_am, _ = oracle_mod.naive_maxnull(x.values, n1, orders.astype(np.int64), False,
                                                 threads=8)
    assert np.array_equal(mx.cpu().numpy(), ref_mx)
    assert np.array_equal(am.cpu().numpy(), ref_am)


@pytest.mark.parametrize("n1", [10, 50])
def test_fp16_accumulation_model(oracle_mod, monkeypatch, n1):
    """The fp16 S-only band is derived (rmx_abi.cu fp16_sonly_error_bound) from
    a model of the tensor core's fp32 accumulation: at most 2^-22 (|C| + sum
    |products|) per K = 16 MMA.  Check the implied |S~ - S| against that bound
    on adversarial rows: one dominant subject (|z| ~ sqrt(n)), alternating
    signs (cancellation in the accumulator), near-constant rows (subnormal
    lo halves)."""
    from paper_1703_01506_b200.naive_engine import NaiveJob, cuda_device, upload

    monkeypatch.setenv("RMX_I8", "0")
    n = 2 * n1
    g = np.random.default_rng(n1)
    v, L = 4096, 256
    vals = g.standard_normal((v, n))
    vals[0::4, 0] += 1e3                                   # one dominant subject
    vals[1::4] = np.where(np.arange(n) % 2, 1.0, -1.0) * (1 + 1e-3 * g.standard_normal(n))
    vals[2::4] = 7.0 + 1e-4 * g.standard_normal((v // 4, n))  # tiny spread around a large mean
    x = rmx.DataMatrix(vals.astype(np.float32).astype(np.float64), n1, n1)
    plan = rmx.PermutationPlan(99, L, n)
    orders = plan_orders(plan)
    xd, od = upload(x.values, orders, cuda_device())
    t_dbg = NaiveJob(xd, n1, od, False).tfill_debug().cpu().numpy().astype(np.float64)
    _, _, T = oracle_mod.naive_maxnull(x.values, n1, orders.astype(np.int64), False,
                                       materialize=True)
    T = T.T
    d1 = float(n1)
    c = (d1 * d1 / n) ** 2
    beta = c * (2.0 / (d1 * d1 * (d1 - 1.0)))
    gamma = c * (n - 1.0) / (d1 * (d1 - 1.0))
    s_of = lambda t: t * np.sqrt(gamma / (1.0 + beta * t * t))  # inverse of t = S / sqrt(gamma - beta S^2)
    ok = np.isfinite(t_dbg)
    dS = np.abs(s_of(t_dbg[ok]) - s_of(T[ok]))
    kpad = (n + 15) // 16 * 16
    P = np.sqrt(n1 * (n - 1.0))
    u = 2.0 ** -22
    e = u * P + n1 * 2.0 ** -25 + (2 * kpad / 16 + 1) * u * 1.001 * P
    slack = 2e-7 * np.abs(s_of(T[ok])) + 1e-7   # the epilogue's own fp32 evaluation of t~
    assert (dS <= e + slack).all(), (dS.max(), e)
    assert dS.max() < 0.25 * e  # the model is conservative by a wide margin
