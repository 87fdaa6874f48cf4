"""SURVEY 8f f3 on the GPU: NaivePT straight from a .mat0 file
(rmx_naive_maxnull_mat0: file -> page-locked ring -> device, K0/K1 per chunk
as it lands) and the streamed --dump-T writer (rmx_tstat_dump_mat0).

The bar is the reference CLI's own path (cli.py:70-116): read_matrix ->
run_naive(materialize=...) -> write_array(mat.values, dump_t).  Maxima and
argmax are bit-identical to the in-memory engine and the CPU oracle; the
dumped file is byte-identical to write_array of the oracle's statistic
matrix (pinned to the reference by tests/test_oracle_golden.py).
"""
import numpy as np
import pytest

import paper_1703_01506_b200 as rmx
from paper_1703_01506_b200 import matfiles as mf
from paper_1703_01506_b200.labels import plan_orders

pytestmark = pytest.mark.gpu


def _data(v, n1, n2, seed):
    g = np.random.default_rng(seed)
    vals = g.standard_normal((v, n1 + n2)).astype(np.float32).astype(np.float64)
    vals[: max(1, v // 50), :n1] += 0.7
    return rmx.DataMatrix(vals, n1, n2)


@pytest.mark.parametrize("v,n1,n2,L,two_sided,staging", [
    (5000, 10, 10, 300, True, 3 * 20 * 8 * 7),      # 7-row slots: ~240 pieces
    (20000, 200, 200, 260, False, 3 * 400 * 8 * 1000),  # int8 path, many chunks
    (3001, 120, 280, 129, False, 192 << 20),       # unbalanced, one piece
    (40, 3, 4, 50, False, 2 * 7 * 8),              # exhaustive exact path, 1-row slots
])
def test_file_engine_bit_identical(tmp_path, oracle_mod, v, n1, n2, L, two_sided, staging):
    x = _data(v, n1, n2, v + L)
    p = tmp_path / "x.mat0"
    mf.write_matrix(x, p)
    plan = rmx.PermutationPlan(1703, L, n1 + n2)
    res = rmx.run_naive_mat0(p, plan, two_sided=two_sided, staging_bytes=staging)
    ref = rmx.run_naive_ex(x, plan, two_sided=two_sided)
    assert np.array_equal(res.maxima, ref.maxima) and np.array_equal(res.argmax, ref.argmax)
    mx, am, _ = oracle_mod.naive_maxnull(x.values, n1, plan_orders(plan).astype(np.int64),
                                         two_sided)
    assert np.array_equal(res.maxima, mx) and np.array_equal(res.argmax, am)


def test_file_engine_permutation_range(tmp_path):
    x = _data(3000, 50, 50, 5)
    p = tmp_path / "x.mat0"
    mf.write_matrix(x, p)
    plan = rmx.PermutationPlan(77, 700, 100)
    full = rmx.run_naive_mat0(p, plan)
    parts = [rmx.run_naive_mat0(p, plan, lo=a, hi=b) for a, b in ((0, 256), (256, 512), (512, 700))]
    assert np.array_equal(np.concatenate([r.maxima for r in parts]), full.maxima)
    assert np.array_equal(np.concatenate([r.argmax for r in parts]), full.argmax)


def test_dump_t_matches_reference_write_array(tmp_path, oracle_mod):
    v, n1, n2, L = 1500, 6, 9, 70
    x = _data(v, n1, n2, 9)
    p = tmp_path / "x.mat0"
    mf.write_matrix(x, p)
    plan = rmx.PermutationPlan(31, L, n1 + n2)
    d = tmp_path / "T.mat0"
    res = rmx.run_naive_mat0(p, plan, dump_t=d)
    _, _, T = oracle_mod.naive_maxnull(x.values, n1, plan_orders(plan).astype(np.int64), False,
                                       materialize=True)
    want = tmp_path / "want.mat0"
    mf.write_array(T, want)  # the reference CLI: write_array(mat.values, dump_t)
    assert d.read_bytes() == want.read_bytes()
    assert np.array_equal(res.maxima, T.max(axis=0))
    # device inputs, slabs forced small: 2 slots of 37 voxel rows -> 41
    # slabs, the last one ragged
    import paper_1703_01506_b200.naive_engine as ne
    from paper_1703_01506_b200.labels import device_orders

    d2 = tmp_path / "T2.mat0"
    xd = ne.data_to_device(x, ne.cuda_device())
    od = device_orders(plan.master_seed, 0, L, n1 + n2, xd.device)
    ne.dump_statistic_matrix_device(xd, n1, od, d2, staging_bytes=2 * 37 * L * 8)
    assert d2.read_bytes() == want.read_bytes()
    d3 = tmp_path / "T3.mat0"
    rmx.dump_statistic_matrix(x, plan, d3)
    assert d3.read_bytes() == want.read_bytes()


def test_file_engine_nonfinite_and_bare(tmp_path):
    x = _data(2000, 10, 10, 3)
    vals = np.array(x.values)
    vals[1234, 7] = np.nan
    p = tmp_path / "bad.mat0"
    mf.write_array(vals, p, 10, 10)
    plan = rmx.PermutationPlan(5, 100, 20)
    with pytest.raises(rmx.DataFormatError) as e:
        rmx.run_naive_mat0(p, plan, staging_bytes=3 * 20 * 8 * 64)
    with pytest.raises(rmx.DataFormatError) as e2:
        mf.read_array(p)
    assert str(e.value) == str(e2.value)  # the reference's message, byte offset included
    q = tmp_path / "bare.mat0"
    mf.write_array(x.values, q)
    with pytest.raises(rmx.DataFormatError) as e3:
        rmx.run_naive_mat0(q, plan)
    with pytest.raises(rmx.DataFormatError) as e4:
        mf.read_matrix(q)
    assert str(e3.value) == str(e4.value)
    with pytest.raises(rmx.UsageError):
        rmx.run_naive_mat0(tmp_path / "bad.mat0", rmx.PermutationPlan(5, 10, 21))


def test_dump_t_degenerate_raises_and_removes(tmp_path):
    vals = np.random.default_rng(2).standard_normal((300, 8))
    vals[211, :] = 0.0
    vals[211, 0] = 1.0  # zero pooled variance under some labelling, nonzero mean difference
    x = rmx.DataMatrix(vals, 4, 4)
    plan = rmx.PermutationPlan(3, 60, 8)
    d = tmp_path / "T.mat0"
    try:
        rmx.run_naive(x, plan)
        degenerate = False
    except rmx.DegenerateVoxelError:
        degenerate = True
    if not degenerate:
        pytest.skip("no degenerate labelling drawn")
    with pytest.raises(rmx.DegenerateVoxelError) as e:
        rmx.dump_statistic_matrix(x, plan, d)
    assert not d.exists()
    with pytest.raises(rmx.DegenerateVoxelError) as e2:
        rmx.run_naive(x, plan)
    assert str(e.value) == str(e2.value)
