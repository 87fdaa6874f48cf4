"""GPU engine vs the reference's own outputs (tests/golden/*.npz), through the
public API and the C ABI.  Bar: bit-identical maxima and statistic matrices."""
import os

import numpy as np
import pytest

import paper_1703_01506_b200 as rmx

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
CASES = ["tiny", "single_voxel", "n20_two", "unbal", "n100", "n400_unbal"]


@pytest.mark.parametrize("name", CASES)
def test_run_naive_matches_reference_bits(name):
    g = np.load(os.path.join(GOLD, "naive_cases.npz"))
    v, n1, n2, L, two, ps = (int(t) for t in g[f"{name}_meta"])
    x = rmx.DataMatrix(g[f"{name}_x"].astype(np.float64), n1, n2)
    plan = rmx.PermutationPlan(ps, L, n1 + n2)
    mat = f"{name}_T" in g.files
    null, T, counters = rmx.run_naive(x, plan, materialize=mat, two_sided=bool(two))
    assert np.array_equal(null.maxima, g[f"{name}_maxima"])
    assert counters["statistic_evaluations"] == int(g[f"{name}_evals"])
    if mat:
        assert np.array_equal(T.values, g[f"{name}_T"])


def test_constant_and_degenerate_cases_match_reference():
    g = np.load(os.path.join(GOLD, "naive_cases.npz"))
    null, _, _ = rmx.run_naive(rmx.DataMatrix(np.full((10, 6), 3.5), 3, 3),
                               rmx.PermutationPlan(5, 20, 6))
    assert np.array_equal(null.maxima, g["const_maxima"])
    null, _, _ = rmx.run_naive(rmx.DataMatrix(g["cvox_x"], 3, 4), rmx.PermutationPlan(9, 33, 7))
    assert np.array_equal(null.maxima, g["cvox_maxima"])
    with pytest.raises(rmx.DegenerateVoxelError) as err:
        rmx.run_naive(rmx.DataMatrix(g["deg_x"], 3, 3), rmx.PermutationPlan(2, 10, 6))
    assert err.value.voxel == int(g["deg_voxel"])
    assert err.value.mean_diff == float(g["deg_mean_diff"])


def test_tstat_full_matches_reference_bits():
    g = np.load(os.path.join(GOLD, "teststat.npz"))
    assert rmx.tstat_full(np.array([[1.0, 2.0, 3.0]]), np.array([[4.0, 5.0, 6.0]]))[0] == g["hand"][0]
    for n1, n2 in ((5, 7), (2, 2), (8, 8), (50, 50), (130, 9), (200, 200)):
        t = rmx.tstat_full(g[f"x1_{n1}_{n2}"], g[f"x2_{n1}_{n2}"])
        assert np.array_equal(t, g[f"t_{n1}_{n2}"])
    idx = np.array([3, 7, 40])
    t = rmx.tstat_subset(g["x1_5_7"], g["x2_5_7"], idx)
    assert np.array_equal(t, g["t_5_7"][idx])


def test_c1_config_matches_reference_bits():
    from paper_1703_01506_b200.datagen import CONFIGS, make_data_numpy

    g = np.load(os.path.join(GOLD, "c1_reference.npz"))
    cfg = CONFIGS["c1"]
    x = rmx.DataMatrix(make_data_numpy(cfg), cfg.n1, cfg.n2)
    null, _, _ = rmx.run_naive(x, rmx.PermutationPlan(cfg.plan_seed, cfg.permutations,
                                                      cfg.subjects), two_sided=True)
    assert np.array_equal(null.maxima, g["maxima"])
