"""Max-null queries and comparison metrics vs the reference's own outputs
(tests/golden/metrics.npz from make_metrics_golden.py; rmx/teststat.py:93-131,
rmx/metrics.py:34-109).  Host code: runs without a GPU.  Bar: bit-exact."""
import os

import numpy as np
import pytest

import paper_1703_01506_b200 as rmx

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def g():
    return np.load(os.path.join(GOLD, "metrics.npz"))


def test_kl_and_histograms(g):
    A, B, C = rmx.MaxNull(g["a"]), rmx.MaxNull(g["b"]), rmx.MaxNull(g["c"])
    for bins in (2, 17, 100):
        assert rmx.kl_divergence(A, B, bins) == g[f"kl_ab_{bins}"]
        assert rmx.kl_divergence(B, A, bins) == g[f"kl_ba_{bins}"]
        h = rmx.build_histogram_pair(A, B, bins)
        assert np.array_equal(h.edges, g[f"hp_edges_{bins}"])
        assert np.array_equal(h.p, g[f"hp_p_{bins}"]) and np.array_equal(h.q, g[f"hp_q_{bins}"])
    assert rmx.kl_divergence(C, C) == g["kl_cc"]
    with pytest.raises(rmx.UsageError, match="need at least 2 bins"):
        rmx.kl_divergence(A, B, 1)


def test_threshold_table_threshold_pvalue_reject(g):
    A, B, C = rmx.MaxNull(g["a"]), rmx.MaxNull(g["b"]), rmx.MaxNull(g["c"])
    rows = rmx.threshold_table(A, B, list(g["alphas"]))
    got = np.array([[r.alpha, r.tau_a, r.tau_b, r.percent_difference] for r in rows])
    assert np.array_equal(got, g["tt"])
    assert np.array_equal([rmx.threshold_at(A, a) for a in g["alphas"]], g["thr_a"])
    assert np.array_equal([rmx.threshold_at(C, a) for a in (0.5, 0.1, 0.05)], g["thr_c"])
    assert np.array_equal([rmx.pvalue(A, o) for o in g["obs"]], g["pv_a"])
    assert np.array_equal(rmx.reject_set(g["smap"], 3.0), g["reject"])
    with pytest.raises(rmx.UsageError, match="alpha must be in"):
        rmx.threshold_at(A, 1.0)
    with pytest.raises(rmx.UsageError, match="below the resolution"):
        rmx.threshold_at(A, 1e-4)


def test_resampling_risk(g):
    r = rmx.resampling_risk(g["r1"], g["r2"])
    assert [r.n_a, r.n_b, r.n_common, r.risk] == list(g["risk"]) and r.defined
    e = rmx.resampling_risk(g["r1"], np.array([], dtype=np.int64))
    assert e.risk is None and not e.defined
    assert [e.n_a, e.n_b, e.n_common] == list(g["risk_empty"][:3])
