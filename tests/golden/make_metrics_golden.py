"""Golden outputs of the reference's max-null queries and comparison metrics
(rmx/teststat.py:93-131, rmx/metrics.py:34-109), produced by the REFERENCE
itself in the build container:

    python tests/golden/make_metrics_golden.py

Inputs are seeded synthetic max-null vectors (with ties) and rejection sets;
outputs are stored beside them in tests/golden/metrics.npz.
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import rapidmaxnull as R  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    g = np.random.default_rng(20261020)
    a = np.round(g.gumbel(4.0, 0.6, 1000), 3)          # rounding creates ties
    b = np.round(g.gumbel(4.05, 0.62, 1500), 3)
    c = np.full(40, 2.5)                               # degenerate all-equal null
    alphas = np.array([0.5, 0.1, 0.05, 0.01, 0.002])
    out = {"a": a, "b": b, "c": c, "alphas": alphas}
    A, B, C = R.MaxNull(a), R.MaxNull(b), R.MaxNull(c)
    for bins in (2, 17, 100):
        out[f"kl_ab_{bins}"] = np.float64(R.kl_divergence(A, B, bins))
        out[f"kl_ba_{bins}"] = np.float64(R.kl_divergence(B, A, bins))
        h = R.build_histogram_pair(A, B, bins)
        out[f"hp_edges_{bins}"], out[f"hp_p_{bins}"], out[f"hp_q_{bins}"] = h.edges, h.p, h.q
    out["kl_cc"] = np.float64(R.kl_divergence(C, C))
    rows = R.threshold_table(A, B, list(alphas))
    out["tt"] = np.array([[r.alpha, r.tau_a, r.tau_b, r.percent_difference] for r in rows])
    out["thr_a"] = np.array([R.threshold_at(A, al) for al in alphas])
    out["thr_c"] = np.array([R.threshold_at(C, al) for al in (0.5, 0.1, 0.05)])
    obs = np.array([2.0, 4.0, 4.5, 5.0, 9.0, float(a[7])])
    out["obs"] = obs
    out["pv_a"] = np.array([R.pvalue(A, o) for o in obs])
    smap = g.standard_normal(500) * 2.0
    out["smap"] = smap
    out["reject"] = R.reject_set(smap, 3.0)
    r1 = g.choice(300, 40, replace=False)
    r2 = np.concatenate([r1[:25], g.choice(np.arange(300, 400), 10, replace=False)])
    res = R.resampling_risk(r1, r2)
    out["r1"], out["r2"] = r1, r2
    out["risk"] = np.array([res.n_a, res.n_b, res.n_common, res.risk])
    e = R.resampling_risk(r1, np.array([], dtype=np.int64))
    out["risk_empty"] = np.array([e.n_a, e.n_b, e.n_common, -1.0 if e.risk is None else e.risk])
    np.savez_compressed(os.path.join(HERE, "metrics.npz"), **out)
    print("wrote metrics.npz")


if __name__ == "__main__":
    main()
