"""Parity at BASELINE.json's own configurations.

Inputs are the configs' seeded synthetic data (datagen.make_data_numpy: the
generator the golden files were made from; a sha256 guards against drift).

  C2  NaivePT in full (L = 10,000, v = 262,144): maxima bit-identical to the
      reference's own run_naive (tests/golden/c2_naive_reference.npz).
  C4  NaivePT, the benchmarked config: the first 256 permutations at full v
      (n = 400, int8 path) bit-identical to the oracle (maxima and argmax).
  C5  NaivePT on the unbalanced design (fp16 S|Q path): the first 256
      permutations bit-identical to the oracle.
  C3  RapidPT vs the reference's own run_rapid on the same data
      (tests/golden/rapid_c3_reference.npz): training maxima bit-exact, U's
      subspace (principal cosines on a row restriction), sigma and mu, and
      the max-null distribution (reference metrics: KL, thresholds) against
      the reference RapidPT null and against the C2 NaivePT null.
  C5  RapidPT vs the engine's own NaivePT null on the same data.

Tolerances are stated per assertion.  RMX_PARITY_OUT=<path> also writes the
measured numbers as JSON (profiles/r02_parity_*.json).
"""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_1703_01506_b200 as rmx
from paper_1703_01506_b200.datagen import CONFIGS, make_data_numpy
from paper_1703_01506_b200.labels import plan_orders

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
ALPHAS = [0.1, 0.05, 0.01]
_CACHE = {}


def _report(key, obj):
    out = os.environ.get("RMX_PARITY_OUT")
    if not out:
        return
    data = {}
    if os.path.exists(out):
        with open(out) as f:
            data = json.load(f)
    data[key] = obj
    with open(out, "w") as f:
        json.dump(data, f, indent=1, default=float)


def _data(name):
    # config 3 runs on config 2's data, config 5 on config 4's grid and noise
    # but its own group split (different effect subjects): key by the data
    cfg = CONFIGS[name]
    key = (cfg.grid, cfg.n1, cfg.n2, cfg.seed, cfg.effect, cfg.sigma)
    if key not in _CACHE:
        _CACHE[key] = make_data_numpy(cfg)
    return cfg, _CACHE[key]


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_c2_full_maxnull_equals_reference():
    g = np.load(os.path.join(GOLD, "c2_naive_reference.npz"))
    cfg, vals = _data("c2")
    assert _sha(vals) == str(g["data_sha"]), "datagen drifted from the golden's data"
    x = rmx.DataMatrix(vals.astype(np.float32), cfg.n1, cfg.n2)
    plan = rmx.PermutationPlan(cfg.plan_seed, cfg.permutations, cfg.subjects)
    res = rmx.run_naive_ex(x, plan, two_sided=cfg.two_sided)
    ref = g["maxima"]
    diff = int(np.sum(res.maxima != ref))
    _report("c2_naive", {"permutations": int(ref.size), "voxels": cfg.voxels,
                         "maxima_differing": diff, "bit_exact": diff == 0,
                         "reference": "rapidmaxnull.run_naive (the unmodified reference)",
                         "engine_stats": dict(res.stats)})
    assert diff == 0  # bar: bit-identical


@pytest.mark.parametrize("name", ["c4", "c5"])
def test_naive_prefix_at_full_size_equals_oracle(oracle_mod, name):
    """The first 256 permutations of the config's plan at its full voxel
    count and subject count (C4: the benchmarked int8 path; C5: unbalanced
    fp16 S|Q path), maxima and argmax bit-identical to the oracle."""
    cfg, vals = _data(name)
    P = 256
    x = rmx.DataMatrix(vals.astype(np.float32), cfg.n1, cfg.n2)
    plan = rmx.PermutationPlan(cfg.plan_seed, P, cfg.subjects)  # = prefix of the L = 1e5 plan
    res = rmx.run_naive_ex(x, plan, two_sided=cfg.two_sided)
    orders = plan_orders(plan).astype(np.int64)
    mx, am, _ = oracle_mod.naive_maxnull(vals, cfg.n1, orders, cfg.two_sided,
                                         threads=os.cpu_count() or 8)
    diff = int(np.sum(res.maxima != mx))
    adiff = int(np.sum(res.argmax != am))
    _report(f"{name}_naive_prefix", {"permutations": P, "voxels": cfg.voxels,
                                     "subjects": cfg.subjects, "maxima_differing": diff,
                                     "argmax_differing": adiff, "bit_exact": diff == 0,
                                     "engine_stats": dict(res.stats)})
    assert diff == 0 and adiff == 0


def _principal_cosines(a, b):
    qa = np.linalg.qr(a)[0]
    qb = np.linalg.qr(b)[0]
    return np.clip(np.linalg.svd(qa.T @ qb, compute_uv=False), 0.0, 1.0)


def _null_compare(a, b):
    A, B = rmx.MaxNull(a), rmx.MaxNull(b)
    rows = rmx.threshold_table(A, B, ALPHAS)
    return {"kl": rmx.kl_divergence(B, A),
            "thresholds": [[r.alpha, r.tau_a, r.tau_b, r.percent_difference] for r in rows]}


def test_c3_rapid_matches_reference_run_rapid():
    g = np.load(os.path.join(GOLD, "rapid_c3_reference.npz"))
    gn = np.load(os.path.join(GOLD, "c2_naive_reference.npz"))
    cfg, vals = _data("c3")
    assert _sha(vals) == str(g["data_sha"])
    x = rmx.DataMatrix(vals.astype(np.float32), cfg.n1, cfg.n2)
    rc = rmx.RunConfig(permutations=cfg.permutations, seed=cfg.plan_seed, engine="rapid",
                       two_sided=cfg.two_sided, training_columns=cfg.training_columns,
                       sample_rate=cfg.sample_rate, rank=cfg.rank)
    null, model, counters = rmx.run_rapid(x, rc)
    ref_counters = json.loads(str(g["counters"]))
    rows = g["rows"]
    cos = _principal_cosines(model.basis.matrix[rows], g["basis_rows"].astype(np.float64))
    sig_rel = abs(model.residual_std - float(g["sigma"])) / float(g["sigma"])
    mu_abs = abs(model.max_shift - float(g["mu"]))
    ref_rapid = g["maxima"]
    naive = gn["maxima"]
    gpu_vs_ref = _null_compare(null.maxima, ref_rapid)
    gpu_vs_naive = _null_compare(null.maxima, naive)
    ref_vs_naive = _null_compare(ref_rapid, naive)
    rep = {
        "passes": model.passes, "ref_passes": int(g["passes"]),
        "min_principal_cosine_rows": float(cos.min()),
        "sigma": model.residual_std, "ref_sigma": float(g["sigma"]), "sigma_rel_err": sig_rel,
        "mu": model.max_shift, "ref_mu": float(g["mu"]), "mu_abs_err": mu_abs,
        "training_maxima_bit_exact": bool(np.array_equal(model.training_maxima, g["train_max"])),
        "kl_ref_rapid_vs_gpu_rapid": gpu_vs_ref["kl"],
        "kl_naive_vs_gpu_rapid": gpu_vs_naive["kl"],
        "kl_naive_vs_ref_rapid": ref_vs_naive["kl"],
        "thresholds_gpu_vs_ref_rapid": gpu_vs_ref["thresholds"],
        "thresholds_gpu_vs_naive": gpu_vs_naive["thresholds"],
        "thresholds_ref_rapid_vs_naive": ref_vs_naive["thresholds"],
        "counters_equal": {k: counters[k] == ref_counters[k] for k in
                           ("statistic_evaluations", "subsampled_statistic_evaluations",
                            "recovery_columns", "observed_rows_per_column",
                            "resampled_evaluations", "training_passes")},
        "train_seconds": counters["train_seconds"], "recover_seconds": counters["recover_seconds"],
        "ref_train_seconds_8_cores": ref_counters["train_seconds"],
        "ref_recover_seconds_8_cores": ref_counters["recover_seconds"],
    }
    _report("c3_rapid", rep)
    assert rep["training_maxima_bit_exact"]
    assert all(rep["counters_equal"].values())
    # GROUSE in fp64 on the same Omega draws: the trained subspaces coincide
    assert cos.min() > 1 - 1e-6
    assert sig_rel < 1e-6
    # mu: max-gap over the reference's own SHIFT_GAP normals, fp32 completion
    # (|error| <= ~1e-6 of the ~5 maxima it averages)
    assert mu_abs < 1e-4
    # distributions: same shape as the reference's RapidPT null (its residual
    # noise is numpy SFC64, ours Philox: two samples of one distribution) --
    # KL on 100 bins between two 10,000-draw samples of one law is ~0.01
    assert gpu_vs_ref["kl"] < 0.03
    for a, ta, tb, pct in gpu_vs_ref["thresholds"]:
        assert pct < 2.0, (a, ta, tb)
    # and as close to (or as far from) NaivePT as the reference's RapidPT is: at
    # config 3 the reference's own RapidPT null sits well below the NaivePT null
    # (KL ~3.9, thresholds ~30% low) -- the algorithm's behaviour at this
    # design, which the engine reproduces, not an engine error
    assert abs(gpu_vs_naive["kl"] - ref_vs_naive["kl"]) < 0.03 + 0.03 * ref_vs_naive["kl"]
    for (a, ta, tb, p1), (_, ra, rb, p2) in zip(gpu_vs_naive["thresholds"],
                                                ref_vs_naive["thresholds"]):
        assert abs(ta - ra) / ra < 0.02, (a, ta, ra)


def test_c5_rapid_close_to_naive_null():
    cfg, vals = _data("c5")
    x = rmx.DataMatrix(vals.astype(np.float32), cfg.n1, cfg.n2)
    rc = rmx.RunConfig(permutations=cfg.permutations, seed=cfg.plan_seed, engine="rapid",
                       two_sided=cfg.two_sided, training_columns=cfg.training_columns,
                       sample_rate=cfg.sample_rate, rank=cfg.rank)
    null, model, counters = rmx.run_rapid(x, rc)
    plan = rmx.PermutationPlan(cfg.plan_seed, cfg.permutations, cfg.subjects)
    naive = rmx.run_naive_ex(x, plan, two_sided=cfg.two_sided)
    assert np.array_equal(null.maxima[:cfg.training_columns], naive.maxima[:cfg.training_columns])
    cmp = _null_compare(null.maxima, naive.maxima)
    _report("c5_rapid", {"kl_naive_vs_gpu_rapid": cmp["kl"],
                         "thresholds_gpu_vs_naive": cmp["thresholds"],
                         "sigma": model.residual_std, "mu": model.max_shift,
                         "train_seconds": counters["train_seconds"],
                         "recover_seconds": counters["recover_seconds"]})
    # reported, not bounded: how far RapidPT's null sits from NaivePT's is the
    # algorithm's property at this design (at config 3 the reference's own
    # RapidPT is ~30% low, test_c3_rapid_matches_reference_run_rapid); what the
    # engine must get right is checked above and at config 3 against the reference
    assert np.isfinite(cmp["kl"]) and all(np.isfinite(t[1]) for t in cmp["thresholds"])
