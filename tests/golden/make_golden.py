"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

Everything stored here is an output of the unmodified reference package
(rapidmaxnull 0.1.0 imported from /root/reference/pkg/src) on seeded inputs;
the tests compare the C oracle and the CUDA engine against these vectors.
The fixtures are small (< 2 MB) and committed; this script is committed so
they can be regenerated.  Nothing on the GPU box reads /root/reference.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

import rapidmaxnull as R  # noqa: E402
from rapidmaxnull import streams as RS  # noqa: E402
from rapidmaxnull.lrmc import ObservedColumn, fit_coefficients, solve_block  # noqa: E402
from rapidmaxnull.rapid import SubspaceModel  # noqa: E402
from rapidmaxnull.teststat import _welch_rows  # noqa: E402


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def orders_of(plan) -> np.ndarray:
    return np.stack([plan.shuffle(i) for i in range(plan.count)]).astype(np.int16)


def shuffles():
    out = {}
    for seed in (7, 1703015061, 1703015062, 1703015064, 1703015065):
        for n in (4, 6, 20, 100, 400):
            plan = R.PermutationPlan(seed, 64, n)
            out[f"s{seed}_n{n}"] = orders_of(plan)
    # Omega draws (rapid.py:158-160 / lrmc.py:237-241)
    for seed, v, k in ((3, 40, 24), (1703015062, 262144, 1311), (1703015065, 524288, 1836)):
        rows = []
        for i in range(8):
            rows.append(np.sort(RS.stream(seed, RS.RECOVER_OMEGA, i).choice(v, size=k, replace=False)))
        out[f"omega_recover_{seed}_{v}_{k}"] = np.stack(rows).astype(np.int32)
        rows = []
        for i in range(4):
            rows.append(np.sort(RS.stream(seed, RS.TRAIN_OMEGA, i, 1).choice(v, size=k, replace=False)))
        out[f"omega_train_{seed}_{v}_{k}"] = np.stack(rows).astype(np.int32)
    out["numpy_version"] = np.array(np.__version__)
    np.savez_compressed(os.path.join(HERE, "shuffles.npz"), **out)


NAIVE_CASES = [
    # name, v, n1, n2, L, two_sided, data seed, plan seed, scale, materialize
    ("tiny", 20, 2, 2, 50, False, 42, 7, 1.0, True),
    ("single_voxel", 1, 3, 3, 30, False, 1, 5, 1.0, True),
    ("n20_two", 300, 10, 10, 200, True, 3, 11, 1.0, True),
    ("unbal", 777, 3, 9, 129, False, 5, 13, 2.0, False),
    ("n100", 800, 50, 50, 130, False, 6, 17, 1.0, False),
    ("n400_unbal", 300, 120, 280, 70, False, 7, 19, 1.0, False),
]


def naive():
    out = {}
    for name, v, n1, n2, L, two, ds, ps, scale, mat in NAIVE_CASES:
        g = np.random.default_rng(ds)
        x = f32(g.standard_normal((v, n1 + n2)) * scale)
        dm = R.DataMatrix(x, n1, n2)
        plan = R.PermutationPlan(ps, L, n1 + n2)
        null, T, counters = R.run_naive(dm, plan, materialize=mat, two_sided=two, threads=1)
        out[f"{name}_x"] = x.astype(np.float32)  # float32-exact values
        out[f"{name}_meta"] = np.array([v, n1, n2, L, int(two), ps], dtype=np.int64)
        out[f"{name}_maxima"] = null.maxima
        out[f"{name}_orders"] = orders_of(plan)
        out[f"{name}_evals"] = np.array(counters["statistic_evaluations"])
        if mat:
            out[f"{name}_T"] = T.values
    # constant matrix -> all-zero null (tests/test_naive.py:54-58)
    x = np.full((10, 6), 3.5)
    out["const_maxima"] = R.run_naive(R.DataMatrix(x, 3, 3), R.PermutationPlan(5, 20, 6))[0].maxima
    # constant voxel whose group means round differently (0.1 x 3 vs 0.1 x 4)
    g = np.random.default_rng(3)
    x = g.standard_normal((50, 7)) * 1e-3
    x[17] = 0.1
    plan = R.PermutationPlan(9, 33, 7)
    out["cvox_x"] = x
    out["cvox_maxima"] = R.run_naive(R.DataMatrix(x, 3, 4), plan)[0].maxima
    # degenerate voxel: the reference raises at the first (perm, voxel)
    g = np.random.default_rng(4)
    x = g.standard_normal((40, 6))
    x[23] = [1.0, 1.0, 1.0, 2.0, 2.0, 2.0]
    x[31] = [5.0, 5.0, 5.0, 7.0, 7.0, 7.0]
    out["deg_x"] = x
    try:
        R.run_naive(R.DataMatrix(x, 3, 3), R.PermutationPlan(2, 10, 6))
        raise SystemExit("expected DegenerateVoxelError")
    except R.DegenerateVoxelError as e:
        out["deg_voxel"] = np.array(e.voxel)
        out["deg_mean_diff"] = np.array(e.mean_diff)
    np.savez_compressed(os.path.join(HERE, "naive_cases.npz"), **out)


def c1():
    from paper_1703_01506_b200.datagen import CONFIGS, make_data_numpy

    cfg = CONFIGS["c1"]
    x = make_data_numpy(cfg)
    plan = R.PermutationPlan(cfg.plan_seed, cfg.permutations, cfg.subjects)
    null, _, _ = R.run_naive(R.DataMatrix(x, cfg.n1, cfg.n2), plan, two_sided=cfg.two_sided)
    np.savez_compressed(os.path.join(HERE, "c1_reference.npz"), maxima=null.maxima,
                        x_sha256=np.array(sha(x)), x_head=x[:64].copy())


def teststat():
    out = {}
    out["hand"] = R.tstat_full(np.array([[1.0, 2.0, 3.0]]), np.array([[4.0, 5.0, 6.0]]))
    g = np.random.default_rng(3)
    for n1, n2 in ((5, 7), (2, 2), (8, 8), (50, 50), (130, 9), (200, 200)):
        x1 = g.standard_normal((64, n1)) * g.uniform(0.01, 100)
        x2 = g.standard_normal((64, n2)) * g.uniform(0.01, 100) + g.uniform(-1, 1)
        out[f"x1_{n1}_{n2}"] = x1
        out[f"x2_{n1}_{n2}"] = x2
        out[f"t_{n1}_{n2}"] = R.tstat_full(x1, x2)
    s = g.standard_normal(1000) * 1e3
    out["sums_x"] = s
    out["sums"] = np.array([np.add.reduce(s[:k]) for k in range(1, 1001)])
    np.savez_compressed(os.path.join(HERE, "teststat.npz"), **out)


def rapid():
    """Small RapidPT runs: model, maxima and the recovery algebra."""
    out = {}
    g = np.random.default_rng(11)
    x = f32(g.standard_normal((80, 6)))
    cfg = R.RunConfig(permutations=120, seed=12, engine="rapid", training_columns=6, rank=5,
                      sample_rate=0.5)
    null, model, counters = R.run_rapid(R.DataMatrix(x, 3, 3), cfg)
    out["r1_x"] = x.astype(np.float32)
    out["r1_meta"] = np.array([80, 3, 3, 120, 12, 6, 5], dtype=np.int64)
    out["r1_eta"] = np.array(0.5)
    out["r1_maxima"] = null.maxima
    out["r1_basis"] = model.basis.matrix
    out["r1_sigma"] = np.array(model.residual_std)
    out["r1_mu"] = np.array(model.max_shift)
    out["r1_train_max"] = model.training_maxima
    out["r1_counters"] = np.array([counters["statistic_evaluations"],
                                   counters["subsampled_statistic_evaluations"],
                                   counters["full_statistic_evaluations"],
                                   counters["resampled_evaluations"]])
    # noise-free recovery with the reference-trained basis: sigma = 0, mu = 0
    m0 = SubspaceModel(basis=model.basis, residual_std=0.0, max_shift=0.0,
                       training_columns=model.training_columns, sample_rate=model.sample_rate,
                       training_maxima=model.training_maxima, two_sided=False, seed=12,
                       passes=model.passes, converged=model.converged)
    plan = cfg.plan_for(R.DataMatrix(x, 3, 3))
    null0, _ = R.recover(R.DataMatrix(x, 3, 3), m0, plan, cfg)
    out["r1_maxima_sigma0"] = null0.maxima
    out["r1_orders"] = orders_of(plan)
    k = int(np.ceil(0.5 * 80))
    om = np.stack([np.sort(RS.stream(12, RS.RECOVER_OMEGA, i).choice(80, size=k, replace=False))
                   for i in range(120)])
    out["r1_omegas"] = om.astype(np.int32)
    # exact regime (tests/test_rapid.py:72-79): v = n = rank, eta = 1, sigma = mu = 0
    g = np.random.default_rng(4)
    x = f32(g.standard_normal((8, 8)))
    cfg = R.RunConfig(permutations=60, seed=3, engine="rapid", training_columns=8, rank=8,
                      sample_rate=1.0, max_passes=5, sigma_override=0.0, shift_override=0.0)
    null, model, _ = R.run_rapid(R.DataMatrix(x, 4, 4), cfg)
    out["exact_x"] = x
    out["exact_maxima"] = null.maxima
    # solve_block / fit_coefficients
    g = np.random.default_rng(6)
    b = R.init_basis(300, 8, seed=11)
    stack, values = [], []
    for _ in range(16):
        idx = np.sort(g.choice(300, size=50, replace=False))
        col = g.standard_normal(300)
        stack.append(b.matrix[idx])
        values.append(col[idx])
    w, conds = solve_block(np.stack(stack), np.stack(values))
    out["sb_u"] = np.stack(stack)
    out["sb_vals"] = np.stack(values)
    out["sb_w"] = w
    out["sb_conds"] = conds
    out["sb_fit0"] = fit_coefficients(b, ObservedColumn(np.arange(50) * 6, b.matrix[::6][:50] @ np.ones(8)))
    # welch rows on gathered blocks (batched, reshaped) -- bit pattern pin
    g = np.random.default_rng(8)
    b1 = g.standard_normal((40, 3))
    b2 = g.standard_normal((40, 5))
    out["wr_b1"], out["wr_b2"], out["wr_t"] = b1, b2, _welch_rows(b1, b2)
    np.savez_compressed(os.path.join(HERE, "rapid_cases.npz"), **out)


def rapid_degenerate():
    """A voxel whose within-group variances vanish under a recovery
    permutation (values {1, 1, 2 | 1, 2, 2}, split 1/2 by some shuffle) but
    not under the training ones: the reference raises DegenerateVoxelError
    from recover() (rapid.py:166 -> teststat.py:42-49) with the flat index
    into the span's (count x k) block."""
    g = np.random.default_rng(5)
    x = f32(g.standard_normal((10, 6)))
    x[3] = [1, 1, 2, 1, 2, 2]
    seed = 1
    cfg = R.RunConfig(permutations=40, seed=seed, engine="rapid", training_columns=3, rank=2,
                      sample_rate=1.0, max_passes=3)
    dm = R.DataMatrix(x, 3, 3)
    model, _, _ = R.train(dm, cfg)
    try:
        R.recover(dm, model, cfg.plan_for(dm), cfg)
        raise SystemExit("expected a degenerate voxel in recovery")
    except R.DegenerateVoxelError as e:
        voxel, mean_diff, msg = e.voxel, e.mean_diff, str(e)
    np.savez_compressed(os.path.join(HERE, "rapid_degenerate.npz"), x=x.astype(np.float32),
                        meta=np.array([40, seed, 3, 2, 3], dtype=np.int64), voxel=np.array(voxel),
                        mean_diff=np.array(mean_diff), msg=np.array(msg))


def matio():
    """Files written by the reference's matio and the reference's error
    messages for malformed files (path replaced by <PATH>)."""
    import struct
    import tempfile

    from rapidmaxnull import matio as M

    g = np.random.default_rng(7)
    vals = g.standard_normal((7, 5))
    vals[0, 0], vals[1, 1], vals[2, 2] = -0.0, 1e-300, 1.2345678901234567e300
    x = R.DataMatrix(vals, 2, 3)
    out = {"values": vals, "n1": 2, "n2": 3}
    with tempfile.TemporaryDirectory() as d:
        pb, pc = os.path.join(d, "x.mat0"), os.path.join(d, "x.csv")
        M.write_matrix(x, pb)
        M.write_matrix_csv(x, pc)
        out["mat0_bytes"] = np.frombuffer(open(pb, "rb").read(), dtype=np.uint8)
        out["csv_bytes"] = np.frombuffer(open(pc, "rb").read(), dtype=np.uint8)
        good = open(pb, "rb").read()
        hdr = struct.Struct("<8sIQQQQ")
        nan = bytearray(good)
        nan[44 + (3 * 5 + 4) * 8:44 + (3 * 5 + 5) * 8] = struct.pack("<d", float("nan"))
        cases = {
            "truncated_header": good[:20],
            "bad_magic": b"RMXMAT1\x00" + good[8:],
            "bad_version": good[:8] + struct.pack("<I", 2) + good[12:],
            "empty_dims": hdr.pack(b"RMXMAT0\x00", 1, 0, 5, 2, 3),
            "short_payload": good[:-8],
            "long_payload": good + b"\x00" * 8,
            "non_finite": bytes(nan),
            "bare": hdr.pack(b"RMXMAT0\x00", 1, 7, 5, 0, 0) + good[44:],
            "bad_split": hdr.pack(b"RMXMAT0\x00", 1, 7, 5, 1, 4) + good[44:],
        }
        names, msgs = [], []
        for name, data in cases.items():
            fp = os.path.join(d, name + ".mat0")
            open(fp, "wb").write(data)
            try:
                M.read_matrix(fp)
                msg = "OK"
            except Exception as e:  # DataFormatError
                msg = type(e).__name__ + ": " + str(e).replace(fp, "<PATH>")
            names.append(name)
            msgs.append(msg)
            out["case_" + name] = np.frombuffer(data, dtype=np.uint8)
        csv_cases = {
            "csv_header": "1,2,3\n",
            "csv_nonint": "a,b,c,d\n",
            "csv_short": "3,2,1,1\n1,2\n3,4\n",
            "csv_cells": "2,2,1,1\n1,2\n3\n",
            "csv_cell": "2,2,1,1\n1,x\n3,4\n",
            "csv_inf": "2,2,1,1\n1,inf\n3,4\n",
            "csv_trailing": "1,4,2,2\n1,2,3,4\n5\n",
            "csv_zero": "0,2,1,1\n",
        }
        for name, text in csv_cases.items():
            fp = os.path.join(d, name + ".csv")
            open(fp, "w").write(text)
            try:
                M.read_matrix_csv(fp)
                msg = "OK"
            except Exception as e:
                msg = type(e).__name__ + ": " + str(e).replace(fp, "<PATH>")
            names.append(name)
            msgs.append(msg)
            out["case_" + name] = np.frombuffer(text.encode(), dtype=np.uint8)
    out["case_names"] = np.array(names)
    out["case_msgs"] = np.array(msgs)
    np.savez_compressed(os.path.join(HERE, "matio.npz"), **out)


if __name__ == "__main__":
    matio()
    shuffles()
    naive()
    c1()
    teststat()
    rapid()
    rapid_degenerate()
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))
