"""Golden RapidPT run at config 3 shape, produced by the REFERENCE itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_rapid_c3.py [--threads 8]

Config 3 (BASELINE.json configs[2]): the config-2 data (n=100,
50/50, v=262,144 on a 64^3 grid, sigma=2 smoothing, +0.5 in a 16^3 cube),
L=10,000, ell=r=100, eta=0.5% (k=1,311), max-gap shift, 50 passes.  The
unmodified reference (`rapidmaxnull.run_rapid`, imported from
/root/reference/pkg/src) is run on exactly the float32-valued data the GPU
tests generate with `datagen.make_data_numpy`; `train_basis` is wrapped (not
changed) to capture its pass residuals.

Stored in tests/golden/rapid_c3_reference.npz (small enough to commit):
  maxima        the reference's RapidPT max-null (10,000 fp64)
  train_max     training maxima (100)
  sigma, mu     residual_std, max_shift
  passes, converged, pass_resid
  basis_rows    U_ref restricted to rows `rows` (every 64th voxel, fp32) --
                a row restriction of the same column space, so principal
                angles between restrictions of U_gpu and U_ref bound the
                subspace agreement without shipping the 210 MB basis
  rows          the restricting row ids
  counters      the reference's counter dict (json)
  data_sha      sha256 of the float64 data matrix (guards generator drift)

The config-2 NaivePT max-null of the same data (reference semantics,
bit-exact) is stored beside it in c2_naive_maxnull.npz by
`make_c2_naive.py` (the C oracle, pinned to the reference).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

import rapidmaxnull as R  # noqa: E402
from rapidmaxnull import lrmc as RL  # noqa: E402
from rapidmaxnull import rapid as RR  # noqa: E402

from paper_1703_01506_b200.datagen import CONFIGS, make_data_numpy  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    ap.add_argument("--out", default=os.path.join(HERE, "rapid_c3_reference.npz"))
    args = ap.parse_args()

    cfg = CONFIGS["c3"]
    t0 = time.time()
    vals = make_data_numpy(cfg)
    print(f"data {vals.shape} in {time.time() - t0:.1f}s", flush=True)
    x = R.DataMatrix(vals, cfg.n1, cfg.n2)
    rc = R.RunConfig(permutations=cfg.permutations, seed=cfg.plan_seed, engine="rapid",
                     two_sided=cfg.two_sided, training_columns=cfg.training_columns,
                     sample_rate=cfg.sample_rate, rank=cfg.rank, threads=args.threads)

    captured = {}
    real_train_basis = RL.train_basis

    def spy(*a, **kw):
        res = real_train_basis(*a, **kw)
        captured["pass_resid"] = list(res.pass_residuals)
        captured["updates"] = res.updates
        return res

    RR.train_basis = spy
    t0 = time.time()
    null, model, counters = R.run_rapid(x, rc)
    print(f"run_rapid {time.time() - t0:.1f}s  counters={counters}", flush=True)

    rows = np.arange(0, cfg.voxels, 64, dtype=np.int64)
    np.savez_compressed(
        args.out,
        maxima=np.asarray(null.maxima, dtype=np.float64),
        train_max=np.asarray(model.training_maxima, dtype=np.float64),
        sigma=np.float64(model.residual_std),
        mu=np.float64(model.max_shift),
        passes=np.int64(model.passes),
        converged=np.bool_(model.converged),
        pass_resid=np.asarray(captured["pass_resid"], dtype=np.float64),
        basis_rows=model.basis.matrix[rows].astype(np.float32),
        rows=rows,
        counters=np.array(json.dumps(counters)),
        data_sha=np.array(hashlib.sha256(np.ascontiguousarray(vals).tobytes()).hexdigest()),
        numpy_version=np.array(np.__version__),
    )
    print("wrote", args.out, flush=True)


if __name__ == "__main__":
    main()
