"""Golden NaivePT max-null at config 2, produced by the REFERENCE itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_c2_naive.py [--threads 8]

Config 2 (BASELINE.json configs[1]): n=100 (50/50), v=262,144 (64^3 grid,
sigma=2, +0.5 in a 16^3 cube), L=10,000, signed max t.  The unmodified
reference `rapidmaxnull.run_naive` (imported from /root/reference/pkg/src)
runs on exactly the float32-valued data `datagen.make_data_numpy` builds
(~20 min on 8 cores).  Stored in tests/golden/c2_naive_reference.npz:
maxima (10,000 fp64), the counters, and the data hash.  The GPU test
(tests/test_gpu_configs.py) asserts the engine's C2 maxima equal these bit
for bit; the C3 RapidPT golden is compared against them distributionally.
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

from paper_1703_01506_b200.datagen import CONFIGS, make_data_numpy  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    ap.add_argument("--out", default=os.path.join(HERE, "c2_naive_reference.npz"))
    args = ap.parse_args()
    cfg = CONFIGS["c2"]
    vals = make_data_numpy(cfg)
    x = R.DataMatrix(vals, cfg.n1, cfg.n2)
    plan = R.PermutationPlan(cfg.plan_seed, cfg.permutations, cfg.subjects)
    t0 = time.time()
    null, _, counters = R.run_naive(x, plan, two_sided=cfg.two_sided, threads=args.threads)
    dt = time.time() - t0
    print(f"run_naive {dt:.1f}s on {args.threads} threads, counters={counters}", flush=True)
    np.savez_compressed(
        args.out,
        maxima=np.asarray(null.maxima, dtype=np.float64),
        counters=np.array(json.dumps(counters)),
        seconds=np.float64(dt),
        threads=np.int64(args.threads),
        data_sha=np.array(hashlib.sha256(np.ascontiguousarray(vals).tobytes()).hexdigest()),
        numpy_version=np.array(np.__version__),
    )
    print("wrote", args.out, flush=True)


if __name__ == "__main__":
    main()
