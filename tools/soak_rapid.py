"""Bit-reproducibility soak of run_rapid at config-3 / config-5 shapes: the
three-stream look-ahead GROUSE chain is ordered by events only, so repeated
runs must give the same basis and maxima bit for bit.
usage: soak_rapid.py [--reps 4]"""
import argparse
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=4)
    args = ap.parse_args()
    import numpy as np
    import torch

    import paper_1703_01506_b200 as rmx
    from paper_1703_01506_b200.datagen import CONFIGS, make_data_torch

    dev = torch.device("cuda", 0)
    ok = True
    for name, L, passes in (("c3", 4000, 50), ("c5", 6000, 12)):
        cfg0 = CONFIGS[name]
        x = rmx.DataMatrix(make_data_torch(cfg0, dev).to(torch.float32).cpu().numpy(),
                           cfg0.n1, cfg0.n2)
        rc = rmx.RunConfig(permutations=L, seed=cfg0.plan_seed, engine="rapid",
                           training_columns=cfg0.training_columns, rank=cfg0.rank,
                           sample_rate=cfg0.sample_rate, max_passes=passes)
        seen = set()
        for rep in range(args.reps):
            null, model, _ = rmx.run_rapid(x, rc)
            u = np.ascontiguousarray(model.basis.matrix)
            h = (hashlib.sha256(u.tobytes()).hexdigest()[:16] + ":" +
                 hashlib.sha256(np.ascontiguousarray(null.maxima).tobytes()).hexdigest()[:16])
            seen.add(h)
            print(f"{name} run {rep}: basis:maxima {h} sigma {model.residual_std:.17g} "
                  f"mu {model.max_shift:.17g} passes {model.passes}", flush=True)
        ok = ok and len(seen) == 1
    print("bit-reproducible" if ok else "RUNS DIFFER")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
