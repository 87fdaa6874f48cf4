"""Wall-time breakdown of run_rapid at a BASELINE config (host RNG draws,
transfers, device phases), for finding host-side overheads.
usage: rapid_phases.py [--config c5] [--after-naive]"""
import argparse
import functools
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    args = ap.parse_args()
    import torch

    import paper_1703_01506_b200 as rmx
    from paper_1703_01506_b200 import rapid_engine as re
    from paper_1703_01506_b200.datagen import CONFIGS, make_data_torch

    acc = {}

    def wrap(mod, name):
        f = getattr(mod, name)

        @functools.wraps(f)
        def g(*a, **k):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = f(*a, **k)
            torch.cuda.synchronize()
            acc[name] = acc.get(name, 0.0) + time.perf_counter() - t0
            return r
        setattr(mod, name, g)

    for nm in ("_lsq_tc", "_complete_max"):
        if hasattr(re, nm):
            wrap(re, nm)
    cfg0 = CONFIGS[args.config]
    dev = torch.device("cuda", 0)
    x = rmx.DataMatrix(make_data_torch(cfg0, dev).to(torch.float32).cpu().numpy(), cfg0.n1, cfg0.n2)
    rc = rmx.RunConfig(permutations=cfg0.permutations, seed=cfg0.plan_seed, engine="rapid",
                       training_columns=cfg0.training_columns, rank=cfg0.rank,
                       sample_rate=cfg0.sample_rate, max_passes=50)
    from paper_1703_01506_b200.datagen import scaled
    cw = scaled(cfg0, (64, 64, 32), 2048)  # warm-up: kernels, allocator
    xw = rmx.DataMatrix(make_data_torch(cw, dev).to(torch.float32).cpu().numpy(), cw.n1, cw.n2)
    rmx.run_rapid(xw, rmx.RunConfig(permutations=2048, seed=cw.plan_seed, engine="rapid",
                                    training_columns=cw.training_columns, rank=cw.rank,
                                    sample_rate=cw.sample_rate, max_passes=1))
    acc.clear()
    torch.cuda.synchronize()
    re._PHASE_LOG = []
    t0 = time.perf_counter()
    null, model, counters = rmx.run_rapid(x, rc)
    torch.cuda.synchronize()
    print(json.dumps({"total_s": time.perf_counter() - t0, "train_s": counters["train_seconds"],
                      "recover_s": counters["recover_seconds"],
                      "phases_s": {k: round(v, 3) for k, v in acc.items()},
                      "train_marks_s": [(tag, round(t - t0, 3)) for tag, t in re._PHASE_LOG]}))


if __name__ == "__main__":
    main()
