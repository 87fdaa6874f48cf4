"""Diagnostics: run_rapid at a config with live phase marks and periodic
Python stack dumps (faulthandler) -- for finding where a run stalls.
usage: diag_rapid.py [--config c5] [--perms L] [--passes P] [--dump-every S]"""
import argparse
import faulthandler
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


class LiveLog(list):
    def __init__(self, t0):
        super().__init__()
        self.t0 = t0

    def append(self, item):
        super().append(item)
        print(f"[mark] {item[0]} {item[1] - self.t0:.3f}s", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--perms", type=int, default=0)
    ap.add_argument("--passes", type=int, default=0)
    ap.add_argument("--dump-every", type=float, default=60.0)
    args = ap.parse_args()
    faulthandler.dump_traceback_later(args.dump_every, repeat=True, file=sys.stderr)
    import torch

    import paper_1703_01506_b200 as rmx
    from paper_1703_01506_b200 import rapid_engine as re
    from paper_1703_01506_b200.datagen import CONFIGS, make_data_torch

    cfg0 = CONFIGS[args.config]
    L = args.perms or cfg0.permutations
    dev = torch.device("cuda", 0)
    t0 = time.perf_counter()
    x = rmx.DataMatrix(make_data_torch(cfg0, dev).to(torch.float32).cpu().numpy(), cfg0.n1,
                       cfg0.n2)
    print(f"data {time.perf_counter() - t0:.2f}s", flush=True)
    rc = rmx.RunConfig(permutations=L, seed=cfg0.plan_seed, engine="rapid",
                       training_columns=cfg0.training_columns, rank=cfg0.rank,
                       sample_rate=cfg0.sample_rate, max_passes=args.passes or 50)
    t0 = time.perf_counter()
    re._PHASE_LOG = LiveLog(t0)
    null, model, counters = rmx.run_rapid(x, rc)
    torch.cuda.synchronize()
    print(f"run_rapid {time.perf_counter() - t0:.2f}s passes={model.passes} "
          f"sigma={model.residual_std} mu={model.max_shift} counters={counters}", flush=True)


if __name__ == "__main__":
    main()
