"""Time RapidPT phases (train / recover) on a BASELINE.json config.
usage: bench_rapid.py --config c3|c5 [--perms L] [--passes P]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--perms", type=int, default=0)
    ap.add_argument("--passes", type=int, default=0, help="override max_passes (0 = 50)")
    args = ap.parse_args()
    import torch

    import paper_1703_01506_b200 as rmx
    from paper_1703_01506_b200 import rapid_engine as re
    from paper_1703_01506_b200.datagen import CONFIGS, make_data_torch

    cfg0 = CONFIGS[args.config]
    L = args.perms or cfg0.permutations
    dev = torch.device("cuda", 0)
    x = rmx.DataMatrix(make_data_torch(cfg0, dev).cpu().numpy(), cfg0.n1, cfg0.n2)
    cfg = rmx.RunConfig(permutations=L, seed=cfg0.plan_seed, engine="rapid",
                        training_columns=cfg0.training_columns, rank=cfg0.rank,
                        sample_rate=cfg0.sample_rate,
                        max_passes=args.passes or 50)
    plan = cfg.plan_for(x)
    from paper_1703_01506_b200.labels import plan_orders
    t0 = time.perf_counter()
    plan_orders(plan)
    re.draw_omegas(cfg.seed, 3, cfg.training_columns, L, x.voxels,
                   int(-(-cfg.sample_rate * x.voxels // 1)))
    t_inputs = time.perf_counter() - t0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    model, _, _, pre = re._train_device(x, cfg, prefetch_recovery=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    null, counters = re.recover(x, model, plan, cfg, _pre=pre)
    model.basis.matrix  # host copy of the basis (overlapped with recovery)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(json.dumps({"config": args.config, "L": L, "v": x.voxels, "passes": model.passes,
                      "train_s": t1 - t0, "recover_s": t2 - t1,
                      "T_entries_per_s": L * x.voxels / (t2 - t0), "sigma": model.residual_std,
                      "mu": model.max_shift, "counters": counters,
                      "host_input_gen_s_first_call": t_inputs,
                      "max_head": null.maxima[:5].tolist()}))


if __name__ == "__main__":
    main()
