"""Run the NaivePT phases once per launch for ncu captures (no timing printed
as a benchmark number).  usage: profile_naive.py --config c4 [--repeat 2]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--repeat", type=int, default=2)
    ap.add_argument("--perms", type=int, default=0, help="override L (0 = config)")
    args = ap.parse_args()
    import torch

    from paper_1703_01506_b200.datagen import CONFIGS
    from paper_1703_01506_b200.datagen import make_data_torch
    from paper_1703_01506_b200.labels import generate_orders
    from paper_1703_01506_b200.naive_engine import NaiveJob

    cfg = CONFIGS[args.config]
    L = args.perms or cfg.permutations
    dev = torch.device("cuda", 0)
    x = make_data_torch(cfg, dev)
    orders = torch.from_numpy(generate_orders(cfg.plan_seed, 0, L, cfg.subjects)).to(dev)
    job = NaiveJob(x, cfg.n1, orders, cfg.two_sided)
    for _ in range(args.repeat):
        job.prepare()
        job.tfill()
        job.finish()
    torch.cuda.synchronize()
    print("stats", job.stats.as_dict())


if __name__ == "__main__":
    main()
