"""Time the host-buffer NaivePT path against the plain H2D copy of X
(diagnostics only).  usage: e2e_probe.py [c4|c2]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import json

    import numpy as np
    import torch

    import paper_1703_01506_b200 as rmx
    from paper_1703_01506_b200 import hostmem
    from paper_1703_01506_b200.datagen import CONFIGS, make_data_torch

    cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
    dev = torch.device("cuda", 0)
    x = rmx.DataMatrix(make_data_torch(cfg, dev).cpu().numpy(), cfg.n1, cfg.n2)
    plan = rmx.PermutationPlan(cfg.plan_seed, cfg.permutations, cfg.subjects)
    xh = hostmem.pinned(np.asarray(x.values, dtype=np.float64))
    xd = torch.empty(xh.shape, dtype=torch.float64, device=dev)
    ht = torch.from_numpy(xh)
    h2d = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        xd.copy_(ht, non_blocking=True)
        torch.cuda.synchronize()
        h2d.append(time.perf_counter() - t0)
    del xd
    runs = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = rmx.run_naive_ex(x, plan, two_sided=cfg.two_sided)
        torch.cuda.synchronize()
        runs.append(time.perf_counter() - t0)
    print(json.dumps({"config": cfg.name if hasattr(cfg, "name") else sys.argv[1:],
                      "x_bytes": xh.nbytes, "h2d_ms": [1e3 * t for t in h2d],
                      "h2d_GBps": xh.nbytes / min(h2d) / 1e9,
                      "run_naive_ex_ms": [1e3 * t for t in runs],
                      "chunks": int(res.stats["chunks"]) if isinstance(res.stats, dict) and "chunks" in res.stats else None,
                      "env_chunks_min": os.environ.get("RMX_CHUNKS_MIN")}))


if __name__ == "__main__":
    main()
