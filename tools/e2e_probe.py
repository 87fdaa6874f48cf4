"""Time the host-buffer NaivePT path phase by phase (diagnostics only)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch

    import paper_1703_01506_b200 as rmx
    from paper_1703_01506_b200 import hostmem, naive_engine
    from paper_1703_01506_b200.datagen import CONFIGS, make_data_torch
    from paper_1703_01506_b200.labels import plan_orders

    cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
    dev = torch.device("cuda", 0)
    x = rmx.DataMatrix(make_data_torch(cfg, dev).cpu().numpy(), cfg.n1, cfg.n2)
    plan = rmx.PermutationPlan(cfg.plan_seed, cfg.permutations, cfg.subjects)
    orders = plan_orders(plan)
    for it in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        xh = hostmem.pinned(np.asarray(x.values, dtype=np.float64))
        oh = hostmem.pinned(np.asarray(plan_orders(plan), dtype=np.int16))
        t1 = time.perf_counter()
        mx, am, job = naive_engine._run_from_host(xh, cfg.n1, oh, cfg.two_sided, dev)
        t2 = time.perf_counter()
        t3 = time.perf_counter()
        res = rmx.run_naive_ex(x, plan, two_sided=cfg.two_sided)
        t4 = time.perf_counter()
        print(f"iter {it}: pin {1e3 * (t1 - t0):.1f} ms, call {1e3 * (t2 - t1):.1f} ms, "
              f"run_naive_ex {1e3 * (t4 - t3):.1f} ms, "
              f"registered={len(hostmem._REGISTERED)} x_ptr_reg={xh.ctypes.data in hostmem._REGISTERED} "
              f"o_ptr_reg={oh.ctypes.data in hostmem._REGISTERED} flags={x.values.flags['C_CONTIGUOUS']}",
              flush=True)
    # plain copy rate for reference
    xd = torch.empty(xh.shape, dtype=torch.float64, device=dev)
    ht = torch.from_numpy(xh)
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        xd.copy_(ht, non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"H2D {xh.nbytes / dt / 1e9:.1f} GB/s ({1e3 * dt:.1f} ms)")


if __name__ == "__main__":
    main()
