"""Diagnostics: rmx_normal_stream_fill_device alone (no other host / GPU work)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["RMX_TRACE_BASIS"] = "1"
import numpy as np, torch
from paper_1703_01506_b200.normals import NormalStream
from paper_1703_01506_b200.rng import BASIS_INIT
from paper_1703_01506_b200.hostmem import pinned_empty
from paper_1703_01506_b200 import _native as nat
nat.load()
dev = torch.device("cuda", 0)
torch.zeros(1, device=dev)
for ring_doubles in (1 << 21, 1 << 23):
    out = torch.empty((524288, 400), dtype=torch.float64, device=dev)
    ring = pinned_empty((ring_doubles,), np.float64)
    side = torch.cuda.Stream(dev)
    g = NormalStream(1703015065, (BASIS_INIT,))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g.fill_device(out, ring, side)
    print(f"ring {ring_doubles * 8 >> 20} MB: fill_device alone {time.perf_counter() - t0:.3f} s", flush=True)
    g.close()
