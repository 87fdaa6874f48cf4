import time, numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_1703_01506_b200.rng import stream
v, r = 524288, 400
dev = torch.device('cuda', 0); torch.ones(1, device=dev)
t = time.perf_counter(); a = stream(5, 5).standard_normal((v, r)); print('single', time.perf_counter() - t)
del a
rows = (32 << 20) // (8 * r)
bufs = [torch.empty((rows, r), dtype=torch.float64, pin_memory=True) for _ in range(2)]
g = stream(5, 5); t = time.perf_counter()
for c, lo in enumerate(range(0, v, rows)):
    hi = min(v, lo + rows); g.standard_normal(out=bufs[c & 1].numpy()[:hi - lo])
print('chunked-pinned', time.perf_counter() - t)
h = np.empty((rows, r)); g = stream(5, 5); t = time.perf_counter()
for c, lo in enumerate(range(0, v, rows)):
    hi = min(v, lo + rows); g.standard_normal(out=h[:hi - lo])
print('chunked-pageable', time.perf_counter() - t)
g = stream(5, 5); t = time.perf_counter()
for c, lo in enumerate(range(0, v, rows)):
    hi = min(v, lo + rows); g.standard_normal(size=(hi - lo, r))
print('chunked-alloc', time.perf_counter() - t)
import numpy.random as npr
print(np.__version__)
