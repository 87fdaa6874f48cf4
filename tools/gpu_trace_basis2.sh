python - <<'PY'
import time, numpy as np, torch
from paper_1703_01506_b200.normals import NormalStream
from paper_1703_01506_b200.rng import BASIS_INIT
from paper_1703_01506_b200.hostmem import pinned_empty
dev=torch.device('cuda',0); out=torch.empty((524288,400),dtype=torch.float64,device=dev)
ring=pinned_empty((1<<21,), np.float64); side=torch.cuda.Stream(dev)
for rep in range(2):
    g=NormalStream(1703015065,(BASIS_INIT,)); t0=time.perf_counter(); g.fill_device(out, ring, side); g.close()
    print('fill_device alone: %.3f s'%(time.perf_counter()-t0), flush=True)
buf=np.empty(1<<20); g=NormalStream(1703015065,(BASIS_INIT,)); t0=time.perf_counter()
for i in range(200): g.fill(buf)
print('fill host alone: %.3f s'%(time.perf_counter()-t0)); g.close()
import os; print('cpus', os.cpu_count(), open('/proc/cpuinfo').read().count('processor'))
print([l for l in open('/proc/cpuinfo').read().splitlines() if 'model name' in l][:1])
PY
