import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1703_01506_b200 import _native as nat
from paper_1703_01506_b200 import rapid_engine as re
dev = torch.device("cuda", 0)
u = torch.randn(524288, 400, dtype=torch.float64, device=dev) / 724.0
for _ in range(3):
    d = ctypes.c_double(0)
    torch.cuda.synchronize()
    nat.call("rmx_orthonormalize", nat.ptr(u), 524288, 400, 0, ctypes.byref(d), re._stream(dev))
torch.cuda.synchronize()
print("drift", d.value)
