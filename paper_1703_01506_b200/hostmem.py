"""Host <-> device transfers for the drop-in entry points.

The reference API hands us numpy arrays (DataMatrix.values is a read-only
float64 array).  Copying 1.7 GB through a fresh pinned staging buffer per
call would cost more than the GPU work, so arrays are page-locked in place
with cudaHostRegister (once per array object; unregistered when the array is
garbage-collected) and copied with cudaMemcpyAsync at full PCIe/NVLink-C2C
rate.  Small arrays just go through torch's pinned allocator.
"""

from __future__ import annotations

import threading
import warnings
import weakref

import numpy as np

_REGISTERED: dict = {}
_LOCK = threading.Lock()
_MIN_REGISTER_BYTES = 64 << 20


def _unregister(ptr: int) -> None:
    import torch

    with _LOCK:
        if _REGISTERED.pop(ptr, None) is not None:
            try:
                torch.cuda.cudart().cudaHostUnregister(ptr)
            except Exception:  # interpreter shutdown
                pass


def _as_tensor(arr: np.ndarray):
    import torch

    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)
        return torch.from_numpy(arr)


def to_device(arr: np.ndarray, device, stream=None):
    """Copy a C-contiguous numpy array to `device` (async on `stream`)."""
    import torch

    arr = np.ascontiguousarray(arr)
    if arr.nbytes >= _MIN_REGISTER_BYTES:
        ptr = arr.ctypes.data
        with _LOCK:
            known = ptr in _REGISTERED and _REGISTERED[ptr][0]() is arr
        if not known:
            rc = torch.cuda.cudart().cudaHostRegister(ptr, arr.nbytes, 0)
            if int(rc) == 0:
                with _LOCK:
                    _REGISTERED[ptr] = (weakref.ref(arr, lambda _r, p=ptr: _unregister(p)),)
                known = True
        host = _as_tensor(arr)
    else:
        host = _as_tensor(arr).pin_memory()
    out = torch.empty(arr.shape, dtype=host.dtype, device=device)
    s = stream if stream is not None else torch.cuda.current_stream(device)
    with torch.cuda.stream(s):
        out.copy_(host, non_blocking=True)
    return out
