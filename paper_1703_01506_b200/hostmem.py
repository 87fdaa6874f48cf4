"""Host <-> device transfers for the drop-in entry points.

The reference API hands us numpy arrays (DataMatrix.values is a read-only
float64 array).  Copying 1.7 GB through a fresh pinned staging buffer per
call would cost more than the GPU work, so arrays are page-locked in place
with cudaHostRegister (once per array object; unregistered when the array is
garbage-collected) and copied with cudaMemcpyAsync at full PCIe/NVLink-C2C
rate.  Small arrays just go through torch's pinned allocator.
"""

from __future__ import annotations

import ctypes
import threading
import warnings
import weakref

import numpy as np

_REGISTERED: dict = {}
# re-entrant: dropping the last reference to a registered array (e.g. an
# _INFLIGHT entry pruned under the lock) runs its weakref callback, which
# takes the lock again on the same thread
_LOCK = threading.RLock()
_MIN_REGISTER_BYTES = 64 << 20


def _lib():
    from . import _native

    return _native.load()


def _unregister(ptr: int) -> None:
    with _LOCK:
        if _REGISTERED.pop(ptr, None) is not None:
            try:
                _lib().rmx_host_unregister(ptr)
            except Exception:  # interpreter shutdown
                pass


def _as_tensor(arr: np.ndarray):
    import torch

    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)
        return torch.from_numpy(arr)


def _owner(arr: np.ndarray) -> np.ndarray:
    """The ndarray that owns `arr`'s memory (views -- e.g. the label cache's
    row slices -- share one registration with their owner)."""
    root = arr
    while isinstance(root.base, np.ndarray):
        root = root.base
    lo, hi = root.ctypes.data, root.ctypes.data + root.nbytes
    if root.flags["C_CONTIGUOUS"] and lo <= arr.ctypes.data and arr.ctypes.data + arr.nbytes <= hi:
        return root
    return arr


def _register(arr: np.ndarray) -> bool:
    """Page-lock a (large, C-contiguous) array's memory in place, once per
    owning array (unregistered when the owner is garbage-collected)."""
    owner = _owner(arr)
    ptr = owner.ctypes.data
    with _LOCK:
        if ptr in _REGISTERED and _REGISTERED[ptr][0]() is owner:
            return True
    rc = _lib().rmx_host_register(ptr, owner.nbytes)  # ctypes: the GIL is released
    if int(rc) != 0:
        return False
    with _LOCK:
        _REGISTERED[ptr] = (weakref.ref(owner, lambda _r, p=ptr: _unregister(p)),)
    return True


def pinned(arr: np.ndarray) -> np.ndarray:
    """A C-contiguous, page-locked view (large arrays, registered in place) or
    copy (small arrays) of `arr`, for asynchronous host->device copies.  When
    registration is refused the contiguous pageable array is returned (copies
    then serialise but stay correct)."""
    arr = np.ascontiguousarray(arr)
    if arr.nbytes >= _MIN_REGISTER_BYTES:
        _register(arr)
        return arr
    out = pinned_empty(arr.shape, arr.dtype)
    out[...] = arr
    return out


def pinned_empty(shape, dtype) -> np.ndarray:
    """A page-locked host array (torch's pinned allocator)."""
    import torch

    t = torch.empty(tuple(int(s) for s in shape), dtype=_torch_dtype(np.dtype(dtype)),
                    pin_memory=True)
    return t.numpy()


def _torch_dtype(dt: np.dtype):
    import torch

    return {np.dtype(np.float64): torch.float64, np.dtype(np.float32): torch.float32,
            np.dtype(np.int16): torch.int16, np.dtype(np.int32): torch.int32,
            np.dtype(np.int64): torch.int64, np.dtype(np.uint8): torch.uint8}[dt]


# (host array, CUDA event) of asynchronous copies out of memory registered in
# place: torch does not track the lifetime of memory it did not allocate, so
# the source (and its registration) is kept alive here until the copy has
# completed -- otherwise a temporary passed by a caller could be freed, and
# unregistered, while the DMA still reads it.
_INFLIGHT: list = []


def _prune_inflight() -> None:
    done, keep = [], []
    with _LOCK:
        for item in _INFLIGHT:
            (done if item[1].query() else keep).append(item)
        _INFLIGHT[:] = keep
    del done  # the sources' last references (and their unregistration) go outside the lock


def to_device(arr: np.ndarray, device, stream=None):
    """Copy a C-contiguous numpy array to `device` (async on `stream`)."""
    import torch

    _prune_inflight()
    arr = np.ascontiguousarray(arr)
    registered = arr.nbytes >= _MIN_REGISTER_BYTES and _register(arr)
    host = _as_tensor(arr) if registered else _as_tensor(arr).pin_memory()
    out = torch.empty(arr.shape, dtype=host.dtype, device=device)
    s = stream if stream is not None else torch.cuda.current_stream(device)
    with torch.cuda.stream(s):
        out.copy_(host, non_blocking=True)
        if registered:
            ev = torch.cuda.Event()
            ev.record(s)
            with _LOCK:
                _INFLIGHT.append((arr, ev))
    return out


def wait_inflight() -> None:
    """Block until every in-place-registered source copy has completed."""
    with _LOCK:
        pending = list(_INFLIGHT)
    for _, ev in pending:
        ev.synchronize()
    _prune_inflight()


_STAGE: dict = {}
_STAGE_LOCK = threading.Lock()


def upload_staged(arr: np.ndarray, device, stream=None):
    """One-shot upload of a (large, pageable) array without page-locking it:
    through a cached 2 x 32 MB page-locked ring (rmx_upload_staged, one
    native call, the GIL released).  An array that is already registered
    goes straight through to_device."""
    import torch

    from . import _native as nat

    arr = np.ascontiguousarray(arr)
    owner = _owner(arr)
    with _LOCK:
        registered = owner.ctypes.data in _REGISTERED
    if registered or arr.nbytes < _MIN_REGISTER_BYTES:
        return to_device(arr, device, stream)
    out = torch.empty(arr.shape, dtype=_torch_dtype(arr.dtype), device=device)
    s = stream if stream is not None else torch.cuda.current_stream(device)
    st = nat.Status()
    with _STAGE_LOCK:  # one ring: uploads from different host threads take turns
        ring = _STAGE.get("ring")
        if ring is None:
            ring = pinned_empty((64 << 20,), np.uint8)
            _STAGE["ring"] = ring
        rc = nat.load().rmx_upload_staged(arr.ctypes.data, arr.nbytes, out.data_ptr(),
                                          ring.ctypes.data, ring.nbytes, nat.stream_handle(s),
                                          ctypes.byref(st))
    nat.raise_for(rc, st)
    return out
