"""ctypes binding of librmx.so (include/rmx.h).

This module is the only door into the CUDA engine.  There is no CPU
fallback: if the library or a B200 device is missing, every call raises
``EngineUnavailableError``.  Status codes are mapped onto the reference's
exception hierarchy (see exceptions.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

from .exceptions import (
    DataFormatError,
    DegenerateVoxelError,
    EngineUnavailableError,
    IllConditionedBasisError,
    NumericalError,
    UsageError,
)

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "librmx.so")
CSRC = os.path.join(_PKG, "csrc")

(RMX_OK, RMX_E_USAGE, RMX_E_DEGENERATE, RMX_E_ILLCOND, RMX_E_CUDA, RMX_E_NUMERIC, RMX_E_FORMAT,
 RMX_E_IO) = range(8)


class Status(ctypes.Structure):
    _fields_ = [
        ("code", ctypes.c_int32),
        ("_pad", ctypes.c_int32),
        ("perm", ctypes.c_int64),
        ("voxel", ctypes.c_int64),
        ("value", ctypes.c_double),
        ("msg", ctypes.c_char * 256),
    ]


class NaiveStats(ctypes.Structure):
    _fields_ = [
        ("suspects", ctypes.c_int64),
        ("band_candidates", ctypes.c_int64),
        ("overflow_perms", ctypes.c_int64),
        ("chunks", ctypes.c_int32),
        ("grid", ctypes.c_int32),
        ("stages", ctypes.c_int32),
        ("bk", ctypes.c_int32),
        ("rare_groups", ctypes.c_int64),
        ("all_groups", ctypes.c_int64),
        ("cg", ctypes.c_int32),
        ("i8", ctypes.c_int32),
    ]

    def as_dict(self) -> dict:
        return {name: int(getattr(self, name)) for name, _ in self._fields_}


class Mat0Info(ctypes.Structure):
    _fields_ = [("magic", ctypes.c_uint8 * 8), ("version", ctypes.c_uint32),
                ("_pad", ctypes.c_uint32), ("rows", ctypes.c_int64), ("cols", ctypes.c_int64),
                ("n1", ctypes.c_int64), ("n2", ctypes.c_int64),
                ("header_bytes", ctypes.c_int64), ("file_bytes", ctypes.c_int64)]


# Every symbol include/rmx.h declares (tests check the library exports them).
EXPORTS = (
    "rmx_abi_version",
    "rmx_device_check",
    "rmx_host_register",
    "rmx_host_unregister",
    "rmx_upload_staged",
    "rmx_naive_workspace_bytes",
    "rmx_naive_maxnull",
    "rmx_naive_maxnull_host",
    "rmx_naive_maxnull_host_plan",
    "rmx_naive_maxnull_host_f32",
    "rmx_naive_maxnull_host_plan_f32",
    "rmx_naive_maxnull_host_plan_range",
    "rmx_naive_maxnull_host_plan_range_f32",
    "rmx_plan_orders",
    "rmx_omega_draws",
    "rmx_naive_prepare",
    "rmx_naive_tfill",
    "rmx_naive_finish",
    "rmx_naive_tfill_debug",
    "rmx_tstat_exact",
    "rmx_tstat_pairs",
    "rmx_rapid_stats",
    "rmx_lsq_workspace_bytes",
    "rmx_lsq_solve",
    "rmx_lsq_solve_tc",
    "rmx_lsq_solve_tc_settle",
    "rmx_lsq_solve_exact",
    "rmx_track_update",
    "rmx_normal_tables_set",
    "rmx_standard_normal",
    "rmx_standard_normal_rows",
    "rmx_normal_stream_open",
    "rmx_normal_stream_fill",
    "rmx_normal_stream_close",
    "rmx_normal_stream_fill_device",
    "rmx_complete_max",
    "rmx_to_f32",
    "rmx_row_max",
    "rmx_resid_batch",
    "rmx_gather_rows",
    "rmx_gemv",
    "rmx_mean_var",
    "rmx_orthonormalize",
    "rmx_grouse_train",
    "rmx_mat0_header",
    "rmx_mat0_read",
    "rmx_mat0_write",
    "rmx_mat0_read_rows",
    "rmx_mat0_create",
    "rmx_mat0_write_rows",
    "rmx_naive_maxnull_mat0",
    "rmx_tstat_dump_mat0",
)



_lib = None

# int (*)(void* user, int32 col, int32 pass, int32 attempt, int32* omega_out)
OMEGA_CB = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32,
                            ctypes.c_int32, ctypes.POINTER(ctypes.c_int32))

_i64, _i32, _vp, _sz = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_size_t
_SP = ctypes.POINTER(Status)
_NP = ctypes.POINTER(NaiveStats)

_SIGS = {
    "rmx_abi_version": ([], ctypes.c_int),
    "rmx_device_check": ([ctypes.c_int, ctypes.POINTER(_i32), _SP], ctypes.c_int),
    "rmx_host_register": ([_vp, _sz], ctypes.c_int),
    "rmx_host_unregister": ([_vp], ctypes.c_int),
    "rmx_upload_staged": ([_vp, _sz, _vp, _vp, _sz, _vp, _SP], ctypes.c_int),
    "rmx_naive_workspace_bytes": ([_i64, _i32, _i64], _sz),
    "rmx_naive_maxnull": ([_vp, _i64, _i32, _i32, _vp, _i64, _i32, _vp, _vp, _vp, _sz, _vp, _SP, _NP],
                          ctypes.c_int),
    "rmx_naive_maxnull_host": ([_vp, _i64, _i32, _i32, _vp, _i64, _i32, _vp, _vp, _vp, _vp, _vp,
                                _vp, _vp, _sz, _vp, _SP, _NP], ctypes.c_int),
    "rmx_naive_maxnull_host_plan": ([_vp, _i64, _i32, _i32, ctypes.c_uint64, _i64, _i32, _vp, _vp,
                                     _vp, _vp, _vp, _vp, _vp, _sz, _vp, _SP, _NP], ctypes.c_int),
    "rmx_naive_maxnull_host_f32": ([_vp, _i64, _i32, _i32, _vp, _i64, _i32, _vp, _vp, _vp, _vp,
                                    _vp, _vp, _vp, _vp, _sz, _vp, _SP, _NP], ctypes.c_int),
    "rmx_naive_maxnull_host_plan_f32": ([_vp, _i64, _i32, _i32, ctypes.c_uint64, _i64, _i32, _vp,
                                         _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp, _SP, _NP],
                                        ctypes.c_int),
    "rmx_naive_maxnull_host_plan_range": ([_vp, _i64, _i32, _i32, ctypes.c_uint64, _i64, _i64, _i32,
                                           _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp, _SP, _NP],
                                          ctypes.c_int),
    "rmx_naive_maxnull_host_plan_range_f32": ([_vp, _i64, _i32, _i32, ctypes.c_uint64, _i64, _i64,
                                               _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz,
                                               _vp, _SP, _NP], ctypes.c_int),
    "rmx_plan_orders": ([ctypes.c_uint64, _i64, _i64, _i32, _vp, _vp, _SP], ctypes.c_int),
    "rmx_omega_draws": ([ctypes.c_uint64, _i32, _i64, _i64, _i64, _i64, _i32, _vp, _vp, _SP],
                        ctypes.c_int),
    "rmx_naive_prepare": ([_vp, _i64, _i32, _i32, _i64, _vp, _sz, _vp, _SP], ctypes.c_int),
    "rmx_naive_tfill": ([_i64, _i32, _i32, _vp, _i64, _i32, _vp, _sz, _vp, _SP, _NP], ctypes.c_int),
    "rmx_naive_finish": ([_vp, _i64, _i32, _i32, _vp, _i64, _i32, _vp, _vp, _vp, _sz, _vp, _SP, _NP],
                         ctypes.c_int),
    "rmx_naive_tfill_debug": ([_i64, _i32, _i32, _vp, _i64, _i32, _vp, _vp, _sz, _vp, _SP],
                              ctypes.c_int),
    "rmx_tstat_exact": ([_vp, _i64, _i32, _i32, _vp, _i64, _vp, _i64, _vp, _SP], ctypes.c_int),
    "rmx_tstat_pairs": ([_vp, _i64, _i32, _i32, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _SP],
                        ctypes.c_int),
    "rmx_rapid_stats": ([_vp, _i64, _i32, _i32, _vp, _vp, _i64, _i32, _vp, _vp, _SP], ctypes.c_int),
    "rmx_lsq_workspace_bytes": ([_i32, _i64], _sz),
    "rmx_mat0_header": ([ctypes.c_char_p, ctypes.POINTER(Mat0Info), _SP], ctypes.c_int),
    "rmx_mat0_read": ([ctypes.c_char_p, _i64, _i64, _vp, _i32, ctypes.POINTER(_i64), _SP],
                      ctypes.c_int),
    "rmx_mat0_write": ([ctypes.c_char_p, _vp, _i64, _i64, _i64, _i64, _SP], ctypes.c_int),
    "rmx_mat0_read_rows": ([ctypes.c_char_p, _i64, _i64, _i64, _vp, _i32, ctypes.POINTER(_i64),
                            _SP], ctypes.c_int),
    "rmx_mat0_create": ([ctypes.c_char_p, _i64, _i64, _i64, _i64, _SP], ctypes.c_int),
    "rmx_mat0_write_rows": ([ctypes.c_char_p, _i64, _i64, _i64, _vp, _i32, _SP], ctypes.c_int),
    "rmx_naive_maxnull_mat0": ([ctypes.c_char_p, _i64, _i32, _i32, ctypes.c_uint64, _i64, _i64,
                                _i32, _vp, _vp, _vp, _sz, _i32, ctypes.POINTER(_i64), _vp, _vp,
                                _vp, _vp, _vp, _sz, _vp, _SP, _NP], ctypes.c_int),
    "rmx_tstat_dump_mat0": ([_vp, _i64, _i32, _i32, _vp, _i64, ctypes.c_char_p, _vp, _sz, _i32,
                             _vp, _SP], ctypes.c_int),
    "rmx_lsq_solve_tc": ([_vp, _i64, _i64, _i32, _vp, _i32, _vp, _i64, _vp, _vp, _vp, _sz, _vp, _vp,
                          _SP], ctypes.c_int),
    "rmx_lsq_solve_tc_settle": ([_vp, _i64, _i64, _i32, _vp, _i32, _vp, _i64, _vp, _vp, _vp, _sz,
                                 _vp, ctypes.c_double, _vp, _SP], ctypes.c_int),
    "rmx_lsq_solve": ([_vp, _i64, _i32, _vp, _i32, _vp, _i64, _vp, _vp, _vp, _vp, _sz, _vp, _SP],
                      ctypes.c_int),
    "rmx_lsq_solve_exact": ([_vp, _i64, _i32, _vp, _i32, _vp, _i64, _vp, _vp, _vp, _vp, _SP],
                            ctypes.c_int),
    "rmx_track_update": ([_vp, _i64, _i32, _vp, _i32, _vp, ctypes.c_double,
                          ctypes.POINTER(ctypes.c_double), _vp, _SP], ctypes.c_int),
    "rmx_normal_tables_set": ([_vp, _vp, _vp], ctypes.c_int),
    "rmx_standard_normal": ([ctypes.c_uint64, _vp, _i32, _i64, _vp, _SP], ctypes.c_int),
    "rmx_standard_normal_rows": ([ctypes.c_uint64, ctypes.c_uint32, _i64, _i64, _i64, _vp, _vp,
                                  _i32, _SP], ctypes.c_int),
    "rmx_normal_stream_open": ([ctypes.c_uint64, _vp, _i32, ctypes.POINTER(_vp), _SP],
                               ctypes.c_int),
    "rmx_normal_stream_fill": ([_vp, _i64, _vp], ctypes.c_int),
    "rmx_normal_stream_close": ([_vp], ctypes.c_int),
    "rmx_normal_stream_fill_device": ([_vp, _i64, _vp, _vp, _i64, _vp, _SP], ctypes.c_int),
    "rmx_complete_max": ([_vp, _i64, _i32, _vp, _i64, _i64, ctypes.c_double, ctypes.c_double,
                          ctypes.c_uint64, _i32, _vp, _vp, _vp, _vp, _SP], ctypes.c_int),
    "rmx_to_f32": ([_vp, _i64, _vp, _vp, _SP], ctypes.c_int),
    "rmx_row_max": ([_vp, _i64, _i64, _i32, _vp, _vp, _SP], ctypes.c_int),
    "rmx_resid_batch": ([_vp, _i32, _vp, _i32, _vp, _vp, _i64, _vp, _vp, _SP], ctypes.c_int),
    "rmx_gather_rows": ([_vp, _i64, _vp, _i32, _i64, _vp, _vp, _SP], ctypes.c_int),
    "rmx_gemv": ([_vp, _i64, _i32, _vp, _vp, _vp, _SP], ctypes.c_int),
    "rmx_mean_var": ([_vp, _i64, _vp, _vp, _SP], ctypes.c_int),
    "rmx_orthonormalize": ([_vp, _i64, _i32, _i32, ctypes.POINTER(ctypes.c_double), _vp, _SP],
                           ctypes.c_int),
    "rmx_grouse_train": ([_vp, _i64, _i32, _i32, _i32, _vp, _i32, ctypes.c_double, _vp, OMEGA_CB,
                          _vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_i32),
                          ctypes.POINTER(_i32), ctypes.POINTER(_i64), _vp, _vp, _SP],
                         ctypes.c_int),
}


def build(force: bool = False) -> str:
    """Compile librmx.so in-tree (nvcc, sm_100a)."""
    cmd = ["make", "-s", "-C", CSRC]
    if force:
        subprocess.run(["make", "-s", "-C", CSRC, "clean"], check=True)
    subprocess.run(cmd, check=True)
    return LIB_PATH


def load() -> ctypes.CDLL:
    """Load librmx.so; raises EngineUnavailableError (never falls back)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise EngineUnavailableError(
            f"{LIB_PATH} is missing: build it with `make -C {CSRC}` (nvcc, sm_100a); "
            "there is no CPU fallback"
        )
    lib = ctypes.CDLL(LIB_PATH)
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def raise_for(rc: int, st: Status) -> None:
    if rc == RMX_OK:
        return
    msg = st.msg.decode(errors="replace")
    if rc == RMX_E_USAGE:
        raise UsageError(msg)
    if rc == RMX_E_DEGENERATE:
        raise DegenerateVoxelError(int(st.voxel), float(st.value))
    if rc == RMX_E_ILLCOND:
        raise IllConditionedBasisError(float(st.value))
    if rc == RMX_E_FORMAT:
        raise DataFormatError(msg)
    if rc == RMX_E_IO:
        raise OSError(msg)
    raise NumericalError(f"librmx error {rc}: {msg}")


def ptr(t) -> int | None:
    return None if t is None else int(t.data_ptr())


def stream_handle(stream) -> int:
    return int(stream.cuda_stream)


def call(name: str, *args) -> None:
    """Invoke an rmx_* entry point whose last argument is rmx_status*."""
    st = Status()
    rc = getattr(load(), name)(*args, ctypes.byref(st))
    raise_for(rc, st)


def device_check(device: int = 0) -> int:
    lib = load()
    st = Status()
    sms = _i32(0)
    rc = lib.rmx_device_check(device, ctypes.byref(sms), ctypes.byref(st))
    if rc != RMX_OK:
        raise EngineUnavailableError(st.msg.decode(errors="replace"))
    return int(sms.value)
