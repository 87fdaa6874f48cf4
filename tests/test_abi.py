"""The C-ABI library builds, loads and exports exactly what include/rmx.h
declares (no compute calls: this runs without a GPU)."""
import os
import re
import subprocess

from paper_1703_01506_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "rmx.h")).read()
    return set(re.findall(r"^(?:int|size_t)\s+(rmx_\w+)\s*\(", hdr, flags=re.M))


def test_header_and_binding_agree():
    assert declared_symbols() == set(_native.EXPORTS)


def test_library_exports_every_declared_symbol():
    _native.load()
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (rmx_\w+)", out))
    missing = declared_symbols() - exported
    assert not missing, missing


def test_abi_version_and_sm100_code():
    lib = _native.load()
    assert lib.rmx_abi_version() == 1
    sass = subprocess.run(["cuobjdump", "-sass", _native.LIB_PATH], capture_output=True,
                          text=True).stdout
    # tcgen05 MMA, TMA tile loads and TMEM loads are in the binary (sm_100a)
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass


def test_no_library_gemm_linked():
    """the GROUSE products are the engine's own kernels
    (csrc/dgemm.cu, k_gram), not cuBLAS: nothing links or imports it."""
    out = subprocess.run(["ldd", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "cublas" not in out.lower()
    und = subprocess.run(["nm", "-D", "--undefined-only", _native.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "cublas" not in und.lower()
