"""The reference's matrix files through the engine's native reader / writer
(rmx_mat0_*; paper_1703_01506_b200/matfiles.py), checked against files and
error messages produced by the reference itself (tests/golden/matio.npz,
made by tests/golden/make_golden.py).  Host-side: runs without a GPU."""
import os

import numpy as np
import pytest

import paper_1703_01506_b200 as rmx
from paper_1703_01506_b200 import matfiles as mf

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "matio.npz"))


def test_reference_file_reads_bit_exact(tmp_path):
    p = tmp_path / "ref.mat0"
    p.write_bytes(GOLD["mat0_bytes"].tobytes())
    x = mf.read_matrix(p)
    assert x.values.tobytes() == GOLD["values"].tobytes()  # -0.0 and extremes included
    assert (x.n1, x.n2) == (int(GOLD["n1"]), int(GOLD["n2"]))
    assert not x.values.flags.writeable
    a, n1, n2 = mf.read_array(p, threads=3)
    assert np.array_equal(a, GOLD["values"]) and (n1, n2) == (2, 3)


def test_writers_match_reference_bytes(tmp_path):
    x = rmx.DataMatrix(GOLD["values"], int(GOLD["n1"]), int(GOLD["n2"]))
    mf.write_matrix(x, tmp_path / "a.mat0")
    assert (tmp_path / "a.mat0").read_bytes() == GOLD["mat0_bytes"].tobytes()
    mf.write_matrix_csv(x, tmp_path / "a.csv")
    assert (tmp_path / "a.csv").read_bytes() == GOLD["csv_bytes"].tobytes()
    y = mf.load_matrix(tmp_path / "a.csv")
    assert y.values.tobytes() == x.values.tobytes()


@pytest.mark.parametrize("name", [str(n) for n in GOLD["case_names"]])
def test_error_messages_match_reference(tmp_path, name):
    i = [str(n) for n in GOLD["case_names"]].index(name)
    want = str(GOLD["case_msgs"][i])
    p = tmp_path / (name + (".csv" if name.startswith("csv") else ".mat0"))
    p.write_bytes(GOLD["case_" + name].tobytes())
    try:
        mf.load_matrix(p)
        got = "OK"
    except Exception as e:
        got = type(e).__name__ + ": " + str(e).replace(str(p), "<PATH>")
    assert got == want


def test_large_parallel_read_and_missing_file(tmp_path):
    g = np.random.default_rng(3)
    a = g.standard_normal((3001, 17))
    mf.write_array(a, tmp_path / "b.mat0", 0, 0)
    b, n1, n2 = mf.read_array(tmp_path / "b.mat0", threads=8)
    assert np.array_equal(a, b) and (n1, n2) == (0, 0)
    with pytest.raises(rmx.DataFormatError, match="bare matrix"):
        mf.read_matrix(tmp_path / "b.mat0")
    with pytest.raises(FileNotFoundError):
        mf.read_array(tmp_path / "missing.mat0")


def test_ranged_rows_read_and_write(tmp_path):
    """rmx_mat0_read_rows / rmx_mat0_create / rmx_mat0_write_rows (the piece
    reader of the streamed engine and the --dump-T writer): ranges of a file
    equal slices of read_array; a file written in ragged row ranges equals
    write_array's bytes."""
    import ctypes

    from paper_1703_01506_b200 import _native as nat

    lib = nat.load()
    a = np.random.default_rng(4).standard_normal((1031, 13))
    p = tmp_path / "a.mat0"
    mf.write_array(a, p, 0, 0)
    st, bad = nat.Status(), ctypes.c_int64(-1)
    for r0, r1 in ((0, 1031), (5, 6), (100, 977), (1000, 1031)):
        out = np.empty((r1 - r0, 13))
        rc = lib.rmx_mat0_read_rows(bytes(p), 13, r0, r1, out.ctypes.data, 3, ctypes.byref(bad),
                                    ctypes.byref(st))
        assert rc == 0 and np.array_equal(out, a[r0:r1])
    q = tmp_path / "b.mat0"
    assert lib.rmx_mat0_create(bytes(q), 1031, 13, 0, 0, ctypes.byref(st)) == 0
    for r0, r1 in ((700, 1031), (0, 3), (3, 700)):
        blk = np.ascontiguousarray(a[r0:r1])
        assert lib.rmx_mat0_write_rows(bytes(q), 13, r0, r1, blk.ctypes.data, 4,
                                       ctypes.byref(st)) == 0
    assert q.read_bytes() == p.read_bytes()
    b = a.copy()
    b[600, 4] = np.inf
    mf.write_array(b, p, 0, 0)
    out = np.empty((500, 13))
    rc = lib.rmx_mat0_read_rows(bytes(p), 13, 500, 1000, out.ctypes.data, 2, ctypes.byref(bad),
                                ctypes.byref(st))
    assert rc == nat.RMX_E_FORMAT and bad.value == 600 * 13 + 4
