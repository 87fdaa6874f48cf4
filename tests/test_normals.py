"""The native standard_normal (csrc/normals.cpp, numpy's ziggurat over the
reference's SFC64 streams) vs numpy itself, bit for bit.  Host code: runs
without a GPU."""
import os
import subprocess

import numpy as np
import pytest

from paper_1703_01506_b200 import normals
from paper_1703_01506_b200.rng import BASIS_INIT, SHIFT_GAP, stream


@pytest.mark.parametrize("seed,path,count", [(5, (5,), 200_000), (1703015065, (BASIS_INIT,), 3_000_000),
                                            (2**63 + 11, (8, 7), 100_000), (0, (), 50_000),
                                            (1703015062, (4, 12345), 262_144)])
def test_stream_bit_exact(seed, path, count):
    got = normals.standard_normal(seed, path, count)
    ref = stream(seed, *path).standard_normal(count)
    assert np.array_equal(got, ref)


def test_pieces_and_rows_bit_exact():
    ref = stream(77, BASIS_INIT).standard_normal(1_000_003)
    gen = normals.NormalStream(77, (BASIS_INIT,))
    parts, lo = [], 0
    for n in (1, 999, 65536, 1 << 19, 1_000_003 - (1 + 999 + 65536 + (1 << 19))):
        parts.append(gen.fill(np.empty(n)))
        lo += n
    gen.close()
    assert np.array_equal(np.concatenate(parts), ref)
    r32 = normals.standard_normal_rows(9, SHIFT_GAP, 3, 40, 20_000, threads=4)
    r64 = normals.standard_normal_rows(9, SHIFT_GAP, 3, 40, 20_000, dtype=np.float64)
    ref = np.stack([stream(9, SHIFT_GAP, i).standard_normal(20_000) for i in range(3, 40)])
    assert np.array_equal(r64, ref) and np.array_equal(r32, ref.astype(np.float32))


def test_tail_and_wedge_paths_exercised():
    """Enough draws that the base-strip tail (|x| > 3.654) and wedge tests
    occur many times, all bit-identical."""
    got = normals.standard_normal(123, (BASIS_INIT,), 4_000_000)
    ref = stream(123, BASIS_INIT).standard_normal(4_000_000)
    assert np.array_equal(got, ref)
    assert np.sum(np.abs(ref) > 3.6541528853610088) > 500


def test_probed_tables_equal_numpys_compiled_tables(tmp_path):
    """The tables read from numpy through the probing bit generator equal the
    ones compiled into numpy's own libnpyrandom.a (when it is installed)."""
    lib = os.path.join(os.path.dirname(np.__file__), "random", "lib", "libnpyrandom.a")
    if not os.path.exists(lib):
        pytest.skip("numpy's static random library is not installed")
    obj = "src_distributions_distributions.c.o"
    subprocess.run(["ar", "x", lib, obj], cwd=tmp_path, check=True)
    subprocess.run(["objcopy", "-O", "binary", "--only-section=.rodata", obj, "ro.bin"],
                   cwd=tmp_path, check=True)
    syms = subprocess.run(["nm", obj], cwd=tmp_path, capture_output=True, text=True).stdout
    off = {ln.split()[2]: int(ln.split()[0], 16) for ln in syms.splitlines()
           if ln.split()[-1] in ("ki_double", "wi_double", "fi_double")}
    ro = (tmp_path / "ro.bin").read_bytes()
    k, w, f = normals.tables()
    assert np.array_equal(k, np.frombuffer(ro[off["ki_double"]:off["ki_double"] + 2048], "<u8"))
    assert np.array_equal(w, np.frombuffer(ro[off["wi_double"]:off["wi_double"] + 2048], "<f8"))
    assert np.array_equal(f, np.frombuffer(ro[off["fi_double"]:off["fi_double"] + 2048], "<f8"))
