"""DTEN / TRNG containers (reference io.hpp:84-129, tr_factors.hpp:161-200).

Bit-exact round trips, a hand-assembled golden byte string of the layout, every malformed-input
error of the reference readers, and a cross-check between the Python module and the C++ facade
(both directions). Host only.
"""
import io
import os
import struct
import subprocess
import tempfile

import numpy as np
import pytest

from paper_1901_01652_b200 import FormatError, read_dten, read_trng, write_dten, write_trng

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1901_01652_b200")


def test_dten_golden_layout():
    t = np.arange(6, dtype=np.float64).reshape((2, 3), order="F") * 0.5
    buf = io.BytesIO()
    write_dten(buf, t)
    want = b"DTEN" + struct.pack("<II", 1, 2) + struct.pack("<QQ", 2, 3) + struct.pack("<6d", 0, .5, 1, 1.5, 2, 2.5)
    assert buf.getvalue() == want


def test_dten_round_trip_bit_exact():
    rng = np.random.default_rng(0)
    t = rng.standard_normal((3, 4, 5))
    t.reshape(-1)[:4] = [np.inf, -np.inf, -0.0, 5e-324]
    buf = io.BytesIO()
    write_dten(buf, t)
    buf.seek(0)
    r = read_dten(buf)
    assert r.shape == t.shape
    assert r.reshape(-1, order="F").view(np.uint64).tolist() == t.reshape(-1, order="F").view(np.uint64).tolist()


@pytest.mark.parametrize("blob,msg", [
    (b"DTEX" + struct.pack("<II", 1, 1) + struct.pack("<Q", 1) + b"\0" * 8, "bad magic"),
    (b"DTEN" + struct.pack("<II", 2, 1) + struct.pack("<Q", 1) + b"\0" * 8, "unsupported DTEN version 2"),
    (b"DTEN" + struct.pack("<II", 1, 0), "order must be at least 1"),
    (b"DTEN" + struct.pack("<II", 1, 2) + struct.pack("<QQ", 2, 0), "extents must be positive"),
    (b"DTEN" + struct.pack("<II", 1, 1) + struct.pack("<Q", 3) + b"\0" * 16, "end of file while reading DTEN values"),
    (b"DTE", "end of file while reading DTEN magic"),
])
def test_dten_errors(blob, msg):
    with pytest.raises(FormatError, match=msg):
        read_dten(io.BytesIO(blob))


def test_trng_round_trip_and_errors():
    rng = np.random.default_rng(1)
    cores = [rng.standard_normal((2, 4, 3)), rng.standard_normal((3, 5, 2))]
    buf = io.BytesIO()
    write_trng(buf, cores)
    buf.seek(0)
    back = read_trng(buf)
    assert all(np.array_equal(a, b) for a, b in zip(cores, back))
    # rank mismatch in the file -> FormatError (the reader validates the ring)
    bad = io.BytesIO()
    bad.write(b"TRNG" + struct.pack("<II", 1, 2))
    write_dten(bad, cores[0])
    write_dten(bad, rng.standard_normal((4, 5, 2)))
    bad.seek(0)
    with pytest.raises(FormatError, match="inconsistent"):
        read_trng(bad)
    with pytest.raises(FormatError, match="at least one core"):
        read_trng(io.BytesIO(b"TRNG" + struct.pack("<II", 1, 0)))
    with pytest.raises(FormatError, match="cannot open"):
        read_trng(os.path.join(ROOT, "does", "not", "exist.trng"))


def test_cpp_facade_exchange():
    if not os.path.exists(os.path.join(LIBDIR, "libtrg.so")):
        from paper_1901_01652_b200 import build

        build.build()
    rng = np.random.default_rng(2)
    t = rng.standard_normal((4, 3, 2))
    cores = [rng.standard_normal((2, 3, 3)), rng.standard_normal((3, 4, 2))]
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "io_main")
        subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "cpp", "io_main.cpp"), "-L", LIBDIR, "-ltrg",
                        f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True, capture_output=True, text=True)
        p = {n: os.path.join(d, n) for n in ("a.dten", "a.trng", "b.dten", "b.trng", "bad1", "bad2")}
        write_dten(p["a.dten"], t)
        write_trng(p["a.trng"], cores)
        open(p["bad1"], "wb").write(b"DTEN" + struct.pack("<II", 7, 1))
        open(p["bad2"], "wb").write(b"DTEN" + struct.pack("<II", 1, 1) + struct.pack("<Q", 0))
        r = subprocess.run([exe, p["a.dten"], p["a.trng"], p["b.dten"], p["b.trng"], p["bad1"], p["bad2"]],
                           capture_output=True, text=True, timeout=60)
        assert r.returncode == 0, r.stderr
        assert "dten order 3 size 24" in r.stdout and "trng cores 2" in r.stdout
        assert "bad 0: format_error: unsupported DTEN version 7" in r.stdout
        assert "bad 1: format_error: DTEN extents must be positive" in r.stdout
        # the C++ writer reproduces the Python bytes exactly
        assert open(p["b.dten"], "rb").read() == open(p["a.dten"], "rb").read()
        assert open(p["b.trng"], "rb").read() == open(p["a.trng"], "rb").read()
