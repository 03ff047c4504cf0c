"""The C++ facade (include/tenring_b200.hpp) over the C ABI.

CPU: the header compiles as C++17 and links against libtrg.so (the reference
caller's view: tenring::b200::sketch / rtrals / rtrsvd / rse / decompose).
GPU: tests/cpp/facade_main.cpp drives the facade on a small TR tensor and its
outputs (P, Q_n, RSE of rTR-ALS and rTR-SVD, SVD ranks) are checked against
the CPU oracle on the same input.
"""
import os
import subprocess
import tempfile

import numpy as np
import pytest

import oracle_ref as orc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1901_01652_b200")


def _build(out):
    if not os.path.exists(os.path.join(LIBDIR, "libtrg.so")):
        from paper_1901_01652_b200 import build

        build.build()
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "facade_main.cpp"), "-L", LIBDIR, "-ltrg",
           f"-Wl,-rpath,{LIBDIR}", "-o", out]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


def test_facade_compiles_and_links():
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "facade_main")
        _build(exe)
        assert os.path.exists(exe)


def test_facade_header_is_c_abi_only():
    # the facade must sit on trg.h alone: no torch / CUDA types cross the boundary
    src = open(os.path.join(ROOT, "include", "tenring_b200.hpp")).read()
    assert '#include "trg.h"' in src
    for banned in ("torch", "cuda_runtime", "Eigen"):
        assert f"#include <{banned}" not in src and f'#include "{banned}' not in src


@pytest.mark.gpu
def test_facade_matches_oracle():
    dims, K, R = [40, 36, 30], [8, 8, 8], [3, 3, 3]
    x = orc.add_noise(orc.reconstruct_full(orc.random_factors(dims, R, 0)), 40.0, 1)
    with tempfile.TemporaryDirectory() as d:
        exe, fin, fout = (os.path.join(d, n) for n in ("facade_main", "in.bin", "out.bin"))
        _build(exe)
        with open(fin, "wb") as f:
            np.array([len(dims)] + dims + K + R, dtype=np.int64).tofile(f)
            np.asarray(x, dtype=np.float64).reshape(-1, order="F").tofile(f)
        r = subprocess.run([exe, fin, fout], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr
        raw = open(fout, "rb").read()
    off = 0

    def take(n, dt=np.float64):
        nonlocal off
        a = np.frombuffer(raw, dtype=dt, count=n, offset=off)
        off += n * 8
        return a

    P = take(int(np.prod(K))).reshape(K, order="F")
    Q = [take(dims[n] * K[n]).reshape((dims[n], K[n]), order="F") for n in range(3)]
    rse_als, rse_svd = take(1)[0], take(1)[0]
    svd_ranks = list(take(3, np.int64))
    same = take(1)[0]
    proj, bases, _ = orc.sketch(x, K, 0)
    assert np.linalg.norm(P - proj) / np.linalg.norm(proj) < 1e-10
    for a, b in zip(Q, bases):
        assert np.linalg.norm(a - b) / np.linalg.norm(b) < 1e-10
    want_als = orc.rtrd("als", x, K, ranks=R, max_sweeps=5)
    want_svd = orc.rtrd("svd", x, K, tol=1e-3)
    assert abs(rse_als - want_als.rse_history[-1]) <= 1e-9 * want_als.rse_history[-1]
    assert svd_ranks == list(want_svd.ranks)
    assert abs(rse_svd - want_svd.rse_history[-1]) <= 1e-9 * want_svd.rse_history[-1]
    assert same == 1.0
