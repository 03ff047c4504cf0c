"""Persistent tail (tail.cu): the last modes of the sequential projection (sketch.hpp:73-87) in one
launch once the working tensor is L2-sized. Each case runs with the tail (default) and without it
(TRG_TAIL_MB=0, the per-mode kernels), both against the oracle at the north_star tolerances, and
checks that the tail launch really ran (its label in the context's kernel statistics)."""
import os

import numpy as np
import pytest

import oracle_ref as orc

pytestmark = pytest.mark.gpu

F64_TOL = 1e-10
F32_TOL = 1e-4


@pytest.fixture(scope="module")
def trg():
    import paper_1901_01652_b200 as trg

    return trg


def relerr(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def run(trg, x, K, seed, tail_mb):
    old = os.environ.get("TRG_TAIL_MB")
    os.environ["TRG_TAIL_MB"] = str(tail_mb)
    try:
        ctx = trg.Context()
        ctx.set_profiling(True)
        sk = trg.DeviceSketch(ctx, trg.DeviceTensor.from_numpy(ctx, x), trg.ProjectionSpec(list(K), seed))
        out = (sk.projected(), [sk.basis(n) for n in range(len(K))], [sk.sketch_matrix(n) for n in range(len(K))],
               [sk.qr_householder(n) for n in range(len(K))])
        labels = ctx.kernel_labels()
        sk.close()
        ctx.close()
    finally:
        if old is None:
            del os.environ["TRG_TAIL_MB"]
        else:
            os.environ["TRG_TAIL_MB"] = old
    return out, labels


# (dims, K, expect the tail): C1 (one CTA per last-mode slab, P summed over the slabs), order 4/5,
# the C2 tail geometry at reduced size (a chunks of the mode-n0 left index), K = 32 (KW 32), K <= 8,
# odd extents, order 2 and 1
CASES = [
    ((100, 100, 100), (10, 10, 10)),
    ((12, 11, 10, 9), (3, 4, 5, 2)),
    ((16, 16, 40, 30), (8, 4, 16, 12)),
    ((8, 7, 6, 5, 4), (2, 3, 5, 2, 3)),
    ((20, 24, 200), (6, 5, 16)),
    ((33, 17, 29), (7, 5, 3)),
    ((300, 7), (6, 3)),
    ((40,), (1,)),
]


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("dims,K", CASES)
def test_tail_matches_oracle(trg, dims, K, dtype):
    rng = np.random.default_rng(sum(dims) + len(dims))
    x = rng.standard_normal(dims).astype(dtype)
    seed = 29
    proj, bases, ys = orc.sketch(x.astype(np.float64), K, seed)
    tol = F64_TOL if dtype == np.float64 else F32_TOL
    got = {}
    for mb in (40, 0):
        (P, Q, Y, hh), labels = run(trg, x, K, seed, mb)
        assert ("tail" in labels) == (mb > 0), labels
        for n in range(len(dims)):
            assert relerr(Y[n], ys[n]) < tol, (mb, n)
            assert relerr(Q[n], bases[n]) < tol, (mb, n)
            assert hh[n] == 0
        assert relerr(P, proj) < tol, mb
        got[mb] = P
    if dtype == np.float64:
        assert relerr(got[40], got[0]) < 1e-13


def test_tail_is_deterministic(trg):
    x = np.random.default_rng(4).standard_normal((100, 100, 100))
    (p1, _, _, _), _ = run(trg, x, (10, 10, 10), 3, 40)
    (p2, _, _, _), _ = run(trg, x, (10, 10, 10), 3, 40)
    np.testing.assert_array_equal(p1, p2)


def test_tail_rank_deficient_falls_back_to_householder(trg):
    """A rank-1 tensor gives rank-1 sketches: the in-kernel CholQR breaks down and the tail's QR CTA
    runs the Householder fallback (sign rule of sketch.hpp:51-52) for every mode."""
    rng = np.random.default_rng(8)
    u, v, w = rng.standard_normal(30), rng.standard_normal(20), rng.standard_normal(10)
    x = np.einsum("i,j,k->ijk", u, v, w)
    K = (4, 3, 2)
    _, bases, ys = orc.sketch(x, K, 11)
    (P, Q, Y, hh), labels = run(trg, x, K, 11, 40)
    assert "tail" in labels
    assert hh == [1, 1, 1]
    for n in range(3):
        assert relerr(Y[n], ys[n]) < F64_TOL
        # the range-spanning first column is determined; the rest depend on rounding in both
        assert np.abs(Q[n][:, :1] - bases[n][:, :1]).max() < 1e-10
        assert np.abs(Q[n].T @ Q[n] - np.eye(K[n])).max() < 1e-12
