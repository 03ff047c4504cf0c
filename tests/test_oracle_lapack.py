"""Independent numpy/LAPACK restatement of the path, used to cross-check the C++ oracle.

The C++ oracle (oracle/tenring_oracle.hpp) restates the reference with its own small dense
linear algebra (Householder QR with Eigen's sign rule, a one-sided Jacobi SVD standing in for
Eigen's BDCSVD, LLT/LDLT). The reference itself cannot be built here (no Eigen),
so this file restates the same algorithms a second time on numpy + LAPACK (geqrf/gesdd via
np.linalg, lstsq) and a vectorised numpy SplitMix64/Box-Muller, sharing no code with the
oracle, and checks the oracle against it on C1-sized inputs (BASELINE.json configs[0]):

* economy_q (sketch.hpp:45-53): LAPACK QR with columns flipped so diag(R) >= 0;
* sketch (sketch.hpp:62-89): sequential shrink, one Gaussian stream across modes;
* the Jacobi SVD against LAPACK's singular values and vectors (up to sign);
* trsvd (solvers.hpp:382-459): ranks, discarded energy, reconstruction and RSE;
* trals (solvers.hpp:297-334, direct least-squares route :238-251): the RSE trajectory and
  cores, with lstsq in place of the Householder solve (same unique LS solution).
"""
import math

import numpy as np
import pytest

import oracle_ref as orc

MASK = np.uint64(0xFFFFFFFFFFFFFFFF)
GAMMA = np.uint64(0x9E3779B97F4A7C15)


def np_gaussian(seed, n, skip=0):
    """random.hpp:14-62, vectorised: draw d uses the uniform pair 2*(d//2), 2*(d//2)+1."""
    first = skip - (skip % 2)
    npair = (skip + n - first + 1) // 2
    k = np.arange(2 * (first // 2), 2 * (first // 2) + 2 * npair, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (k + np.uint64(1)) * GAMMA
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    u = ((z >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * 2.0 ** -53
    u1, u2 = u[0::2], u[1::2]
    r = np.sqrt(-2.0 * np.log(u1))
    g = np.empty(2 * npair)
    g[0::2] = r * np.cos(2.0 * math.pi * u2)
    g[1::2] = r * np.sin(2.0 * math.pi * u2)
    return g[skip - first: skip - first + n]


def np_economy_q(y):
    q, r = np.linalg.qr(y)
    s = np.where(np.diag(r) < 0, -1.0, 1.0)
    return q * s


def np_unfold(x, n):  # unfold_classic, tensor.hpp:133-142
    return np.moveaxis(x, n, 0).reshape(x.shape[n], -1, order="F")


def np_mode_product(x, n, m):  # tensor.hpp:193-207
    return np.moveaxis(np.tensordot(m, x, axes=([1], [n])), 0, n)


def np_sketch(x, K, seed):
    cur, bases, D = np.array(x, dtype=np.float64), [], 0
    for n in range(x.ndim):
        if K[n] == x.shape[n]:
            bases.append(np.eye(K[n]))
            continue
        xn = np_unfold(cur, n)
        om = np_gaussian(seed, xn.shape[1] * K[n], skip=D).reshape(xn.shape[1], K[n], order="F")
        D += xn.shape[1] * K[n]
        q = np_economy_q(xn @ om)
        bases.append(q)
        cur = np_mode_product(cur, n, q.T)
    return cur, bases


def np_reconstruct(cores):
    t = cores[0]
    for g in cores[1:]:
        t = np.tensordot(t, g, axes=([t.ndim - 1], [0]))
    return np.trace(t, axis1=0, axis2=t.ndim - 1)


def np_rse(x, y):
    return float(np.linalg.norm(x - y) / np.linalg.norm(x))


def np_unfold_tr(x, n):  # tensor.hpp:147-157: columns (i_{n+1}, ..., i_{N-1}, i_0, ..., i_{n-1})
    N = x.ndim
    return np.transpose(x, [n] + list(range(n + 1, N)) + list(range(n))).reshape(x.shape[n], -1, order="F")


def np_subchain_matrix(cores, n):
    """unfold_tr(subchain(f, n), 1) (tr_factors.hpp:111-119): S(p, a + R_n b) = sub(b, p, a)."""
    N = len(cores)
    t = cores[(n + 1) % N]
    for s in range(2, N):
        t = np.tensordot(t, cores[(n + s) % N], axes=([t.ndim - 1], [0]))
    rb, ra = t.shape[0], t.shape[-1]
    sub = t.reshape(rb, -1, ra, order="F")
    return np.transpose(sub, (1, 2, 0)).reshape(sub.shape[1], ra * rb, order="F")


def np_trals(x, ranks, sweeps, seed):
    N = x.ndim
    dims = x.shape
    scale = (np.linalg.norm(x) / float(np.prod(ranks))) ** (1.0 / N)  # solvers.hpp:80-95
    sizes = [ranks[n] * dims[n] * ranks[(n + 1) % N] for n in range(N)]
    draws = np_gaussian(seed, sum(sizes))
    cores, off = [], 0
    for n in range(N):
        cores.append(scale * draws[off:off + sizes[n]].reshape(ranks[n], dims[n], ranks[(n + 1) % N], order="F"))
        off += sizes[n]
    hist = []
    for _ in range(sweeps):
        for n in range(N):
            S = np_subchain_matrix(cores, n)
            assert S.shape[0] <= 4096 and S.shape[0] >= S.shape[1]  # the direct route (solvers.hpp:242)
            z = np.linalg.lstsq(S, np_unfold_tr(x, n).T, rcond=None)[0]  # (R_n R_{n+1}) x I_n
            rn, rn1 = ranks[n], ranks[(n + 1) % N]
            cores[n] = np.transpose(z.reshape(rn, rn1, dims[n], order="F"), (0, 2, 1))
        hist.append(np_rse(x, np_reconstruct(cores)))
    return cores, hist


def lapack_svd_signed_like_oracle(m):
    """LAPACK thin SVD under the sign convention the oracle and the product share: the
    largest-magnitude entry of every left singular vector is positive.

    trsvd is sign-dependent beyond its first split: flipping singular pair (p, q) of the first
    SVD negates entries (q, p) of the next unfolding, where q indexes its rows and p its
    columns, which is not a row or column scaling, so the later singular values (and the
    truncation ranks) change. BDCSVD fixes no sign (solvers.hpp:398-435), so the reference's
    own ranks beyond the first split depend on Eigen's internal sign choices; a fixed rule
    makes them reproducible."""
    u, s, vt = np.linalg.svd(m, full_matrices=False)
    arg = np.argmax(np.abs(u), axis=0)
    sg = np.where(u[arg, np.arange(u.shape[1])] < 0, -1.0, 1.0)
    return u * sg, s, vt * sg[:, None]


def np_trsvd(x, tol):
    """solvers.hpp:382-459 with LAPACK's SVD; returns (cores, discarded energy)."""
    N = x.ndim
    dims = x.shape
    budget_sq = (tol * np.linalg.norm(x) / math.sqrt(N)) ** 2
    disc = [0.0]

    def trunc(s):
        r, tail = len(s), 0.0
        while r > 1 and tail + s[r - 1] ** 2 <= budget_sq:
            tail += s[r - 1] ** 2
            r -= 1
        disc[0] += tail
        return r

    def split(r):
        t = int(math.isqrt(r))
        best = 1
        for d in range(1, r + 1):
            if r % d == 0 and abs(d - t) < abs(best - t):
                best = d
        return best, r // best

    u, s, vt = lapack_svd_signed_like_oracle(x.reshape(dims[0], -1, order="F"))
    r01 = trunc(s)
    ra, rb = split(r01)
    cores = [np.transpose(u[:, :r01].reshape(dims[0], ra, rb, order="F"), (1, 0, 2))]
    rest = x.size // dims[0]
    w = (s[:r01, None] * vt[:r01]).reshape(ra, rb, rest, order="F")  # row p + ra q
    cur = np.transpose(w, (1, 2, 0)).reshape(-1, order="F")  # (q, c, p): R_1 leads, R_0 trails
    lead = rb
    for k in range(1, N - 1):
        rows = lead * dims[k]
        m = cur.reshape(rows, -1, order="F")
        u, s, vt = lapack_svd_signed_like_oracle(m)
        r = trunc(s)
        cores.append(u[:, :r].reshape(lead, dims[k], r, order="F"))
        cur = (s[:r, None] * vt[:r]).reshape(-1, order="F")
        lead = r
    cores.append(cur.reshape(lead, dims[N - 1], ra, order="F"))
    return cores, disc[0]


def tr_input(dims, R, seed, snr):
    return orc.add_noise(orc.reconstruct_full(orc.random_factors(dims, [R] * len(dims), seed)), snr, seed + 1)


def test_numpy_rng_matches_golden():
    import json
    import os

    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "rng_kat.json")))
    for seed, vals in gold["gaussian"].items():
        np.testing.assert_allclose(np_gaussian(int(seed), len(vals)), vals, rtol=1e-15, atol=1e-15)
    np.testing.assert_allclose(np_gaussian(7, 9, skip=13), np_gaussian(7, 40)[13:22], rtol=0, atol=0)


@pytest.mark.parametrize("shape,cond", [((100, 10), 1.0), ((1024, 64), 1.0), ((200, 16), 1e8), ((60, 12), 1e10)])
def test_economy_q_matches_lapack(shape, cond):
    rng = np.random.default_rng(3)
    u, _ = np.linalg.qr(rng.standard_normal(shape))
    v, _ = np.linalg.qr(rng.standard_normal((shape[1], shape[1])))
    y = (u * np.logspace(0, -math.log10(cond), shape[1])) @ v.T
    got, want = orc.economy_q(y), np_economy_q(y)
    # first-order perturbation of Q: O(u * cond(Y)) for any backward-stable QR
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < max(1e-14 * cond, 1e-13)


def test_sketch_matches_numpy_c1():
    """C1 shape (100^3 f64, K=10): the oracle's sketch() against numpy/LAPACK + numpy RNG."""
    x = tr_input([100, 100, 100], 5, 0, 40.0)
    proj, bases, _ = orc.sketch(x, [10, 10, 10], 0)
    want_p, want_b = np_sketch(x, [10, 10, 10], 0)
    assert np.linalg.norm(proj - want_p) / np.linalg.norm(want_p) < 1e-12
    for a, b in zip(bases, want_b):
        assert np.linalg.norm(a - b) / np.linalg.norm(b) < 1e-12


def test_sketch_skipped_mode_matches_numpy():
    x = tr_input([20, 12, 18, 9], 3, 4, 30.0)
    K = [6, 12, 5, 9]
    proj, bases, _ = orc.sketch(x, K, 11)
    want_p, want_b = np_sketch(x, K, 11)
    assert np.linalg.norm(proj - want_p) / np.linalg.norm(want_p) < 1e-12


@pytest.mark.parametrize("shape", [(10, 100), (100, 10), (36, 48), (144, 12)])
def test_jacobi_svd_matches_lapack(shape):
    a = np.random.default_rng(5).standard_normal(shape)
    s, u, v = orc.svd(a)
    uw, sw, vwt = np.linalg.svd(a, full_matrices=False)
    np.testing.assert_allclose(s, sw, rtol=1e-12, atol=1e-13 * sw[0])
    # vectors equal under the shared sign convention
    uw, _, vwt = lapack_svd_signed_like_oracle(a)
    np.testing.assert_allclose(u, uw, atol=1e-10)
    np.testing.assert_allclose(v, vwt.T, atol=1e-10)
    np.testing.assert_allclose((u * s) @ v.T, a, atol=1e-12 * sw[0])


@pytest.mark.parametrize("tol", [1e-3, 0.05])
def test_trsvd_matches_lapack_on_c1_projection(tol):
    """C1's projected tensor (10^3), and a C2-shaped 16^4 projection: ranks, discarded energy,
    reconstruction and RSE of the oracle's trsvd against the LAPACK restatement."""
    for dims, R, K in (([100, 100, 100], 5, [10] * 3), ([40, 40, 40, 40], 3, [16] * 4)):
        x = tr_input(dims, R, 0, 30.0)
        p, _, _ = orc.sketch(x, K, 0)
        rep = orc.solve("svd", p, tol=tol)
        cores, disc = np_trsvd(p, tol)
        assert rep.ranks == [c.shape[0] for c in cores]
        assert abs(rep.discarded_sq - disc) <= 1e-10 * np.vdot(p, p)
        rec_o, rec_n = orc.reconstruct_full(rep.cores), np_reconstruct(cores)
        assert np.linalg.norm(rec_o - rec_n) / np.linalg.norm(rec_n) < 1e-10
        for a, b in zip(rep.cores, cores):  # same sign rule: the cores themselves agree
            assert np.linalg.norm(a - b) / np.linalg.norm(b) < 1e-9
        assert abs(rep.rse_history[-1] - np_rse(p, rec_n)) <= 1e-10 * np_rse(p, rec_n) + 1e-13  # floor: exact fits


def test_trals_matches_lapack_on_c1_projection():
    """C1 end to end on the small side: the projected 10^3 tensor, TR rank 5, 20 sweeps, seed 0
    (the direct least-squares route). The RSE trajectory and the cores of the oracle's trals
    against the numpy/lstsq restatement."""
    x = tr_input([100, 100, 100], 5, 0, 40.0)
    p, _, _ = orc.sketch(x, [10] * 3, 0)
    rep = orc.solve("als", p, ranks=[5, 5, 5], max_sweeps=20, seed=0)
    cores, hist = np_trals(p, [5, 5, 5], 20, 0)
    np.testing.assert_allclose(rep.rse_history, hist, rtol=1e-9)
    for a, b in zip(rep.cores, cores):
        assert np.linalg.norm(a - b) / np.linalg.norm(b) < 1e-8
