"""Opt-in Khatri-Rao test matrices (include/trg.h TRG_OMEGA_KHATRI_RAO).

The GPU path (factor draws, Khatri-Rao blocks, products inside the streaming sketch kernels) is
checked against the numpy restatement in oracle_ref.kr_sketch on the same seeds, at the fp64
tolerance of the Gaussian path (1e-10 relative on Y_n, Q_n and P).
"""
import numpy as np
import pytest

import oracle_ref as orc

pytestmark = pytest.mark.gpu

F64_TOL = 1e-10


@pytest.fixture(scope="module")
def trg():
    import paper_1901_01652_b200 as trg

    return trg


def relerr(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def tr_tensor(dims, ranks, seed, snr=None):
    x = orc.reconstruct_full(orc.random_factors(dims, ranks, seed))
    if snr is not None:
        x = orc.add_noise(x, snr, seed + 1)
    return x


CASES = [
    ((100, 100, 100), (10, 10, 10), 0),   # C1 shape, sequential
    ((20, 18, 16, 14), (4, 4, 4, 4), 0),  # every split of the factors (A, F, H) is non-trivial somewhere
    ((40, 36, 30), (6, 4, 4), 1),         # fused variant: every Y_n from the original X
    ((24, 22, 20, 18), (4, 22, 6, 2), 0),  # mode 1 skipped: no factors drawn for it
]


@pytest.mark.parametrize("dims,K,variant", CASES)
def test_kr_sketch_matches_oracle(trg, dims, K, variant):
    x = tr_tensor(list(dims), [3] * len(dims), 11, snr=30.0)
    seed = 23
    proj, bases, ys = orc.kr_sketch(x, list(K), seed, variant)
    spec = trg.ProjectionSpec(list(K), seed, omega="khatri_rao")
    got = trg.sketch(x, spec, variant=variant)
    for n in range(len(dims)):
        if K[n] == dims[n]:
            np.testing.assert_array_equal(got.bases[n], np.eye(dims[n]))
            continue
        assert relerr(got.sketches[n], ys[n]) < F64_TOL, n
        assert relerr(got.bases[n], bases[n]) < F64_TOL, n
    assert relerr(got.projected, proj) < F64_TOL


def test_kr_differs_from_gaussian_and_is_deterministic(trg):
    x = tr_tensor([30, 28, 26], [3, 3, 3], 5)
    g = trg.sketch(x, trg.ProjectionSpec([6, 6, 6], 3))
    k1 = trg.sketch(x, trg.ProjectionSpec([6, 6, 6], 3, omega="khatri_rao"))
    k2 = trg.sketch(x, trg.ProjectionSpec([6, 6, 6], 3, omega="khatri_rao"))
    assert relerr(k1.sketches[0], g.sketches[0]) > 0.1
    np.testing.assert_array_equal(k1.projected, k2.projected)


def test_kr_unsupported_paths_fail_loudly(trg):
    x = np.random.default_rng(0).standard_normal((300, 20, 10))  # mode-0 extent beyond the streaming kernel
    with pytest.raises(Exception, match="Khatri-Rao"):
        trg.sketch(x, trg.ProjectionSpec([8, 4, 4], 0, omega="khatri_rao"))
    with pytest.raises(ValueError):
        trg.sketch(x, trg.ProjectionSpec([8, 4, 4], 0, omega="philox-kr"))


def test_kr_decomposition_quality(trg):
    # a structured test matrix is still a range finder: rTR-ALS through it reaches the same
    # reconstruction error as through the reference Gaussian sketch on a noisy TR tensor
    x = tr_tensor([60, 60, 60], [4, 4, 4], 2, snr=40.0)
    cfg = trg.SolverConfig(ranks=[4, 4, 4], tolerance=0.0, max_sweeps=10, seed=0)
    rg = trg.rtrals(x, cfg, trg.ProjectionSpec([16, 16, 16], 1))
    rk = trg.rtrals(x, cfg, trg.ProjectionSpec([16, 16, 16], 1, omega="khatri_rao"))
    assert rk.rse_history[-1] < 2.0 * rg.rse_history[-1] + 1e-6
