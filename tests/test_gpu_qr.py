"""K4 thin QR (detail::economy_q, sketch.hpp:45-53) against the oracle's
Householder restatement: Q within 1e-10 (fp64), sign convention diag(R) >= 0,
CholQR2 fast path and the Householder fallback both exercised."""
import numpy as np
import pytest

import oracle_ref as orc

pytestmark = pytest.mark.gpu

# every (I_n, K_n) of the BASELINE configs plus edge shapes
SHAPES = [(100, 10), (100, 16), (1000, 20), (1024, 64), (200, 32), (60, 12), (8, 8), (37, 1), (513, 33),
          (300, 64), (2000, 7)]


@pytest.fixture(scope="module")
def trg():
    import paper_1901_01652_b200 as trg

    return trg


@pytest.mark.parametrize("m,k", SHAPES)
def test_qr_matches_oracle(trg, m, k):
    y = np.random.default_rng(m * 131 + k).standard_normal((m, k))
    q, path = trg.economy_q(y, return_path=True)
    want = orc.economy_q(y)
    assert path == 0  # well-conditioned Gaussian sketch: CholQR2
    assert np.abs(q - want).max() < 1e-10
    assert np.abs(q.T @ q - np.eye(k)).max() < 1e-12


def test_qr_ill_conditioned_takes_householder(trg):
    rng = np.random.default_rng(1)
    u, _ = np.linalg.qr(rng.standard_normal((120, 12)))
    v, _ = np.linalg.qr(rng.standard_normal((12, 12)))
    y = u @ np.diag(np.logspace(0, -9, 12)) @ v.T  # cond 1e9 > CholQR2's eps^-1/2 range
    q, path = trg.economy_q(y, return_path=True)
    want = orc.economy_q(y)
    assert path == 1
    assert np.abs(q - want).max() < 1e-6  # Q itself is cond-sensitive; both are Householder


def test_qr_rank_deficient(trg):
    rng = np.random.default_rng(2)
    y = rng.standard_normal((50, 3)) @ rng.standard_normal((3, 6))  # rank 3 < 6
    q, path = trg.economy_q(y, return_path=True)
    assert path == 1
    want = orc.economy_q(y)
    # the range-spanning first 3 columns are determined; the rest depend on rounding in both
    assert np.abs(q[:, :3] - want[:, :3]).max() < 1e-10


def test_qr_wide_k_uses_householder_kernel(trg):
    y = np.random.default_rng(3).standard_normal((150, 80))
    q, path = trg.economy_q(y, return_path=True)
    assert path == 1
    assert np.abs(q - orc.economy_q(y)).max() < 1e-10


def test_qr_errors(trg):
    with pytest.raises(ValueError):
        trg.economy_q(np.zeros((3, 5)))


@pytest.mark.parametrize("m,k", [(1000, 20), (1024, 64), (200, 32)])
def test_qr_cluster_ill_conditioned_falls_back(trg, m, k):
    """K_n > 16 runs the cluster CholQR2; cond 1e9 must reach the Householder fallback (rank 0)."""
    rng = np.random.default_rng(m + k)
    u, _ = np.linalg.qr(rng.standard_normal((m, k)))
    v, _ = np.linalg.qr(rng.standard_normal((k, k)))
    y = u @ np.diag(np.logspace(0, -9, k)) @ v.T
    q, path = trg.economy_q(y, return_path=True)
    assert path == 1
    assert np.abs(q - orc.economy_q(y)).max() < 1e-6


def test_qr_cluster_rank_deficient(trg):
    rng = np.random.default_rng(5)
    y = rng.standard_normal((300, 5)) @ rng.standard_normal((5, 24))  # rank 5 < 24
    q, path = trg.economy_q(y, return_path=True)
    assert path == 1
    assert np.abs(q[:, :5] - orc.economy_q(y)[:, :5]).max() < 1e-10


def test_qr_cluster_moderate_condition_two_passes(trg):
    """cond 1e4: CholQR's first pass is not orthonormal to 1e-13, the second pass must run."""
    rng = np.random.default_rng(6)
    u, _ = np.linalg.qr(rng.standard_normal((1024, 64)))
    v, _ = np.linalg.qr(rng.standard_normal((64, 64)))
    y = u @ np.diag(np.logspace(0, -4, 64)) @ v.T
    q, path = trg.economy_q(y, return_path=True)
    assert path == 0
    assert np.abs(q.T @ q - np.eye(64)).max() < 1e-13
    assert np.abs(q - orc.economy_q(y)).max() < 1e-10
