"""K8 / K9 reconstruction on the FP64 tensor pipe (tr.cu k_recon_dmma): the RSE (solvers.hpp:47-54
over tr_factors.hpp:123-137) and the synthesis X := Xhat, against the oracle and against the SIMT
kernel it replaces (TRG_RECON_SIMT=1) on shapes with ragged row tiles (I_0 not a multiple of 8,
several 128-row blocks), K = R_0 R_1 not a multiple of 4 and at its 64 limit, and column tails."""
import os

import numpy as np
import pytest

import oracle_ref as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def trg():
    import paper_1901_01652_b200 as trg

    return trg


def relerr(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300)


def with_env(var, val, fn):
    old = os.environ.get(var)
    if val is None:
        os.environ.pop(var, None)
    else:
        os.environ[var] = val
    try:
        return fn()
    finally:
        if old is None:
            os.environ.pop(var, None)
        else:
            os.environ[var] = old


CASES = [
    ([100, 100, 100], [5, 5, 5]),       # C1: K = 25
    ([37, 19, 23], [3, 7, 2]),          # ragged rows, K = 21
    ([300, 11, 13], [8, 8, 3]),         # three row blocks, K = 64
    ([20, 9, 8, 7], [4, 3, 2, 5]),      # order 4
    ([64, 33], [6, 6]),                 # order 2, K = 36
]


@pytest.mark.parametrize("dims,ranks", CASES)
def test_rse_dmma_f64(trg, dims, ranks):
    x = orc.add_noise(orc.reconstruct_full(orc.random_factors(dims, ranks, 3)), 25.0, 4)
    cores = orc.random_factors(dims, ranks, 9)
    want = orc.rse(x, orc.reconstruct_full(cores))
    got = with_env("TRG_RECON_SIMT", None, lambda: trg.rse(x, cores))
    simt = with_env("TRG_RECON_SIMT", "1", lambda: trg.rse(x, cores))
    assert abs(got - want) <= 1e-10 * want
    assert abs(got - simt) <= 1e-12 * want


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("dims,ranks", CASES[1:4])
def test_synthesize_dmma(trg, dims, ranks, dtype):
    ctx = trg.default_context()
    cores = orc.random_factors(dims, ranks, 1)
    want = orc.reconstruct_full(cores)
    got = with_env("TRG_RECON_SIMT", None,
                   lambda: trg.DeviceTensor(ctx, dims, dtype).synthesize(cores).numpy())
    assert relerr(got, want) < (1e-13 if dtype == np.float64 else 1e-6)


def test_rse_f32_near_exact_fit_dmma(trg):
    """fp32 fits below RSE 1e-2 are re-measured in fp64 arithmetic: that pass is the DMMA kernel."""
    dims, ranks = [60, 24, 18], [6, 6, 6]
    cores = orc.random_factors(dims, ranks, 5)
    xf = orc.reconstruct_full(cores).astype(np.float32)
    want = orc.rse(xf.astype(np.float64), orc.reconstruct_full(cores))
    assert want < 1e-2
    got = trg.rse(xf, cores)
    assert abs(got - want) <= 1e-4 * want
