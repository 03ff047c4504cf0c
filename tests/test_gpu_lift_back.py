"""lift_back (sketch.hpp:93-101) on the device against the oracle.

The device result (resident sketch, or a host SketchResult uploaded) must equal the oracle's
P x_0 Q_0 x_1 Q_1 ... within the fp64 bound; square exactly-identity bases are skipped, so a
projection with every mode skipped lifts back to X bit-exactly.
"""
import numpy as np
import pytest

import oracle_ref as orc

pytestmark = pytest.mark.gpu

CASES = [
    ((30, 20, 10), (6, 20, 4)),   # mode 1 skipped
    ((12, 11, 10, 9), (3, 4, 5, 2)),
    ((300, 7), (6, 3)),
    ((40,), (1,)),
]


@pytest.fixture(scope="module")
def trg():
    import paper_1901_01652_b200 as trg

    return trg


@pytest.mark.parametrize("dims,K", CASES)
def test_lift_back_matches_oracle(trg, dims, K):
    rng = np.random.default_rng(5)
    x = rng.standard_normal(dims)
    ctx = trg.default_context()
    xd = trg.DeviceTensor.from_numpy(ctx, x)
    sk = trg.DeviceSketch(ctx, xd, trg.ProjectionSpec(list(K), 3))
    res = sk.result()
    want = orc.lift_back(res.projected, res.bases)
    dev = trg.lift_back(sk)
    got = dev.numpy()
    assert got.shape == tuple(dims)
    assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)
    host = trg.lift_back(res)  # SketchResult path: uploaded, identity bases detected on the host
    assert np.linalg.norm(host - want) <= 1e-12 * np.linalg.norm(want)
    dev.close()
    sk.close()
    xd.close()


def test_lift_back_all_skipped_is_exact(trg):
    x = np.random.default_rng(6).standard_normal((5, 4, 3))
    ctx = trg.default_context()
    xd = trg.DeviceTensor.from_numpy(ctx, x)
    sk = trg.DeviceSketch(ctx, xd, trg.ProjectionSpec([5, 4, 3], 0))
    assert np.array_equal(trg.lift_back(sk).numpy(), x)
    res = sk.result()
    assert np.array_equal(trg.lift_back(res), x)


def test_lift_back_rejects_bad_bases(trg):
    res = trg.SketchResult(projected=np.zeros((2, 2)), bases=[np.zeros((5, 3)), np.zeros((4, 2))])
    with pytest.raises(ValueError):
        trg.lift_back(res)
