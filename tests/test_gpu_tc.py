"""tcgen05 (kind::tf32, 3xTF32) fp32 mode-0 sketch and shrink (csrc/tc_f32.cu) against the
fp64 oracle on the fp32-rounded input: Y_0, Q_0 and P (sketch.hpp:80-85). Shapes cover M-tile
tails (I_0 not a multiple of 32 / 128), N padding (K not a multiple of 16), column tails and
more CTAs than tiles. The bound on Y_0 is far tighter than plain TF32 could meet (~5e-4)."""
import numpy as np
import pytest

import oracle_ref as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def trg():
    import paper_1901_01652_b200 as trg

    return trg


def relerr(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


SHAPES = [
    ((60, 40, 30), (12, 6, 5)),        # C5's mode 0: one M tile of 128 rows, half padding
    ((1000, 30, 7), (20, 5, 4)),       # C3's I_0 and K_0: 1000 = 31.25 row blocks
    ((1024, 64, 50), (64, 8, 8)),      # C4's I_0 and K_0: all 512 TMEM columns
    ((132, 33, 65), (33, 6, 9)),       # K = 33 -> 48 columns
    ((100, 2000, 3), (16, 10, 3)),     # many column tiles per CTA
    ((64, 257, 9), (1, 7, 5)),         # K = 1
    ((256, 31, 29), (40, 9, 7)),
]


@pytest.fixture
def forced(monkeypatch):
    # every shape below on the tensor-core kernels (the default dispatch takes them only where
    # they beat the FFMA kernels: tc_f32.cu)
    monkeypatch.setenv("TRG_TC_FORCE", "1")


@pytest.mark.parametrize("dims,K", SHAPES)
def test_tc_mode0_parity(trg, forced, dims, K):
    rng = np.random.default_rng(sum(dims) + sum(K))
    x = rng.standard_normal(dims).astype(np.float32)
    proj, bases, ys = orc.sketch(x.astype(np.float64), K, 3)
    got = trg.sketch(x, trg.ProjectionSpec(list(K), 3))
    ey, eq, ep = relerr(got.sketches[0], ys[0]), relerr(got.bases[0], bases[0]), relerr(got.projected, proj)
    print(f"{dims} {K}: Y0 {ey:.2e} Q0 {eq:.2e} P {ep:.2e}")
    assert ey < 2e-5
    assert eq < 1e-4 and ep < 1e-4
