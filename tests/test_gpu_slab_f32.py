"""fp32 sketch / shrink for modes n >= 1 (csrc/slab_f32.cu) against the fp64 oracle on the
fp32-rounded input (sketch.hpp:62-89). Mode 0 is skipped (K_0 = I_0) or projected so that mode 1
sees the (left, dim, K) of the BASELINE fp32 configs' later modes: C3 (20, 1000, 20),
C4 (64, 1024, 64) and (4096, 200, 32), C5 (12, 60, 12) ... plus odd extents and K."""
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


CASES = [
    ((20, 1000, 9), (20, 20, 5)),       # C3's mode 1: left 20, dim 1000, K 20
    ((64, 1024, 5), (64, 64, 5)),       # C4's mode 1: left 64, dim 1024, K 64
    ((64, 64, 200), (64, 64, 32)),      # C4's mode 2: left 4096, dim 200, K 32
    ((12, 60, 60, 20), (12, 12, 12, 20)),  # C5-like: left 12, dim 60, K 12
    ((60, 60, 40), (12, 12, 7)),        # mode 0 projected first (fp32 P^(1) on the FFMA shrink)
    ((16, 37, 23), (16, 5, 3)),         # odd dim, K
    ((8, 100, 11), (8, 33, 4)),         # K = 33 -> two k-groups
    ((4, 7, 300), (4, 1, 3)),           # K = 1 (and mode 2 with K <= rank 4 of its unfolding)
    ((12, 12, 60, 30), (12, 12, 12, 7)),  # left 144 in l-blocks, partial slab blocks (slab_st.cu)
    ((20, 400, 33), (20, 20, 9)),       # d-chunks over several CTA groups, ragged right
    ((6, 50, 40), (6, 10, 5)),          # left 6: not a multiple of 4 (the slab_f32.cu kernels)
    ((1728, 60), (1728, 12)),           # left 1728, right 1 (C5's mode-4 shape class)
    ((60, 60, 30), (12, 60, 30)),       # mode 0 only, short fibres (slab_st.cu k_st0_*: C5's mode 0)
    ((400, 50, 21), (20, 50, 21)),      # mode-0 sketch with long fibres, K 20 (C3's mode-0 class)
    ((1000, 7, 9), (20, 7, 9)),         # C3's I_0 = 1000 with few columns (partial fibre stages)
    # tcgen05 sketch for modes >= 1 (tc_f32.cu k_tc_sketch_n_f32: left % 32 == 0, K >= 32)
    ((96, 150, 20), (96, 40, 8)),       # left 96 (three 32-column chunks), K 40 (Kp 48)
    ((64, 300, 7), (64, 48, 3)),        # ragged 256-row d tile (300 = 256 + 44)
    ((32, 520, 3, 4), (32, 33, 3, 2)),  # three d tiles, K 33 (Kp 48), right 12
    ((128, 64, 9), (128, 64, 9)),       # mode 1 skipped; left 128 ... then mode 2 left 8192
    ((32, 60, 50), (32, 32, 7)),        # dim 60 <= 64: one M = 64 tile per item
    # tcgen05 shrink for modes >= 1 (tc_f32.cu k_tc_ttm_n_f32: left % 64 == 0, K >= 32)
    ((64, 100, 13), (64, 32, 5)),       # two slabs per tile, odd slab count, dim 100 (partial 32-d chunk), K 32
    ((32, 45, 10), (32, 36, 3)),        # left 32: four slabs per tile, right 10 (a partial last tile)
    ((128, 70, 6), (128, 48, 2)),       # M = 128 tiles, K 48 (Kp 48)
    ((64, 1024, 3), (64, 64, 3)),       # C4's mode-1 shrink class (left 64, dim 1024, K 64)
]


@pytest.mark.parametrize("dims,K", CASES)
def test_slab_f32_modes(trg, dims, K):
    rng = np.random.default_rng(sum(dims) + 3 * sum(K))
    x = rng.standard_normal(dims).astype(np.float32)
    proj, bases, ys = orc.sketch(x.astype(np.float64), K, 11)
    got = trg.sketch(x, trg.ProjectionSpec(list(K), 11))
    for n in range(len(dims)):
        if K[n] != dims[n]:
            assert relerr(got.sketches[n], ys[n]) < 2e-5, n
            assert relerr(got.bases[n], bases[n]) < 1e-4, n
    assert relerr(got.projected, proj) < 1e-4
