"""The sharded (multi-GPU) CUDA path executed on ONE GPU through the loopback communicator.

X is sharded along its last mode. Every rank runs the real sharded
program on its own host thread and context: its slab's sketch with the GLOBAL test-matrix rows
(col_off != 0, rows_glob != local columns), the world > 1 QR path, the scatter of the last
mode's local Y rows, the shrink with the local rows of Q_{N-1}, and the sums of the partials.
Only the collective differs from the NCCL contexts: a rank-ordered same-device sum between two
host barriers (trg.h trg_loopback). Results are compared with the UNSHARDED oracle
(sketch.hpp:62-89) at the north-star tolerances, on every rank (the results are replicated).
"""
import numpy as np
import pytest

import oracle_ref as orc

pytestmark = pytest.mark.gpu

F64_TOL, F32_TOL = 1e-10, 1e-4


@pytest.fixture(scope="module")
def trg():
    import paper_1901_01652_b200 as trg

    return trg


def relerr(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def tr_tensor(dims, ranks, seed, snr=None):
    x = orc.reconstruct_full(orc.random_factors(dims, ranks, seed))
    return orc.add_noise(x, snr, seed + 1) if snr is not None else x


CASES = [
    # dims, K, world, dtype
    ([23, 17, 19], [5, 4, 6], 2, np.float64),
    ([23, 17, 19], [5, 17, 6], 3, np.float64),          # mode 1 skipped
    ([40, 34, 28, 22], [6, 4, 4, 4], 3, np.float64),    # modes >= 1 on the TMA slab kernels
    ([9, 8, 7, 6, 13], [3, 4, 2, 3, 5], 8, np.float64), # order 5, shards of 1 and 2 slices
    ([64, 48, 37], [16, 8, 12], 8, np.float64),
    ([23, 17, 19], [5, 4, 19], 3, np.float64),          # last mode skipped: padded gather of P
    ([64, 48, 37], [16, 8, 12], 3, np.float32),
    ([50, 40, 30, 21], [8, 6, 5, 7], 8, np.float32),
]


@pytest.mark.parametrize("dims,K,world,dtype", CASES)
def test_loopback_sketch_matches_unsharded_oracle(trg, dims, K, world, dtype):
    x = tr_tensor(dims, [3] * len(dims), 5, snr=30.0).astype(dtype)
    proj, bases, ys = orc.sketch(x.astype(np.float64), K, 7)
    tol = F64_TOL if dtype == np.float64 else F32_TOL

    def rank(ctx, r):
        t = trg.DeviceTensor.from_numpy(ctx, x)
        assert (t.lo, t.hi) == trg.shard_range(dims[-1], r, world)
        sk = trg.DeviceSketch(ctx, t, trg.ProjectionSpec(K, 7))
        out = (sk.projected(), [sk.basis(n) for n in range(len(dims))], [sk.sketch_matrix(n) for n in range(len(dims))])
        sk.close()
        t.close()
        return out

    for P, Q, Y in trg.run_loopback(world, rank):
        assert relerr(P, proj) < tol
        for n in range(len(dims)):
            assert relerr(Q[n], bases[n]) < tol, n
            if K[n] != dims[n]:
                assert relerr(Y[n], ys[n]) < tol, n


def test_loopback_synthesis_and_decompose_match_oracle(trg):
    """K9 synthesis (noise norms and the [0,1] rescale reduced across ranks) and Algorithm 1
    end to end (sketch, small solve, back-projection, final RSE reduced across ranks)."""
    dims, R, K, world = [30, 26, 23], [3, 3, 3], [9, 9, 9], 3
    cores = orc.random_factors(dims, R, 0)
    x = orc.add_noise(orc.reconstruct_full(cores), 30.0, 1)
    want = orc.rtrd("als", x, K, ranks=R, max_sweeps=6, cfg_seed=0, spec_seed=0)
    lo_hi = [trg.shard_range(dims[-1], r, world) for r in range(world)]

    def rank(ctx, r):
        t = trg.DeviceTensor(ctx, dims, np.float64).synthesize(cores, snr_db=30.0, noise_seed=1)
        slab = t.numpy()
        rep = trg.rtrals(t, trg.SolverConfig(ranks=R, max_sweeps=6, seed=0), trg.ProjectionSpec(K, 0))
        t.close()
        return slab, rep

    for r, (slab, rep) in enumerate(trg.run_loopback(world, rank)):
        lo, hi = lo_hi[r]
        assert relerr(slab, x[..., lo:hi]) < 1e-12
        assert rep.ranks == R
        np.testing.assert_allclose(rep.rse_history, want.rse_history, rtol=F64_TOL)
        for a, b in zip(rep.factors, want.cores):
            assert relerr(a, b) < F64_TOL


def test_loopback_rescaled_synthesis(trg):
    dims, R, world = [20, 18, 17], [2, 3, 2], 4
    cores = orc.random_factors(dims, R, 3)
    full = orc.reconstruct_full(cores)
    want = (full - full.min()) / (full.max() - full.min())  # global min / max across the shards

    def rank(ctx, r):
        t = trg.DeviceTensor(ctx, dims, np.float64).synthesize(cores, rescale01=True)
        out = (t.lo, t.hi, t.numpy())
        t.close()
        return out

    for lo, hi, slab in trg.run_loopback(world, rank):
        assert relerr(slab, want[..., lo:hi]) < 1e-12


def test_loopback_c5_eight_shards(trg):
    """BASELINE configs[4] (60^5 fp32, K=12) on 8 last-mode shards of 7 and 8 slices, against the
    unsharded host restatement of the projection (tests/test_gpu_configs.host_projection)."""
    from paper_1901_01652_b200.synthetic import CONFIGS, make_tensor
    from test_gpu_configs import host_projection

    cfg = CONFIGS["c5"]
    K, world = cfg["K"], 8

    def rank(ctx, r):
        t, _ = make_tensor(ctx, cfg, seed=0)
        slab = t.numpy()
        sk = trg.DeviceSketch(ctx, t, trg.ProjectionSpec(K, 0))
        out = (t.lo, t.hi, slab, sk.projected(), [sk.basis(n) for n in range(5)])
        sk.close()
        t.close()
        return out

    res = trg.run_loopback(world, rank)
    assert sorted(r[1] - r[0] for r in res) == [7, 7, 7, 7, 8, 8, 8, 8]
    x = np.concatenate([r[2] for r in res], axis=4)  # the global tensor from the shards
    del res[1:]  # keep rank 0's results only (host memory)
    Ys, Qs, P = host_projection(x, K, 0)
    _, _, _, gP, gQ = res[0]
    assert relerr(gP, P) < F32_TOL
    for n in range(5):
        assert relerr(gQ[n], Qs[n]) < F32_TOL
