"""Multi-rank (last-mode slab) host logic on CPU with torch.distributed gloo.

The product's partition (trg_shard_range) and test-matrix placement
(trg_sketch_offsets) drive the same dataflow libtrg runs under NCCL
(runtime.cpp run_sketch): per-rank Omega rows regenerated from the global
stream, partial Y_n summed by allreduce for n < N-1, the last mode's Y rows
scattered into a zeroed I x K buffer and allreduced, the last shrink with the
rank's rows of Q_{N-1} followed by an allreduce of P. The dense algebra here is
the oracle (checker); the assertions are that world_size 2 and 3 reproduce the
unsharded reference sketch (P, Q_n) of the oracle within 1e-12.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle_ref as orc


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _omega(seed, draw_off, col_off, rows_glob, ncols, K):
    """Omega rows [col_off, col_off + ncols) of the reference test matrix (sketch.hpp:32-38)."""
    om = np.empty((ncols, K))
    for k in range(K):
        om[:, k] = orc.gaussian(seed, ncols, skip=draw_off + col_off + rows_glob * k)
    return om


def _sharded_sketch(rank, world, x, K, seed, variant):
    import paper_1901_01652_b200 as trg

    dims = list(x.shape)
    N = len(dims)
    lo, hi = trg.shard_range(dims[-1], rank, world)
    rows_glob, col_off, draw_off = trg.sketch_offsets(dims, K, rank, world, variant)
    xloc = np.asfortranarray(x[..., lo:hi])

    def allreduce(a):
        t = torch.from_numpy(np.ascontiguousarray(a))
        dist.all_reduce(t)
        return t.numpy()

    Qs = [np.eye(dims[n], K[n]) for n in range(N)]
    cur = xloc  # sequential: the shrinking working tensor; fused: every Y_n from X
    for n in range(N):
        if rows_glob[n] == 0:
            continue
        Xn = orc.unfold(xloc if variant == 1 else cur, n)
        om = _omega(seed, draw_off[n], col_off[n], rows_glob[n], Xn.shape[1], K[n])
        if n < N - 1:
            Y = allreduce(Xn @ om)
        else:
            Yfull = np.zeros((dims[n], K[n]))
            Yfull[lo:hi] = Xn @ om  # local rows of the sharded mode
            Y = allreduce(Yfull)
        Qs[n] = orc.economy_q(Y)
        if variant == 0:
            cur = _shrink(cur, n, Qs[n], N, lo, hi, allreduce)
    if variant == 1:
        cur = xloc
        for n in range(N):
            if rows_glob[n] != 0:
                cur = _shrink(cur, n, Qs[n], N, lo, hi, allreduce)
    if K[-1] == dims[-1]:  # last mode unprojected: zero-padded gather by allreduce
        shp = list(cur.shape)
        full = np.zeros(shp[:-1] + [dims[-1]], order="F")
        full[..., lo:hi] = cur
        cur = allreduce(full.reshape(-1, order="F")).reshape(shp[:-1] + [dims[-1]], order="F")
    return cur, Qs


def _shrink(cur, n, Q, N, lo, hi, allreduce):
    if n < N - 1:
        return orc.mode_n_product(cur, n, Q.T)
    part = orc.mode_n_product(cur, n, Q[lo:hi].T)
    flat = allreduce(part.reshape(-1, order="F"))
    return flat.reshape(part.shape, order="F")


def _worker(rank, world, port, case, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dims, K, variant = case
        x = np.asfortranarray(np.random.default_rng(7).standard_normal(dims))
        P, Qs = _sharded_sketch(rank, world, x, K, 3, variant)
        if rank == 0:
            want_P, want_Q, _ = orc.sketch(x, K, 3, variant)
            errs = [float(np.abs(P - want_P).max() / np.abs(want_P).max())]
            errs += [float(np.abs(a - b).max()) for a, b in zip(Qs, want_Q)]
            out.put(errs)
    finally:
        dist.destroy_process_group()


CASES = [
    ((12, 10, 9), (4, 3, 5), 0),       # all modes projected, uneven last-mode shards
    ((8, 7, 6, 5), (3, 7, 2, 3), 0),   # mode 1 skipped (no draws)
    ((9, 8, 7), (3, 4, 7), 0),         # last mode skipped: padded gather of P
    ((10, 9, 8), (3, 3, 3), 1),        # fused variant: Omega sized against X
]


@pytest.mark.parametrize("world,case", [(2, c) for c in CASES] + [(3, CASES[0]), (3, CASES[2])])
def test_sharded_sketch_matches_unsharded_oracle(world, case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    errs = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert max(errs) < 1e-12, errs


def test_offsets_partition_the_reference_stream():
    """Rank-local Omega blocks tile the unsharded test matrix exactly (no gaps, no overlap)."""
    import paper_1901_01652_b200 as trg

    dims, K = [6, 5, 7], [2, 3, 4]
    full_rows, full_cols, full_D = trg.sketch_offsets(dims, K, 0, 1)
    for world in (2, 3, 7):
        seen = {n: [] for n in range(len(dims) - 1)}
        for r in range(world):
            lo, hi = trg.shard_range(dims[-1], r, world)
            rows, cols, D = trg.sketch_offsets(dims, K, r, world)
            assert rows == full_rows and D == full_D
            for n in range(len(dims) - 1):
                ncols = full_rows[n] // dims[-1] * (hi - lo)
                seen[n].append((cols[n], cols[n] + ncols))
        for n, spans in seen.items():
            spans.sort()
            assert spans[0][0] == 0 and spans[-1][1] == full_rows[n]
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
