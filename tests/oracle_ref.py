"""ctypes front-end of the CPU oracle (oracle/build/liboracle.so).

TEST INFRASTRUCTURE: imported only by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs, as the checker. Tensors are numpy float64 arrays
in the reference's first-index-fastest layout (tensor.hpp:33-38), i.e. numpy
order='F'. Cores are lists of (R_n, I_n, R_{n+1}) Fortran-ordered arrays.
"""
import ctypes
import os

import numpy as np

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_LIB_PATH = os.path.join(_ROOT, "oracle", "build", "liboracle.so")

_i64p = ctypes.POINTER(ctypes.c_int64)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_dp = ctypes.POINTER(ctypes.c_double)

_lib = None


class OracleError(Exception):
    pass


def build():
    import subprocess

    subprocess.run(["make", "-s", "-C", os.path.join(_ROOT, "oracle")], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = ctypes.CDLL(_LIB_PATH)
        _lib.oracle_last_error.restype = ctypes.c_char_p
        _lib.oracle_max_threads.restype = ctypes.c_int
    return _lib


def _check(rc):
    if rc == 1:
        raise ValueError(lib().oracle_last_error().decode())
    if rc == 2:
        raise IndexError(lib().oracle_last_error().decode())
    if rc != 0:
        raise OracleError(lib().oracle_last_error().decode())


def _i64(seq):
    arr = np.ascontiguousarray(np.asarray(seq, dtype=np.int64))
    return arr, arr.ctypes.data_as(_i64p)


def _f64(a):
    arr = np.asarray(a, dtype=np.float64)
    flat = np.ascontiguousarray(arr.reshape(-1, order="F"))
    return flat, flat.ctypes.data_as(_dp)


def _out(n):
    arr = np.zeros(int(n), dtype=np.float64)
    return arr, arr.ctypes.data_as(_dp)


def set_threads(n):
    lib().oracle_set_threads(int(n))


def max_threads():
    return int(lib().oracle_max_threads())


def splitmix_u64(seed, n):
    out = np.zeros(n, dtype=np.uint64)
    _check(lib().oracle_splitmix_u64(ctypes.c_uint64(seed), ctypes.c_int64(n), out.ctypes.data_as(_u64p)))
    return out


def gaussian(seed, n, skip=0):
    out, p = _out(n)
    _check(lib().oracle_gaussian(ctypes.c_uint64(seed), ctypes.c_int64(skip), ctypes.c_int64(n), p))
    return out


def unfold(x, mode, tr=False):
    x = np.asarray(x, dtype=np.float64)
    d, dp = _i64(x.shape)
    xf, xp = _f64(x)
    rows = x.shape[mode]
    out, op = _out(x.size)
    _check(lib().oracle_unfold(x.ndim, dp, xp, int(mode), int(tr), op))
    return out.reshape((rows, x.size // rows), order="F")


def fold(m, mode, shape, tr=False):
    d, dp = _i64(shape)
    mf, mp = _f64(m)
    out, op = _out(int(np.prod(shape)))
    _check(lib().oracle_fold(len(shape), dp, mp, int(mode), int(tr), op))
    return out.reshape(shape, order="F")


def mode_n_product(x, mode, m):
    x = np.asarray(x, dtype=np.float64)
    m = np.asarray(m, dtype=np.float64)
    d, dp = _i64(x.shape)
    xf, xp = _f64(x)
    mf, mp = _f64(m)
    shape = list(x.shape)
    shape[mode] = m.shape[0]
    out, op = _out(int(np.prod(shape)))
    _check(lib().oracle_mode_n_product(x.ndim, dp, xp, int(mode), ctypes.c_int64(m.shape[0]),
                                       ctypes.c_int64(m.shape[1]), mp, op))
    return out.reshape(shape, order="F")


def economy_q(y):
    y = np.asarray(y, dtype=np.float64)
    yf, yp = _f64(y)
    k = min(y.shape)
    out, op = _out(y.shape[0] * k)
    _check(lib().oracle_economy_q(ctypes.c_int64(y.shape[0]), ctypes.c_int64(y.shape[1]), yp, op))
    return out.reshape((y.shape[0], k), order="F")


def svd(a):
    """The oracle's thin SVD (one-sided Jacobi standing in for BDCSVD): (s, U, V)."""
    a = np.asarray(a, dtype=np.float64)
    af, ap = _f64(a)
    k = min(a.shape)
    s, sp = _out(k)
    u, up = _out(a.shape[0] * k)
    v, vp = _out(a.shape[1] * k)
    _check(lib().oracle_svd(ctypes.c_int64(a.shape[0]), ctypes.c_int64(a.shape[1]), ap, sp, up, vp))
    return s, u.reshape((a.shape[0], k), order="F"), v.reshape((a.shape[1], k), order="F")


def sketch(x, K, seed, variant=0):
    """Returns (projected, bases, ys) — ys[n] is Y_n (zeros for skipped modes)."""
    x = np.asarray(x, dtype=np.float64)
    d, dp = _i64(x.shape)
    k, kp = _i64(K)
    xf, xp = _f64(x)
    proj, pp = _out(int(np.prod(K)))
    nb = int(sum(int(a) * int(b) for a, b in zip(x.shape, K)))
    bases, bp = _out(nb)
    ys, yp = _out(nb)
    _check(lib().oracle_sketch(x.ndim, dp, xp, kp, ctypes.c_uint64(seed), int(variant), pp, bp, yp))
    outb, outy, off = [], [], 0
    for I, Kn in zip(x.shape, K):
        outb.append(bases[off:off + I * Kn].reshape((I, Kn), order="F"))
        outy.append(ys[off:off + I * Kn].reshape((I, Kn), order="F"))
        off += I * Kn
    return proj.reshape(tuple(K), order="F"), outb, outy


def kr_factor_layout(dims, K, variant=0):
    """Draw layout of the opt-in Khatri-Rao test matrices (include/trg.h TRG_OMEGA_KHATRI_RAO):
    per projected mode n, the factors F_{n,m} (m != n, ascending) of S_m x K_n draws, column-major,
    consecutive in the stream from draw 0; S = the working shape of mode n (K_m for m < n in the
    sequential variant, I_m otherwise). Returns ({n: {m: (offset, S_m)}}, total draws)."""
    layout, total = {}, 0
    for n, (I, Kn) in enumerate(zip(dims, K)):
        if Kn == I:
            continue
        layout[n] = {}
        for m in range(len(dims)):
            if m == n:
                continue
            S = K[m] if (m < n and variant == 0) else dims[m]
            layout[n][m] = (total, S)
            total += S * Kn
    return layout, total


def kr_omega(draws, layout_n, Kn):
    """Omega_n(c, k) = prod_m F_{n,m}(i_m, k), c = sum_m i_m stride_m (first index fastest)."""
    cols = []
    for k in range(Kn):
        v = np.ones(1)
        for m in sorted(layout_n):
            off, S = layout_n[m]
            f = draws[off:off + S * Kn].reshape((S, Kn), order="F")[:, k]
            v = np.kron(f, v)  # mode m varies slower than the modes before it
        cols.append(v)
    return np.stack(cols, axis=1)


def kr_sketch(x, K, seed, variant=0):
    """The projection of sketch() with Khatri-Rao test matrices: returns (projected, bases, ys)."""
    x = np.asarray(x, dtype=np.float64)
    dims, N = list(x.shape), x.ndim
    layout, total = kr_factor_layout(dims, K, variant)
    draws = gaussian(seed, total) if total else np.zeros(0)
    bases = [np.eye(I) for I in dims]
    ys = [np.zeros((I, Kn)) for I, Kn in zip(dims, K)]
    P = x.copy()
    for n in range(N):
        if n not in layout:
            continue
        src = P if variant == 0 else x
        ys[n] = unfold(src, n) @ kr_omega(draws, layout[n], K[n])
        bases[n] = economy_q(ys[n])
        if variant == 0:
            P = mode_n_product(P, n, bases[n].T)
    if variant != 0:
        for n in layout:
            P = mode_n_product(P, n, bases[n].T)
    return P, bases, ys


def lift_back(projected, bases):
    projected = np.asarray(projected, dtype=np.float64)
    K = projected.shape
    dims = [b.shape[0] for b in bases]
    k, kp = _i64(K)
    d, dp = _i64(dims)
    pf, pp = _f64(projected)
    bf, bp = _f64(np.concatenate([np.asarray(b, dtype=np.float64).reshape(-1, order="F") for b in bases]))
    out, op = _out(int(np.prod(dims)))
    _check(lib().oracle_lift_back(len(K), kp, pp, dp, bp, op))
    return out.reshape(dims, order="F")


def _cores_flat(cores):
    return np.concatenate([np.asarray(c, dtype=np.float64).reshape(-1, order="F") for c in cores])


def _split_cores(flat, dims, ranks):
    N = len(dims)
    out, off = [], 0
    for n in range(N):
        shape = (int(ranks[n]), int(dims[n]), int(ranks[(n + 1) % N]))
        sz = int(np.prod(shape))
        out.append(flat[off:off + sz].reshape(shape, order="F").copy())
        off += sz
    return out


def reconstruct_full(cores, mode=0):
    dims = [c.shape[1] for c in cores]
    ranks = [c.shape[0] for c in cores]
    d, dp = _i64(dims)
    r, rp = _i64(ranks)
    cf, cp = _f64(_cores_flat(cores))
    out, op = _out(int(np.prod(dims)))
    _check(lib().oracle_reconstruct_full(len(dims), dp, rp, cp, int(mode), op))
    return out.reshape(dims, order="F")


def reconstruct_elementwise(cores, index):
    dims = [c.shape[1] for c in cores]
    ranks = [c.shape[0] for c in cores]
    d, dp = _i64(dims)
    r, rp = _i64(ranks)
    cf, cp = _f64(_cores_flat(cores))
    ix, ixp = _i64(index)
    out = ctypes.c_double()
    _check(lib().oracle_reconstruct_elementwise(len(dims), dp, rp, cp, ixp, ctypes.byref(out)))
    return out.value


def subchain(cores, mode):
    dims = [c.shape[1] for c in cores]
    ranks = [c.shape[0] for c in cores]
    N = len(dims)
    d, dp = _i64(dims)
    r, rp = _i64(ranks)
    cf, cp = _f64(_cores_flat(cores))
    P = int(np.prod(dims)) // dims[mode]
    shape = (ranks[(mode + 1) % N], P, ranks[mode])
    out, op = _out(int(np.prod(shape)))
    _check(lib().oracle_subchain(N, dp, rp, cp, int(mode), op))
    return out.reshape(shape, order="F")


def rse(ref, approx):
    a, ap = _f64(ref)
    b, bp = _f64(approx)
    out = ctypes.c_double()
    _check(lib().oracle_rse(ctypes.c_int64(a.size), ap, bp, ctypes.byref(out)))
    return out.value


def back_project(small_cores, bases):
    K = [c.shape[1] for c in small_cores]
    ranks = [c.shape[0] for c in small_cores]
    dims = [b.shape[0] for b in bases]
    k, kp = _i64(K)
    r, rp = _i64(ranks)
    d, dp = _i64(dims)
    cf, cp = _f64(_cores_flat(small_cores))
    bf, bp = _f64(np.concatenate([np.asarray(b, dtype=np.float64).reshape(-1, order="F") for b in bases]))
    n = sum(ranks[i] * dims[i] * ranks[(i + 1) % len(dims)] for i in range(len(dims)))
    out, op = _out(n)
    _check(lib().oracle_back_project(len(K), kp, rp, cp, dp, bp, op))
    return _split_cores(out, dims, ranks)


class Report:
    def __init__(self, cores, rse_history, sweeps_run, discarded_sq=None):
        self.cores = cores
        self.rse_history = rse_history
        self.sweeps_run = sweeps_run
        self.discarded_sq = discarded_sq

    @property
    def ranks(self):
        return [c.shape[0] for c in self.cores]


def _run_report(fn, dims, max_sweeps, extra_tail=()):
    N = len(dims)
    ranks_out = np.zeros(N, dtype=np.int64)
    cores_len = ctypes.c_int64()
    n_rse = ctypes.c_int64()
    sweeps = ctypes.c_int64()
    rse_cap = int(max_sweeps) + 2
    rse_out, rsp = _out(rse_cap)
    # first call learns the core length, second fills it
    _check(fn(ranks_out.ctypes.data_as(_i64p), None, ctypes.c_int64(0), ctypes.byref(cores_len), rsp,
              ctypes.c_int64(rse_cap), ctypes.byref(n_rse), ctypes.byref(sweeps), *extra_tail))
    cores, cp = _out(cores_len.value)
    _check(fn(ranks_out.ctypes.data_as(_i64p), cp, cores_len, ctypes.byref(cores_len), rsp,
              ctypes.c_int64(rse_cap), ctypes.byref(n_rse), ctypes.byref(sweeps), *extra_tail))
    return _split_cores(cores, dims, ranks_out), list(rse_out[:n_rse.value]), sweeps.value


def solve(method, x, ranks=None, tol=0.0, max_sweeps=50, seed=0):
    """method 'als' -> trals (solvers.hpp:297), 'svd' -> trsvd (solvers.hpp:382)."""
    x = np.asarray(x, dtype=np.float64)
    d, dp = _i64(x.shape)
    xf, xp = _f64(x)
    rk = _i64(ranks) if ranks is not None else (None, None)
    disc = ctypes.c_double()

    def fn(ranks_out, cores_out, cap, cores_len, rse_out, rse_cap, n_rse, sweeps):
        return lib().oracle_solve(0 if method == "als" else 1, x.ndim, dp, xp, rk[1], ctypes.c_double(tol),
                                  ctypes.c_int64(max_sweeps), ctypes.c_uint64(seed), ranks_out, cores_out, cap,
                                  cores_len, rse_out, rse_cap, n_rse, sweeps, ctypes.byref(disc))

    cores, hist, sw = _run_report(fn, x.shape, max_sweeps)
    return Report(cores, hist, sw, disc.value)


def rtrd(method, x, K, ranks=None, tol=0.0, max_sweeps=50, cfg_seed=0, spec_seed=0, variant=0):
    """rtrals (method 'als', sketch.hpp:154) / rtrsvd ('svd', sketch.hpp:161)."""
    x = np.asarray(x, dtype=np.float64)
    d, dp = _i64(x.shape)
    xf, xp = _f64(x)
    k, kp = _i64(K)
    rk = _i64(ranks) if ranks is not None else (None, None)

    def fn(ranks_out, cores_out, cap, cores_len, rse_out, rse_cap, n_rse, sweeps):
        return lib().oracle_rtrd(0 if method == "als" else 1, int(variant), x.ndim, dp, xp, rk[1],
                                 ctypes.c_double(tol), ctypes.c_int64(max_sweeps), ctypes.c_uint64(cfg_seed), kp,
                                 ctypes.c_uint64(spec_seed), ranks_out, cores_out, cap, cores_len, rse_out, rse_cap,
                                 n_rse, sweeps)

    cores, hist, sw = _run_report(fn, x.shape, max_sweeps)
    return Report(cores, hist, sw)


def random_factors(dims, ranks, seed, scale=1.0):
    d, dp = _i64(dims)
    r, rp = _i64(ranks)
    N = len(dims)
    n = sum(ranks[i] * dims[i] * ranks[(i + 1) % N] for i in range(N))
    out, op = _out(n)
    _check(lib().oracle_random_factors(N, dp, rp, ctypes.c_uint64(seed), ctypes.c_double(scale), op))
    return _split_cores(out, dims, ranks)


def add_noise(x, snr_db, seed):
    x = np.asarray(x, dtype=np.float64)
    xf, xp = _f64(x)
    out, op = _out(x.size)
    _check(lib().oracle_add_noise(ctypes.c_int64(x.size), xp, ctypes.c_double(snr_db), ctypes.c_uint64(seed), op))
    return out.reshape(x.shape, order="F")
