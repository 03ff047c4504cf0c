"""Python mirror of the reference's public API for the rTRD hot path.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/tenring/sketch.hpp and solvers.hpp:

  ProjectionSpec, SolverConfig, SketchResult, SolveReport   sketch.hpp:18-28, solvers.hpp:24-38
  sketch(x, spec)                                          sketch.hpp:62-89
  back_project(z, sketch_result)                           sketch.hpp:106-122
  rtrals(x, cfg, spec) / rtrsvd(x, cfg, spec)              sketch.hpp:154-165
  rse(x, cores)                                            solvers.hpp:47-54 (x vs reconstruct_full(cores))
  gaussian_matrix(rows, cols, seed, offset)                sketch.hpp:32-38
  mode_n_product(x, mode, m)                               tensor.hpp:193-207

std::invalid_argument surfaces as ValueError, std::out_of_range as IndexError.
Tensors are numpy arrays in the reference layout (first index fastest, i.e.
numpy order='F'); all compute runs in libtrg.so on the B200.
"""
import ctypes
import weakref
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib as L


@dataclass
class ProjectionSpec:
    sketch_dims: List[int]
    seed: int = 0
    # "gaussian": the reference's i.i.d. test matrices (sketch.hpp:32-38). "khatri_rao": opt-in
    # structured test matrices, products of per-mode Gaussian factors (trg.h TRG_OMEGA_KHATRI_RAO);
    # different results, no per-element draws
    omega: str = "gaussian"


def _variant(variant, spec):
    if spec.omega == "gaussian":
        return variant
    if spec.omega == "khatri_rao":
        return variant | L.TRG_OMEGA_KHATRI_RAO
    raise ValueError(f"ProjectionSpec.omega must be 'gaussian' or 'khatri_rao', not {spec.omega!r}")


@dataclass
class SolverConfig:
    ranks: Optional[List[int]] = None
    tolerance: float = 0.0
    max_sweeps: int = 50
    seed: int = 0


@dataclass
class SketchResult:
    projected: np.ndarray
    bases: List[np.ndarray]
    sketches: List[np.ndarray] = field(default_factory=list)
    elapsed_ms: float = 0.0
    qr_householder: List[int] = field(default_factory=list)


@dataclass
class SolveReport:
    factors: List[np.ndarray]
    rse_history: List[float]
    sweeps_run: int
    elapsed_seconds: float
    timings_ms: dict = field(default_factory=dict)
    projected: Optional[np.ndarray] = None

    @property
    def ranks(self):
        return [c.shape[0] for c in self.factors]


def _dtype_code(dt):
    dt = np.dtype(dt)
    if dt == np.float64:
        return L.TRG_F64
    if dt == np.float32:
        return L.TRG_F32
    raise ValueError("DenseTensor: dtype must be float32 or float64")


class Context:
    """One CUDA device (one process per GPU); optionally a rank of an NCCL group
    in which tensors are sharded along their last mode."""

    def __init__(self, device=0, rank=0, world=1, nccl_id=None, loopback=None):
        self._h = ctypes.c_void_p()
        if loopback is not None:
            L.call("trg_ctx_create_loopback", ctypes.c_int(device), ctypes.c_int(rank), loopback.handle,
                   ctypes.byref(self._h))
            world = loopback.world
        elif world == 1:
            L.call("trg_ctx_create", ctypes.c_int(device), ctypes.byref(self._h))
        else:
            buf = (ctypes.c_ubyte * 128).from_buffer_copy(bytes(nccl_id))
            L.call("trg_ctx_create_dist", ctypes.c_int(device), ctypes.c_int(rank), ctypes.c_int(world), buf,
                   ctypes.byref(self._h))
        self.device, self.rank, self.world = device, rank, world
        # handles created on this context; closed before the context itself so that a
        # child's destructor never runs against a destroyed context (interpreter exit)
        self._children = weakref.WeakSet()

    def _adopt(self, child):
        self._children.add(child)

    @staticmethod
    def nccl_unique_id():
        buf = (ctypes.c_ubyte * 128)()
        L.call("trg_nccl_unique_id", buf)
        return bytes(buf)

    @property
    def handle(self):
        return self._h

    def synchronize(self):
        L.call("trg_ctx_synchronize", self._h)

    def stream(self):
        s = ctypes.c_void_p()
        L.call("trg_ctx_stream", self._h, ctypes.byref(s))
        return s.value

    def set_profiling(self, on):
        L.call("trg_ctx_set_profiling", self._h, ctypes.c_int(1 if on else 0))

    def kernel_stats(self, label=None):
        ms = ctypes.c_double()
        n = ctypes.c_int64()
        L.call("trg_ctx_kernel_stats", self._h, label.encode() if label else None, ctypes.byref(ms), ctypes.byref(n))
        return ms.value, n.value

    def kernel_labels(self):
        buf = ctypes.create_string_buffer(1 << 16)
        L.call("trg_ctx_kernel_labels", self._h, buf, ctypes.c_int64(1 << 16))
        return [s for s in buf.value.decode().split("\n") if s]

    def launch_count(self):
        n = ctypes.c_int64()
        L.call("trg_ctx_launch_count", self._h, ctypes.byref(n))
        return n.value

    def reset_stats(self):
        L.call("trg_ctx_reset_stats", self._h)

    def close(self):
        if self._h:
            for child in list(self._children):
                try:
                    child.close()
                except Exception:
                    pass
            L.call("trg_ctx_destroy", self._h)
            self._h = ctypes.c_void_p()

    @property
    def alive(self):
        return bool(self._h)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LoopbackGroup:
    """trg_loopback (include/trg.h): `world` ranks of the sharded path in this process, one host
    thread and one Context(loopback=group) each, all on one device. Collectives are host
    barriers around rank-ordered same-device reductions; for tests of the sharded CUDA path."""

    def __init__(self, world):
        self._h = ctypes.c_void_p()
        L.call("trg_loopback_create", ctypes.c_int(world), ctypes.byref(self._h))
        self.world = world

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            L.call("trg_loopback_destroy", self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run_loopback(world, fn, device=0, timeout=900.0):
    """fn(ctx, rank) on `world` loopback ranks (one thread and one context each); returns the
    list of results in rank order and re-raises the first rank's exception. ctypes releases
    the GIL inside every libtrg call, so the ranks' host code runs concurrently."""
    import threading

    group = LoopbackGroup(world)
    out, err = [None] * world, [None] * world

    def body(r):
        ctx = None
        try:
            ctx = Context(device, r, loopback=group)
            out[r] = fn(ctx, r)
        except BaseException as e:  # noqa: BLE001 - reported to the caller below
            err[r] = e
        finally:
            if ctx is not None:
                try:
                    ctx.close()
                except Exception:
                    pass

    ts = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout)
    if any(t.is_alive() for t in ts):
        raise TimeoutError(f"loopback ranks still running after {timeout} s: {[e for e in err if e]}")
    group.close()
    for e in err:
        if e is not None:
            raise e
    return out


def shard_range(extent, rank, world):
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    L.call("trg_shard_range", ctypes.c_int64(extent), ctypes.c_int(rank), ctypes.c_int(world), ctypes.byref(lo),
           ctypes.byref(hi))
    return lo.value, hi.value


def sketch_offsets(dims, K, rank=0, world=1, variant=L.TRG_SEQUENTIAL):
    """Per-mode test-matrix placement for a rank's last-mode slab (pure host, no device):
    Omega_n(c, k) = reference draw draw_off[n] + col_off[n] + c + rows_glob[n] * k
    for local unfolding column c; rows_glob[n] == 0 marks a skipped mode."""
    N = len(dims)
    d, dp = L.i64(dims)
    k, kp = L.i64(K)
    rows = np.zeros(N, dtype=np.int64)
    cols = np.zeros(N, dtype=np.int64)
    draw = np.zeros(N, dtype=np.uint64)
    L.call("trg_sketch_offsets", ctypes.c_int(N), dp, kp, ctypes.c_int(rank), ctypes.c_int(world),
           ctypes.c_int(variant), rows.ctypes.data_as(L.c_i64p), cols.ctypes.data_as(L.c_i64p),
           draw.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
    return [int(v) for v in rows], [int(v) for v in cols], [int(v) for v in draw]


class DeviceTensor:
    """DenseTensor (tensor.hpp:42-108) resident in HBM; local last-mode slab when sharded."""

    def __init__(self, ctx, shape, dtype=np.float64):
        self.ctx = ctx
        self.shape = tuple(int(s) for s in shape)
        self.dtype = np.dtype(dtype)
        self._h = ctypes.c_void_p()
        d, dp = L.i64(self.shape)
        L.call("trg_tensor_create", ctx.handle, ctypes.c_int(_dtype_code(dtype)), ctypes.c_int(len(self.shape)), dp,
               ctypes.byref(self._h))
        lo, hi = ctypes.c_int64(), ctypes.c_int64()
        L.call("trg_tensor_info", self._h, None, None, None, ctypes.byref(lo), ctypes.byref(hi))
        self.lo, self.hi = lo.value, hi.value
        ctx._adopt(self)

    @property
    def local_shape(self):
        return self.shape[:-1] + (self.hi - self.lo,)

    @classmethod
    def from_numpy(cls, ctx, x, dtype=None):
        x = np.asarray(x)
        t = cls(ctx, x.shape if ctx.world == 1 else x.shape, dtype or x.dtype)
        t.upload(x if ctx.world == 1 else x[..., t.lo:t.hi])
        return t

    def upload(self, local):
        a = np.asarray(local, dtype=self.dtype)
        if a.shape != self.local_shape:
            raise ValueError(f"upload: expected local shape {self.local_shape}, got {a.shape}")
        flat = np.ascontiguousarray(a.reshape(-1, order="F"))
        L.call("trg_tensor_upload", self._h, flat.ctypes.data_as(ctypes.c_void_p))

    def numpy(self):
        out = np.empty(int(np.prod(self.local_shape)), dtype=self.dtype)
        L.call("trg_tensor_download", self._h, out.ctypes.data_as(ctypes.c_void_p))
        return out.reshape(self.local_shape, order="F")

    def device_ptr(self):
        p = ctypes.c_void_p()
        n = ctypes.c_int64()
        L.call("trg_tensor_device_ptr", self._h, ctypes.byref(p), ctypes.byref(n))
        return p.value, n.value

    def synthesize(self, cores, rescale01=False, snr_db=None, noise_seed=0):
        ranks = [c.shape[0] for c in cores]
        r, rp = L.i64(ranks)
        flat = np.ascontiguousarray(np.concatenate([np.asarray(c, np.float64).reshape(-1, order="F") for c in cores]))
        L.call("trg_tensor_synthesize", self._h, rp, flat.ctypes.data_as(L.c_dp), ctypes.c_int(1 if rescale01 else 0),
               ctypes.c_double(float("inf") if snr_db is None else float(snr_db)), ctypes.c_uint64(noise_seed))
        return self

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            if self.ctx.alive:  # a closed context has already closed its children
                L.call("trg_tensor_destroy", self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DeviceSketch:
    """Handle of a projection left on the device (trg_sketch)."""

    def __init__(self, ctx, x, spec, variant=L.TRG_SEQUENTIAL):
        self.ctx = ctx
        self._x = x  # keeps the input alive while the enqueued projection reads it
        self.dims = list(x.shape)
        self.K = [int(k) for k in spec.sketch_dims]
        self._h = ctypes.c_void_p()
        if len(self.K) != len(self.dims):
            raise ValueError("sketch: projection size list must match tensor order")
        k, kp = L.i64(self.K)
        L.call("trg_sketch_run", ctx.handle, x.handle, kp, ctypes.c_uint64(spec.seed),
               ctypes.c_int(_variant(variant, spec)), ctypes.byref(self._h))
        ctx._adopt(self)

    def projected(self):
        out = np.empty(int(np.prod(self.K)), dtype=np.float64)
        L.call("trg_sketch_projected", self._h, out.ctypes.data_as(L.c_dp))
        return out.reshape(self.K, order="F")

    def basis(self, n):
        out = np.empty(self.dims[n] * self.K[n], dtype=np.float64)
        L.call("trg_sketch_basis", self._h, ctypes.c_int(n), out.ctypes.data_as(L.c_dp))
        return out.reshape((self.dims[n], self.K[n]), order="F")

    def sketch_matrix(self, n):
        out = np.empty(self.dims[n] * self.K[n], dtype=np.float64)
        L.call("trg_sketch_y", self._h, ctypes.c_int(n), out.ctypes.data_as(L.c_dp))
        return out.reshape((self.dims[n], self.K[n]), order="F")

    def qr_householder(self, n):
        v = ctypes.c_int()
        L.call("trg_sketch_qr_path", self._h, ctypes.c_int(n), ctypes.byref(v))
        return v.value

    def elapsed_ms(self):
        ms = ctypes.c_double()
        L.call("trg_sketch_elapsed_ms", self._h, ctypes.byref(ms))
        return ms.value

    def result(self):
        N = len(self.dims)
        return SketchResult(projected=self.projected(), bases=[self.basis(n) for n in range(N)],
                            sketches=[self.sketch_matrix(n) for n in range(N)], elapsed_ms=self.elapsed_ms(),
                            qr_householder=[self.qr_householder(n) for n in range(N)])

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            if self.ctx.alive:
                L.call("trg_sketch_destroy", self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx = None


def default_context():
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


def _as_device(x, ctx):
    if isinstance(x, DeviceTensor):
        return x, False
    x = np.asarray(x)
    if x.dtype not in (np.float32, np.float64):
        x = x.astype(np.float64)
    return DeviceTensor.from_numpy(ctx, x), True


def sketch(x, spec, variant=L.TRG_SEQUENTIAL, ctx=None):
    """sketch.hpp:62-89 — returns SketchResult(projected, bases) computed on the GPU."""
    ctx = ctx or default_context()
    xt, _ = _as_device(x, ctx)
    sk = DeviceSketch(ctx, xt, spec, variant)
    try:
        return sk.result()
    finally:
        sk.close()


def gaussian_matrix(rows, cols, seed, offset=0, ctx=None):
    """Reference test matrix (sketch.hpp:32-38) starting at stream draw `offset`."""
    ctx = ctx or default_context()
    out = np.empty(int(rows) * int(cols), dtype=np.float64)
    L.call("trg_omega", ctx.handle, ctypes.c_uint64(seed), ctypes.c_uint64(offset), ctypes.c_int64(rows),
           ctypes.c_int64(cols), out.ctypes.data_as(L.c_dp))
    return out.reshape((rows, cols), order="F")


def economy_q(y, ctx=None, return_path=False):
    """detail::economy_q (sketch.hpp:45-53) on the device: thin Q with diag(R) >= 0."""
    ctx = ctx or default_context()
    y = np.asfortranarray(np.asarray(y, dtype=np.float64))
    m, k = y.shape
    q = np.empty((m, k), dtype=np.float64, order="F")
    hh = ctypes.c_int(0)
    L.call("trg_thin_qr", ctx.handle, ctypes.c_int64(m), ctypes.c_int64(k), y.ctypes.data_as(L.c_dp),
           q.ctypes.data_as(L.c_dp), ctypes.byref(hh))
    return (q, hh.value) if return_path else q


def mode_n_product(x, mode, m, ctx=None):
    """tensor.hpp:193-207 on the GPU (dtype of x)."""
    ctx = ctx or default_context()
    xt, _ = _as_device(x, ctx)
    m = np.asarray(m, dtype=np.float64)
    if m.ndim != 2 or mode < 0 or mode >= len(xt.shape) or m.shape[1] != xt.shape[mode]:
        if 0 <= mode < len(xt.shape):
            raise ValueError("mode_n_product: inner dimensions do not match")
        raise IndexError(f"DenseTensor: mode {mode} out of range")
    flat = np.ascontiguousarray(m.reshape(-1, order="F"))
    h = ctypes.c_void_p()
    L.call("trg_mode_n_product", ctx.handle, xt.handle, ctypes.c_int(mode), ctypes.c_int64(m.shape[0]),
           flat.ctypes.data_as(L.c_dp), ctypes.byref(h))
    shape = list(xt.shape)
    shape[mode] = m.shape[0]
    out = DeviceTensor.__new__(DeviceTensor)
    out.ctx, out.shape, out.dtype, out._h, out.lo, out.hi = ctx, tuple(shape), xt.dtype, h, 0, shape[-1]
    res = out.numpy()
    out.close()
    return res


def lift_back(sk, ctx=None):
    """lift_back (sketch.hpp:93-101): P x_0 Q_0 x_1 Q_1 ..., the plain TRP approximation of x.

    A DeviceSketch is lifted from its resident P and Q_n (result: DeviceTensor). A host
    SketchResult is uploaded and lifted on the device (result: numpy); like the reference, a
    basis that is square and exactly the identity is skipped.
    """
    if isinstance(sk, DeviceSketch):
        h = ctypes.c_void_p()
        L.call("trg_sketch_lift_back", sk.handle, ctypes.byref(h))
        out = DeviceTensor.__new__(DeviceTensor)
        shape = tuple(sk.dims)
        out.ctx, out.shape, out._h, out.lo, out.hi = sk.ctx, shape, h, 0, shape[-1]
        dt = ctypes.c_int()
        L.call("trg_tensor_info", h, ctypes.byref(dt), None, None, None, None)
        out.dtype = np.dtype(np.float32 if dt.value == L.TRG_F32 else np.float64)
        sk.ctx._adopt(out)
        return out
    ctx = ctx or default_context()
    P = np.asarray(sk.projected, dtype=np.float64)
    bases = [np.asarray(q, dtype=np.float64) for q in sk.bases]
    if len(bases) != P.ndim or any(q.ndim != 2 or q.shape[1] != P.shape[n] for n, q in enumerate(bases)):
        raise ValueError("lift_back: bases must be I_n x K_n with K_n the projected extents")
    dims = [q.shape[0] for q in bases]
    d, dp = L.i64(dims)
    k, kp = L.i64(P.shape)
    flatP = np.ascontiguousarray(P.reshape(-1, order="F"))
    flats = [np.ascontiguousarray(q.reshape(-1, order="F")) for q in bases]
    ptrs = (L.c_dp * len(flats))(*[f.ctypes.data_as(L.c_dp) for f in flats])
    h = ctypes.c_void_p()
    L.call("trg_lift_back", ctx.handle, ctypes.c_int(len(dims)), dp, kp, flatP.ctypes.data_as(L.c_dp), ptrs,
           ctypes.byref(h))
    out = DeviceTensor.__new__(DeviceTensor)
    out.ctx, out.shape, out.dtype, out._h, out.lo, out.hi = ctx, tuple(dims), np.dtype(np.float64), h, 0, dims[-1]
    res = out.numpy()
    out.close()
    return res


def _flat_cores(cores):
    return np.ascontiguousarray(np.concatenate([np.asarray(c, np.float64).reshape(-1, order="F") for c in cores]))


def _split(flat, dims, ranks):
    N = len(dims)
    out, off = [], 0
    for n in range(N):
        shp = (int(ranks[n]), int(dims[n]), int(ranks[(n + 1) % N]))
        sz = int(np.prod(shp))
        out.append(flat[off:off + sz].reshape(shp, order="F").copy())
        off += sz
    return out


def back_project(z, sk, ctx=None):
    """sketch.hpp:106-122: G_n = Z_n x_2 Q_n. `sk` is a live DeviceSketch."""
    ctx = ctx or sk.ctx
    K = [c.shape[1] for c in z]
    ranks = [c.shape[0] for c in z]
    if len(z) != len(sk.dims):
        raise ValueError("back_project: need one basis per core")
    k, kp = L.i64(K)
    r, rp = L.i64(ranks)
    flat = _flat_cores(z)
    N = len(z)
    out = np.empty(sum(ranks[n] * sk.dims[n] * ranks[(n + 1) % N] for n in range(N)), dtype=np.float64)
    L.call("trg_back_project", ctx.handle, ctypes.c_int(N), kp, rp, flat.ctypes.data_as(L.c_dp), sk.handle,
           out.ctypes.data_as(L.c_dp))
    return _split(out, sk.dims, ranks)


def rse(x, cores, ctx=None):
    """rse(x, reconstruct_full(cores)) (solvers.hpp:47-54) fused on the GPU."""
    ctx = ctx or default_context()
    xt, _ = _as_device(x, ctx)
    ranks = [c.shape[0] for c in cores]
    r, rp = L.i64(ranks)
    flat = _flat_cores(cores)
    out = ctypes.c_double()
    L.call("trg_rse", ctx.handle, xt.handle, rp, flat.ctypes.data_as(L.c_dp), ctypes.byref(out))
    return out.value


def _report(h, dims):
    N = len(dims)
    ranks = np.zeros(N, dtype=np.int64)
    L.call("trg_report_ranks", h, ranks.ctypes.data_as(L.c_i64p))
    n = ctypes.c_int64()
    L.call("trg_report_cores_len", h, ctypes.byref(n))
    cores = np.empty(n.value, dtype=np.float64)
    L.call("trg_report_cores", h, cores.ctypes.data_as(L.c_dp))
    L.call("trg_report_rse_history", h, None, ctypes.byref(n))
    hist = np.empty(n.value, dtype=np.float64)
    L.call("trg_report_rse_history", h, hist.ctypes.data_as(L.c_dp), ctypes.byref(n))
    sw = ctypes.c_int64()
    L.call("trg_report_sweeps", h, ctypes.byref(sw))
    ms = np.zeros(6, dtype=np.float64)
    L.call("trg_report_timings", h, ms.ctypes.data_as(L.c_dp))
    L.call("trg_report_projected", h, None, ctypes.byref(n))
    proj = np.empty(n.value, dtype=np.float64)
    L.call("trg_report_projected", h, proj.ctypes.data_as(L.c_dp), ctypes.byref(n))
    L.call("trg_report_destroy", h)
    keys = ["h2d", "sketch", "small_solve", "back_project", "rse", "total"]
    return SolveReport(factors=_split(cores, dims, ranks), rse_history=list(hist), sweeps_run=int(sw.value),
                       elapsed_seconds=ms[5] / 1e3, timings_ms=dict(zip(keys, ms.tolist())), projected=proj)


def decompose(x, method, cfg, spec, variant=L.TRG_SEQUENTIAL, ctx=None):
    """randomized_decompose (sketch.hpp:126-147). x: DeviceTensor (device-resident) or a host
    array (the H2D copy is then part of the call, trg_decompose_host)."""
    ctx = ctx or (x.ctx if isinstance(x, DeviceTensor) else default_context())
    m = L.TRG_ALS if method in ("als", L.TRG_ALS) else L.TRG_SVD
    dims = list(x.shape)
    if len(spec.sketch_dims) != len(dims):
        raise ValueError("sketch: projection size list must match tensor order")
    k, kp = L.i64(spec.sketch_dims)
    rk = L.i64(cfg.ranks) if cfg.ranks is not None else (None, None)
    if rk[0] is not None and len(rk[0]) != len(dims):
        raise ValueError("trals: rank vector length must equal tensor order")
    h = ctypes.c_void_p()
    common = (ctypes.c_int(m), rk[1], ctypes.c_double(cfg.tolerance), ctypes.c_int64(cfg.max_sweeps),
              ctypes.c_uint64(cfg.seed), kp, ctypes.c_uint64(spec.seed), ctypes.c_int(_variant(variant, spec)),
              ctypes.byref(h))
    if isinstance(x, DeviceTensor):
        L.call("trg_decompose", ctx.handle, x.handle, *common)
    else:
        a = np.asarray(x)
        if a.dtype not in (np.float32, np.float64):
            a = a.astype(np.float64)
        d, dp = L.i64(a.shape)
        flat = np.ascontiguousarray(a.reshape(-1, order="F"))
        L.call("trg_decompose_host", ctx.handle, ctypes.c_int(_dtype_code(a.dtype)), ctypes.c_int(a.ndim), dp,
               flat.ctypes.data_as(ctypes.c_void_p), *common)
    return _report(h, dims)


def rtrals(x, cfg, spec, variant=L.TRG_SEQUENTIAL, ctx=None):
    """sketch.hpp:154-158"""
    return decompose(x, "als", cfg, spec, variant, ctx)


def rtrsvd(x, cfg, spec, variant=L.TRG_SEQUENTIAL, ctx=None):
    """sketch.hpp:161-165"""
    return decompose(x, "svd", cfg, spec, variant, ctx)
