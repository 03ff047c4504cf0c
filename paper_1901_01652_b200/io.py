"""DTEN / TRNG containers (the reference's on-disk formats, io.hpp:84-129 and
tr_factors.hpp:161-200), host-side, for exchanging tensors and TR factors with
the reference tools.

DTEN: magic "DTEN", u32 version (1), u32 order N >= 1, N x u64 extents (each >= 1),
then prod(I_n) little-endian f64 values, first index fastest.
TRNG: magic "TRNG", u32 version (1), u32 core count >= 1, then the cores as
consecutive DTEN records; every core is (R_n, I_n, R_{n+1 mod N}).
Both round-trip bit-exactly. Malformed input raises FormatError (io.hpp:16-20).
"""
import struct

import numpy as np


class FormatError(RuntimeError):
    """Malformed or unreadable on-disk data (the reference's format_error)."""


def _open(path_or_file, mode):
    if hasattr(path_or_file, "read" if "r" in mode else "write"):
        return path_or_file, False
    try:
        return open(path_or_file, mode), True
    except OSError as e:
        verb = "reading" if "r" in mode else "writing"
        raise FormatError(f"cannot open '{path_or_file}' for {verb}") from e


def _read_exact(f, n, what):
    b = f.read(n)
    if len(b) != n:
        raise FormatError(f"unexpected end of file while reading {what}")
    return b


def _write_dten(f, t):
    a = np.asarray(t, dtype=np.float64)
    if a.ndim < 1:
        raise ValueError("DenseTensor: order must be at least 1")
    f.write(b"DTEN")
    f.write(struct.pack("<II", 1, a.ndim))
    f.write(struct.pack(f"<{a.ndim}Q", *a.shape))
    f.write(np.ascontiguousarray(a.reshape(-1, order="F")).astype("<f8", copy=False).tobytes())


def _read_dten(f):
    if _read_exact(f, 4, "DTEN magic") != b"DTEN":
        raise FormatError("not a DTEN file (bad magic)")
    (version,) = struct.unpack("<I", _read_exact(f, 4, "DTEN version"))
    if version != 1:
        raise FormatError(f"unsupported DTEN version {version}")
    (order,) = struct.unpack("<I", _read_exact(f, 4, "DTEN order"))
    if order == 0:
        raise FormatError("DTEN order must be at least 1")
    shape = []
    for _ in range(order):
        (d,) = struct.unpack("<Q", _read_exact(f, 8, "DTEN extent"))
        if d == 0:
            raise FormatError("DTEN extents must be positive")
        shape.append(d)
    n = int(np.prod(shape))
    data = np.frombuffer(_read_exact(f, 8 * n, "DTEN values"), dtype="<f8").astype(np.float64)
    return data.reshape(shape, order="F")


def write_dten(path_or_file, t):
    f, own = _open(path_or_file, "wb")
    try:
        _write_dten(f, t)
    finally:
        if own:
            f.close()


def read_dten(path_or_file):
    f, own = _open(path_or_file, "rb")
    try:
        return _read_dten(f)
    finally:
        if own:
            f.close()


def write_trng(path_or_file, cores):
    cores = [np.asarray(c, dtype=np.float64) for c in cores]
    _check_ring(cores, ValueError)
    f, own = _open(path_or_file, "wb")
    try:
        f.write(b"TRNG")
        f.write(struct.pack("<II", 1, len(cores)))
        for c in cores:
            _write_dten(f, c)
    finally:
        if own:
            f.close()


def read_trng(path_or_file):
    f, own = _open(path_or_file, "rb")
    try:
        if _read_exact(f, 4, "TRNG magic") != b"TRNG":
            raise FormatError("not a TRNG file (bad magic)")
        (version,) = struct.unpack("<I", _read_exact(f, 4, "TRNG version"))
        if version != 1:
            raise FormatError(f"unsupported TRNG version {version}")
        (n,) = struct.unpack("<I", _read_exact(f, 4, "TRNG core count"))
        if n == 0:
            raise FormatError("TRNG must contain at least one core")
        cores = [_read_dten(f) for _ in range(n)]
    finally:
        if own:
            f.close()
    try:
        _check_ring(cores, ValueError)
    except ValueError as e:
        raise FormatError(f"TRNG cores are inconsistent: {e}") from e
    return cores


def _check_ring(cores, exc):
    """TRFactors invariants (tr_factors.hpp:22-71): order-3 cores whose ranks close the ring."""
    if not cores:
        raise exc("TRFactors: need at least one core")
    for n, c in enumerate(cores):
        if c.ndim != 3:
            raise exc(f"TRFactors: core {n} must have order 3")
        nxt = cores[(n + 1) % len(cores)]
        if c.shape[2] != nxt.shape[0]:
            raise exc(f"TRFactors: rank mismatch between core {n} and core {(n + 1) % len(cores)}")
