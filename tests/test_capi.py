"""CPU-side checks of the C ABI boundary: libtrg.so loads, exports every symbol
include/trg.h declares, reports errors through the reference's exception
mapping, and refuses to compute without a device (no CPU fallback)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "trg.h")).read()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(trg_\w+)\(", src, flags=re.M)))


def test_header_and_binding_agree():
    from paper_1901_01652_b200 import _lib

    assert header_symbols() == sorted(_lib.EXPORTS)


def test_library_exports_every_header_symbol():
    from paper_1901_01652_b200 import _lib

    lib = _lib.load()
    missing = [s for s in header_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.trg_abi_version() == 1


def test_shard_range_partition():
    import paper_1901_01652_b200 as trg

    for extent in (1, 7, 100, 1000, 60):
        for world in (1, 2, 4, 8):
            if world > extent:
                continue
            spans = [trg.shard_range(extent, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == extent
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [h - l for l, h in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        trg.shard_range(10, 3, 2)


def test_no_cpu_fallback_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("device present")
    import paper_1901_01652_b200 as trg
    from paper_1901_01652_b200._lib import NoDeviceError

    with pytest.raises(NoDeviceError):
        trg.Context(0)
    with pytest.raises(NoDeviceError):
        trg.sketch([[1.0, 2.0], [3.0, 4.0]], trg.ProjectionSpec([1, 1], 0))


def test_last_error_is_thread_local_string():
    from paper_1901_01652_b200 import _lib

    lib = _lib.load()
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    rc = lib.trg_shard_range(ctypes.c_int64(0), 0, 1, ctypes.byref(lo), ctypes.byref(hi))
    assert rc == 1
    assert b"extent" in lib.trg_last_error()
