"""ctypes binding of libtrg.so (include/trg.h).

The library is built in-tree by paper_1901_01652_b200/build.py. There is no
CPU fallback: if libtrg.so is missing or no sm_100 device is present the
calls raise, they never silently compute elsewhere.
"""
import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TRG_LIB_PATH") or os.path.join(HERE, "libtrg.so")  # override: A/B builds (development)

c_i64p = ctypes.POINTER(ctypes.c_int64)
c_dp = ctypes.POINTER(ctypes.c_double)
c_vp = ctypes.c_void_p

# every symbol declared in include/trg.h (checked by tests/test_capi.py)
EXPORTS = [
    "trg_abi_version", "trg_last_error", "trg_device_count",
    "trg_ctx_create", "trg_nccl_unique_id", "trg_ctx_create_dist", "trg_loopback_create",
    "trg_loopback_destroy", "trg_ctx_create_loopback", "trg_ctx_destroy", "trg_ctx_synchronize",
    "trg_ctx_stream", "trg_ctx_set_profiling", "trg_ctx_kernel_stats", "trg_ctx_kernel_labels",
    "trg_ctx_launch_count", "trg_ctx_reset_stats", "trg_shard_range", "trg_sketch_offsets",
    "trg_tensor_create", "trg_tensor_info", "trg_tensor_upload", "trg_tensor_download", "trg_tensor_device_ptr",
    "trg_tensor_synthesize", "trg_tensor_destroy",
    "trg_sketch_run", "trg_sketch_projected", "trg_sketch_basis", "trg_sketch_y", "trg_sketch_qr_path",
    "trg_sketch_elapsed_ms", "trg_sketch_destroy", "trg_thin_qr", "trg_omega",
    "trg_mode_n_product", "trg_back_project", "trg_rse", "trg_sketch_lift_back", "trg_lift_back",
    "trg_decompose", "trg_decompose_host", "trg_report_ranks", "trg_report_cores_len", "trg_report_cores",
    "trg_report_rse_history", "trg_report_sweeps", "trg_report_timings", "trg_report_projected",
    "trg_report_destroy",
]

TRG_OK, TRG_EINVAL, TRG_ERANGE, TRG_ECUDA, TRG_ENCCL, TRG_ENUMERIC, TRG_ENODEV = 0, 1, 2, 3, 4, 5, 6
TRG_F32, TRG_F64 = 0, 1
TRG_SEQUENTIAL, TRG_FUSED = 0, 1
TRG_OMEGA_KHATRI_RAO = 16  # flag OR-ed into the variant (trg.h)
TRG_ALS, TRG_SVD = 0, 1


class TrgError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"libtrg error {code}: {msg}")
        self.code = code


class NoDeviceError(TrgError):
    pass


_lib = None


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built; run `python -m paper_1901_01652_b200.build` "
                              "(there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        lib.trg_last_error.restype = ctypes.c_char_p
        _lib = lib
    return _lib


def check(rc):
    if rc == TRG_OK:
        return
    msg = load().trg_last_error().decode(errors="replace")
    if rc == TRG_EINVAL:
        raise ValueError(msg)  # std::invalid_argument
    if rc == TRG_ERANGE:
        raise IndexError(msg)  # std::out_of_range
    if rc == TRG_ENODEV:
        raise NoDeviceError(rc, msg)
    raise TrgError(rc, msg)


def call(name, *args):
    check(getattr(load(), name)(*args))


def i64(seq):
    import numpy as np

    arr = np.ascontiguousarray(np.asarray(seq, dtype=np.int64))
    return arr, arr.ctypes.data_as(c_i64p)
