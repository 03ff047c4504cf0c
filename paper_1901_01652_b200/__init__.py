"""B200-native randomized tensor-ring decomposition hot path (arXiv 1901.01652).

Product: libtrg.so (paper_1901_01652_b200/csrc, C ABI in include/trg.h) with
hand-written sm_100a kernels for the tensor random projection (sketch, thin
QR, TTM shrink), back-projection and the fused reconstruction error, plus the
host small solve. This package is the Python mirror of the reference API.
"""
from .api import (  # noqa: F401
    Context,
    DeviceSketch,
    DeviceTensor,
    LoopbackGroup,
    ProjectionSpec,
    SketchResult,
    SolveReport,
    SolverConfig,
    back_project,
    decompose,
    default_context,
    gaussian_matrix,
    economy_q,
    lift_back,
    mode_n_product,
    rse,
    rtrals,
    rtrsvd,
    run_loopback,
    shard_range,
    sketch_offsets,
    sketch,
)
from .io import FormatError, read_dten, read_trng, write_dten, write_trng  # noqa: F401
