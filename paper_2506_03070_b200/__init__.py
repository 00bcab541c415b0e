"""paper_2506_03070_b200 -- B200-native sketch-and-precondition least squares.

Drop-in for the hot path of the reference header library ``sketchlsq``
(sparse-sign sketch generation, sketch apply, preconditioner build,
preconditioned LSQR), executed by hand-written sm_100a CUDA kernels in
``libslq_b200.so`` behind the C-ABI ``include/slq_b200.h``.
"""
from . import _capi  # noqa: F401  (raises ImportError if the library is not built)
from .api import (  # noqa: F401
    Context,
    CscMatrix,
    CudaError,
    DeviceMatrix,
    DimensionMismatch,
    Divergence,
    Error,
    GradientParams,
    InvalidArgument,
    InvalidDims,
    InvalidDistortion,
    InvalidSparsity,
    NcclError,
    OutOfMemory,
    Preconditioner,
    QrResult,
    RankDeficient,
    RejectionStats,
    RowPartition,
    SingularTriangular,
    SketchParams,
    SolveOptions,
    SolveReport,
    SparseDeviceMatrix,
    SparseSignSketch,
    Termination,
    Unsupported,
    apply,
    apply_M,
    apply_Mt,
    build_preconditioner,
    default_context,
    gd_params,
    gd_step_size,
    generate_sparse_sign,
    gradient_descent_hbm,
    hbm_params,
    householder_qr,
    initial_guess,
    lsqr,
    lsqr_one_sync,
    partition_rows,
    rejection_sample_columns,
    sketch_vector,
    solve,
    sparse_sign_block,
    tri_inverse,
    tri_upper_matvec,
    tri_upper_rmatvec,
)

LIB_PATH = _capi.LIB_PATH
__version__ = _capi.lib.slq_version().decode()
