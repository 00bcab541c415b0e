"""Python mirror of the reference's hot-path API (namespace ``sketchlsq``).

Same names, argument meaning and error behaviour as the C++ headers in
/root/reference/proj/include/sketchlsq (file:line in each docstring); every
call runs on the B200 through the C-ABI (``include/slq_b200.h``).  Matrices
are numpy float64 arrays in the reference's column-major convention
(``dense_matrix.hpp:14-35``); results are returned by value like the
reference.  There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as ct
import enum
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _capi as C

# ------------------------------------------------------------------ errors


class Error(RuntimeError):
    """errors.hpp:9-11 sketchlsq::Error"""


class RankDeficient(Error):
    """errors.hpp:16"""


class SingularTriangular(Error):
    """errors.hpp:21"""


class DimensionMismatch(Error):
    """errors.hpp:26"""


class InvalidSparsity(Error):
    """errors.hpp:31"""


class InvalidDims(Error):
    """errors.hpp:46"""


class InvalidDistortion(Error):
    """errors.hpp:39"""


class Divergence(Error):
    """errors.hpp:64"""


class CudaError(Error):
    pass


class NcclError(Error):
    pass


class OutOfMemory(Error):
    pass


class Unsupported(Error):
    pass


class InvalidArgument(Error):
    pass


_STATUS = {
    1: InvalidSparsity,
    2: InvalidDims,
    3: DimensionMismatch,
    4: RankDeficient,
    5: SingularTriangular,
    6: CudaError,
    7: NcclError,
    8: OutOfMemory,
    9: Unsupported,
    10: InvalidArgument,
    11: InvalidDistortion,
    12: Divergence,
}


def _check(code: int) -> None:
    if code != 0:
        msg = C.lib.slq_last_error().decode(errors="replace")
        raise _STATUS.get(code, Error)(msg)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _d(a):
    return None if a is None else a.ctypes.data_as(C.dp)


def _i(a):
    return None if a is None else a.ctypes.data_as(C.ip)


def _f64(a):
    return np.asfortranarray(a, dtype=np.float64)


def _vec(a):
    return np.ascontiguousarray(a, dtype=np.float64).reshape(-1)


# ----------------------------------------------------------------- context


class Context:
    """One device context (stream, workspace, optional NCCL communicator)."""

    def __init__(self, device: int = 0):
        h = C.vp()
        _check(C.lib.slq_ctx_create(device, ct.byref(h)))
        self.handle = h
        self.device = device
        self.rank = 0
        self.nranks = 1

    def close(self):
        if self.handle:
            C.lib.slq_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def synchronize(self):
        _check(C.lib.slq_ctx_synchronize(self.handle))

    @property
    def kernel_launches(self) -> int:
        return int(C.lib.slq_ctx_kernel_launches(self.handle))

    def set_stream(self, cuda_stream_ptr: int):
        _check(C.lib.slq_ctx_set_stream(self.handle, C.vp(cuda_stream_ptr)))

    # multi-GPU: replaces WorkerPool (distsim.hpp:77-146)
    @staticmethod
    def unique_id() -> bytes:
        buf = ct.create_string_buffer(128)
        _check(C.lib.slq_comm_unique_id(buf))
        return buf.raw

    def init_comm(self, uid: bytes, rank: int, nranks: int):
        _check(C.lib.slq_ctx_init_comm(self.handle, uid, rank, nranks))
        self.rank, self.nranks = rank, nranks

    def set_host_comm(self, comm, rank: int, nranks: int):
        """Collectives through the caller's host transport instead of NCCL
        (slq_ctx_set_host_comm): ``comm`` has allreduce_sum(buf),
        reduce_sum_root(buf) and broadcast_root(buf), each in place on a float64
        numpy view of the library's pinned staging buffer.  Every rank's solve
        then runs the same per-rank sequence as with NCCL (reduce of the sketch
        partials, rank-0 preconditioner, status / M / M^T / x0 broadcasts, one
        allreduce per LSQR iteration), one host round trip per collective."""
        import traceback

        def wrap(fn):
            def cb(_user, buf, count):
                try:
                    fn(np.ctypeslib.as_array(buf, shape=(count,)))
                    return 0
                except Exception:  # a failed collective surfaces as SLQ_NCCL on this rank
                    traceback.print_exc()
                    return 1
            return C.HostCollective(cb)

        self._host_comm = [wrap(comm.allreduce_sum), wrap(comm.reduce_sum_root), wrap(comm.broadcast_root)]
        hc = C.HostComm(*self._host_comm, None)
        _check(C.lib.slq_ctx_set_host_comm(self.handle, ct.byref(hc), rank, nranks))
        self.rank, self.nranks = rank, nranks


_tls = threading.local()


def default_context(device: int | None = None) -> Context:
    if device is None:
        device = getattr(_tls, "device", 0)
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    if device not in ctxs:
        ctxs[device] = Context(device)
    return ctxs[device]


def _ctx(ctx):
    return ctx if ctx is not None else default_context()


# ------------------------------------------------------------- data types


@dataclass
class CscMatrix:
    """csc_matrix.hpp:19-60"""
    rows: int
    cols: int
    values: np.ndarray
    row_indices: np.ndarray
    col_pointers: np.ndarray

    def nnz(self) -> int:
        return int(self.values.size)

    def todense(self) -> np.ndarray:
        A = np.zeros((self.rows, self.cols), order="F")
        for j in range(self.cols):
            s, e = self.col_pointers[j], self.col_pointers[j + 1]
            A[self.row_indices[s:e], j] = self.values[s:e]
        return A


@dataclass
class SparseSignSketch:
    """sketch.hpp:39-43"""
    matrix: CscMatrix
    zeta: int
    seed: int


@dataclass
class RejectionStats:
    """sketch.hpp:65-68"""
    columns_resampled: int = 0
    resample_rounds: int = 0


@dataclass
class QrResult:
    """qr.hpp:15-18"""
    Q: np.ndarray
    R: np.ndarray


@dataclass
class Preconditioner:
    """preconditioner.hpp:15-30"""
    M: np.ndarray
    Q: np.ndarray | None
    build_time: float = 0.0
    d: int = 0

    def n(self) -> int:
        return self.M.shape[0]

    @staticmethod
    def identity(n: int) -> "Preconditioner":
        return Preconditioner(np.eye(n, order="F"), np.eye(n, order="F"), 0.0, n)


class Termination(enum.IntEnum):
    """solve_report.hpp:11"""
    Tolerance = 0
    MaxIter = 1
    Breakdown = 2

    def __str__(self):
        return self.name.lower()


@dataclass
class SolveOptions:
    """lsqr.hpp:14-22 (+ opt-in backward-error stop, an extension)"""
    eps: float = 1e-10
    maxit: int = 100
    x_star: np.ndarray | None = None
    track_true_residual: bool = False
    on_bidiag: object = None  # callable(t, u_norm, v_norm)
    backward_tol: float = 0.0
    a_norm_est: float = 0.0


@dataclass
class SolveReport:
    """solve_report.hpp:23-49"""
    iterates_error: list = field(default_factory=list)
    residual_estimate: list = field(default_factory=list)
    residual_true: list = field(default_factory=list)
    iterations: int = 0
    termination: Termination = Termination.MaxIter
    sync_count: int = 0
    broadcasts: int = 0
    init_reductions: int = 0
    init_broadcasts: int = 0
    wall_time: float = 0.0
    backward_error: float = -1.0

    def reductions_per_iteration(self) -> float:
        return (self.sync_count - self.init_reductions) / self.iterations if self.iterations > 0 else 0.0

    def broadcasts_per_iteration(self) -> float:
        return (self.broadcasts - self.init_broadcasts) / self.iterations if self.iterations > 0 else 0.0

    def to_json(self) -> dict:
        """solve_report.hpp:51-66"""
        j = {
            "iterations": self.iterations,
            "termination": str(self.termination),
            "sync_count": self.sync_count,
            "broadcasts": self.broadcasts,
            "init_reductions": self.init_reductions,
            "init_broadcasts": self.init_broadcasts,
            "reductions_per_iteration": self.reductions_per_iteration(),
            "broadcasts_per_iteration": self.broadcasts_per_iteration(),
            "wall_time": self.wall_time,
            "residual_estimate": list(self.residual_estimate),
        }
        if self.iterates_error:
            j["iterates_error"] = list(self.iterates_error)
        if self.residual_true:
            j["residual_true"] = list(self.residual_true)
        return j


@dataclass
class RowPartition:
    """distsim.hpp:21-29"""
    m: int
    boundaries: list

    def blocks(self) -> int:
        return len(self.boundaries) - 1

    def begin(self, k: int) -> int:
        return self.boundaries[k]

    def end(self, k: int) -> int:
        return self.boundaries[k + 1]

    def size(self, k: int) -> int:
        return self.end(k) - self.begin(k)


# --------------------------------------------------------------- sketching


def _stats_out(stats, st):
    if stats is not None:
        stats.columns_resampled += st.columns_resampled
        stats.resample_rounds += st.resample_rounds


def sparse_sign_block(d, zeta, seed, col_begin, col_end, stats=None, ctx=None) -> CscMatrix:
    """sketch.hpp:149-173 detail::sparse_sign_block (global column ids)."""
    ncols = int(col_end - col_begin)
    rows = np.zeros(max(ncols * zeta, 1), np.int64)
    vals = np.zeros(max(ncols * zeta, 1), np.float64)
    colptr = np.zeros(ncols + 1, np.int64)
    st = C.RejectionStats()
    _check(C.lib.slq_generate_sparse_sign(_ctx(ctx).handle, d, col_begin, ncols, zeta, seed & (2**64 - 1),
                                          _i(rows), _d(vals), _i(colptr), ct.byref(st)))
    _stats_out(stats, st)
    return CscMatrix(d, ncols, vals[: ncols * zeta], rows[: ncols * zeta], colptr)


def generate_sparse_sign(d, m, zeta=None, seed=None, stats=None, ctx=None) -> SparseSignSketch:
    """sketch.hpp:178-194 generate_sparse_sign(d, m, zeta, seed[, stats]) and the
    SketchParams overload sketch.hpp:191 (pass a SketchParams as ``d``)."""
    if isinstance(d, SketchParams):
        p = d
        return generate_sparse_sign(p.d, m, p.zeta, p.seed, stats=zeta if stats is None else stats, ctx=ctx)
    mat = sparse_sign_block(d, zeta, seed, 0, m, stats, ctx)
    return SparseSignSketch(mat, zeta, seed)


def rejection_sample_columns(d, m, zeta, seed, stats=None, ctx=None) -> np.ndarray:
    """sketch.hpp:105-124"""
    out = np.zeros(max(m * zeta, 1), np.int64)
    st = C.RejectionStats()
    _check(C.lib.slq_rejection_sample_columns(_ctx(ctx).handle, d, m, zeta, seed & (2**64 - 1), _i(out),
                                              ct.byref(st)))
    _stats_out(stats, st)
    return out[: m * zeta]


@dataclass
class SketchParams:
    """sketch.hpp:20-35 (sparse sign kind only)"""
    d: int = 0
    zeta: int = 8
    seed: int = 0

    def validate(self, m: int, n: int) -> None:
        if not (n < self.d <= m):
            raise InvalidDims(f"SketchParams: need n < d <= m, got n={n} d={self.d} m={m}")
        if not (1 <= self.zeta <= self.d):
            raise InvalidSparsity("SketchParams: need 1 <= zeta <= d")


def apply(S: SparseSignSketch, A, ctx=None) -> np.ndarray:
    """sketch.hpp:297 apply(SparseSignSketch, DenseMatrix) -> csc_matrix.hpp:103-120,
    sketch.hpp:298 apply(SparseSignSketch, CscMatrix) -> csc_matrix.hpp:123-136.
    Bit-identical to the reference (same accumulation order, IEEE mul+add)."""
    if isinstance(A, CscMatrix):
        M = S.matrix
        if M.cols != A.rows:
            raise DimensionMismatch("spmm(csc,csc): inner dimensions disagree")
        Y = np.zeros((M.rows, A.cols), order="F")
        _check(C.lib.slq_spmm_csc_csc(_ctx(ctx).handle, M.rows, M.cols, _i(M.row_indices), _d(M.values),
                                      _i(M.col_pointers), A.cols, _i(_i64(A.col_pointers)), _i(_i64(A.row_indices)),
                                      _d(_vec(A.values)), _d(Y)))
        return Y
    A = _f64(A)
    m, n = A.shape
    M = S.matrix
    if M.cols != m:
        raise DimensionMismatch(f"spmm: S is {M.rows}x{M.cols}, A is {m}x{n}")
    Y = np.zeros((M.rows, n), order="F")
    _check(C.lib.slq_spmm_csc_dense(_ctx(ctx).handle, M.rows, m, _i(M.row_indices), _d(M.values),
                                    _i(M.col_pointers), _d(A), n, max(m, 1), _d(Y)))
    return Y


def sketch_vector(S: SparseSignSketch, b, ctx=None) -> np.ndarray:
    """sketch.hpp:304 -> csc_matrix.hpp:71-82 (S b); same order, bit-identical."""
    b = _vec(b)
    if b.size != S.matrix.cols:
        raise DimensionMismatch("matvec(csc): length mismatch")
    return apply(S, b.reshape(-1, 1), ctx)[:, 0].copy()


# ---------------------------------------------------------- factorizations


def householder_qr(Y, ctx=None) -> QrResult:
    """qr.hpp:21-89"""
    Y = _f64(Y)
    d, n = Y.shape
    if d < n:
        raise DimensionMismatch("householder_qr: need rows >= cols")
    Q = np.zeros((d, n), order="F")
    R = np.zeros((n, n), order="F")
    _check(C.lib.slq_householder_qr(_ctx(ctx).handle, _d(Y), d, n, max(d, 1), _d(Q), _d(R)))
    return QrResult(Q, R)


def tri_inverse(R, ctx=None) -> np.ndarray:
    """triangular.hpp:14-33"""
    R = _f64(R)
    n = R.shape[0]
    if R.shape[1] != n:
        raise DimensionMismatch("tri_inverse: matrix not square")
    M = np.zeros((n, n), order="F")
    _check(C.lib.slq_tri_inverse(_ctx(ctx).handle, _d(R), n, _d(M)))
    return M


def tri_upper_matvec(R, x, ctx=None) -> np.ndarray:
    """triangular.hpp:36-47"""
    R = _f64(R)
    x = _vec(x)
    if x.size != R.shape[0]:
        raise DimensionMismatch("tri_upper_matvec")
    y = np.zeros(R.shape[0])
    _check(C.lib.slq_tri_upper_matvec(_ctx(ctx).handle, _d(R), R.shape[0], _d(x), _d(y), 0))
    return y


def tri_upper_rmatvec(R, x, ctx=None) -> np.ndarray:
    """triangular.hpp:50-61"""
    R = _f64(R)
    x = _vec(x)
    if x.size != R.shape[0]:
        raise DimensionMismatch("tri_upper_rmatvec")
    y = np.zeros(R.shape[0])
    _check(C.lib.slq_tri_upper_matvec(_ctx(ctx).handle, _d(R), R.shape[0], _d(x), _d(y), 1))
    return y


def build_preconditioner(Y, ctx=None, Sb=None, want_q=True):
    """preconditioner.hpp:35-44.  With ``Sb`` also returns x0 = M Q^T Sb
    (preconditioner.hpp:48-53) computed from the same factorization.
    want_q=False never forms Q (P.Q is None) -- the solve path's form, and the
    only one for d > 12400 (TSQR)."""
    Y = _f64(Y)
    d, n = Y.shape
    if d < n:
        raise DimensionMismatch("householder_qr: need rows >= cols")
    M = np.zeros((n, n), order="F")
    Q = np.zeros((d, n), order="F") if want_q else None
    bt = np.zeros(1)
    x0 = np.zeros(n) if Sb is not None else None
    _check(C.lib.slq_build_preconditioner(_ctx(ctx).handle, _d(Y), d, n, max(d, 1),
                                          _d(_vec(Sb)) if Sb is not None else None, _d(M), _d(Q), _d(x0), _d(bt)))
    P = Preconditioner(M, Q, float(bt[0]), d)
    return (P, x0) if Sb is not None else P


def initial_guess(P: Preconditioner, Sb, ctx=None) -> np.ndarray:
    """preconditioner.hpp:48-53"""
    Sb = _vec(Sb)
    if P.Q is None or Sb.size != P.Q.shape[0]:
        raise DimensionMismatch("initial_guess: Sb length does not match sketch dimension")
    n = P.M.shape[0]
    x0 = np.zeros(n)
    _check(C.lib.slq_initial_guess(_ctx(ctx).handle, _d(_f64(P.M)), _d(_f64(P.Q)), P.Q.shape[0], n, _d(Sb), _d(x0)))
    return x0


def apply_M(P: Preconditioner, v, ctx=None) -> np.ndarray:
    """preconditioner.hpp:55"""
    return tri_upper_matvec(P.M, v, ctx)


def apply_Mt(P: Preconditioner, v, ctx=None) -> np.ndarray:
    """preconditioner.hpp:56"""
    return tri_upper_rmatvec(P.M, v, ctx)


# ---------------------------------------------------------- device matrix


class DeviceMatrix:
    """A row block of A resident in HBM (device layout: row-major [A | b]).

    ``row_begin`` is the global id of the block's first row (sketch columns
    are keyed by it, distsim.hpp:346-361)."""

    def __init__(self, handle, m, n, row_begin, ctx, owner=None):
        self.handle = handle
        self.m, self.n, self.row_begin = m, n, row_begin
        self.ctx = ctx
        self._owner = owner  # keeps a wrapped torch tensor alive

    @classmethod
    def from_numpy(cls, A, b=None, row_begin=0, ctx=None):
        ctx = _ctx(ctx)
        A = _f64(A)
        m, n = A.shape
        bb = _vec(b) if b is not None else None
        h = C.vp()
        _check(C.lib.slq_dense_upload(ctx.handle, _d(A), m, n, max(m, 1), _d(bb), row_begin, ct.byref(h)))
        return cls(h, m, n, row_begin, ctx, owner=(A, bb))

    @classmethod
    def from_host_ptr(cls, ptr, m, n, lda, b_ptr=None, row_begin=0, ctx=None, owner=None):
        ctx = _ctx(ctx)
        h = C.vp()
        _check(C.lib.slq_dense_upload(ctx.handle, ct.cast(ptr, C.dp), m, n, lda,
                                      ct.cast(b_ptr, C.dp) if b_ptr else None, row_begin, ct.byref(h)))
        return cls(h, m, n, row_begin, ctx, owner=owner)

    @classmethod
    def wrap(cls, dev_ptr, m, n, ld, row_begin=0, ctx=None, owner=None):
        ctx = _ctx(ctx)
        h = C.vp()
        _check(C.lib.slq_dense_wrap(ctx.handle, C.vp(dev_ptr), m, n, ld, row_begin, ct.byref(h)))
        return cls(h, m, n, row_begin, ctx, owner=owner)

    @staticmethod
    def ld_for(n: int) -> int:
        return ((n + 1 + 3) // 4) * 4

    def set_rhs(self, b):
        _check(C.lib.slq_dense_set_rhs(self.handle, _d(_vec(b))))

    def free(self):
        if self.handle:
            C.lib.slq_dense_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def sketch(self, d, zeta, seed, exact=False):
        """apply + sketch_vector fused (sketch.hpp:297/304); multi-rank: summed."""
        Y = np.zeros((d, self.n), order="F")
        Sb = np.zeros(d)
        _check(C.lib.slq_sketch_apply(self.ctx.handle, self.handle, d, zeta, seed & (2**64 - 1), int(exact),
                                      _d(Y), _d(Sb)))
        return Y, Sb


class SparseDeviceMatrix:
    """A row block of a sparse A resident in HBM as CSR (the reference's
    CscMatrix operand, converted on the device)."""

    def __init__(self, handle, m, n, row_begin, ctx, owner=None):
        self.handle = handle
        self.m, self.n, self.row_begin = m, n, row_begin
        self.ctx = ctx
        self._owner = owner

    @classmethod
    def from_csc(cls, A: CscMatrix, b=None, row_begin=0, ctx=None):
        ctx = _ctx(ctx)
        cp, rw, vl = _i64(A.col_pointers), _i64(A.row_indices), _vec(A.values)
        bb = _vec(b) if b is not None else None
        h = C.vp()
        _check(C.lib.slq_sparse_upload_csc(ctx.handle, A.rows, A.cols, _i(cp), _i(rw), _d(vl), _d(bb), row_begin,
                                           ct.byref(h)))
        return cls(h, A.rows, A.cols, row_begin, ctx)

    @classmethod
    def create_csr(cls, m, n, nnz, row_begin=0, with_b=True, ctx=None):
        """Allocate a device CSR to be filled in place; returns (matrix, (row_ptr, col_idx, values, b) pointers)."""
        ctx = _ctx(ctx)
        h = C.vp()
        ptrs = [C.vp() for _ in range(4)]
        _check(C.lib.slq_sparse_create_csr(ctx.handle, m, n, nnz, row_begin, int(with_b), ct.byref(h),
                                           *[ct.byref(p) for p in ptrs]))
        return cls(h, m, n, row_begin, ctx), tuple(p.value for p in ptrs)

    def set_rhs(self, b):
        _check(C.lib.slq_sparse_set_rhs(self.handle, _d(_vec(b))))

    def fill_random(self, nnz_per_row, seed, col_scale=None):
        """Benchmark harness (config C4): nnz_per_row distinct random columns per row."""
        cs = _vec(col_scale) if col_scale is not None else None
        _check(C.lib.slq_sparse_fill_random(self.handle, nnz_per_row, seed & (2**64 - 1), _d(cs)))

    def prepare(self):
        """(Re)build the row-blocked CSC copy the solves stream for A^T u (done
        implicitly by the first solve; needed after rewriting the CSR in place)."""
        _check(C.lib.slq_sparse_prepare(self.ctx.handle, self.handle))

    def free(self):
        if self.handle:
            C.lib.slq_sparse_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def sketch(self, d, zeta, seed):
        Y = np.zeros((d, self.n), order="F")
        Sb = np.zeros(d)
        _check(C.lib.slq_sketch_apply_sparse(self.ctx.handle, self.handle, d, zeta, seed & (2**64 - 1), _d(Y), _d(Sb)))
        return Y, Sb


# ------------------------------------------------------------------- LSQR


def _opts(o: SolveOptions | None, one_sync: bool, n: int):
    o = o or SolveOptions()
    co = C.SolveOpts()
    C.lib.slq_solve_opts_default(ct.byref(co))
    co.eps = o.eps
    co.maxit = int(o.maxit)
    keep = []
    if o.x_star is not None:
        xs = _vec(o.x_star)
        if xs.size != n:
            raise DimensionMismatch("x_star length")
        keep.append(xs)
        co.x_star = _d(xs)
    co.track_true_residual = int(bool(o.track_true_residual))
    co.one_sync = int(one_sync)
    co.backward_tol = o.backward_tol
    co.a_norm_est = o.a_norm_est
    if o.on_bidiag is not None:
        fn = o.on_bidiag
        cb = C.BIDIAG_CB(lambda user, t, un, vn: fn(int(t), float(un), float(vn)))
        keep.append(cb)
        co.on_bidiag = cb
    return co, keep


def _report(r: C.Report, est, err, tru) -> SolveReport:
    return SolveReport(
        iterates_error=list(err[: r.n_err]) if err is not None else [],
        residual_estimate=list(est[: r.n_estimate]),
        residual_true=list(tru[: r.n_true]) if tru is not None else [],
        iterations=int(r.iterations),
        termination=Termination(int(r.termination)),
        sync_count=int(r.sync_count),
        broadcasts=int(r.broadcasts),
        init_reductions=int(r.init_reductions),
        init_broadcasts=int(r.init_broadcasts),
        wall_time=float(r.wall_time),
        backward_error=float(r.backward_error),
    )


def _lsqr(A, P, b, x0, opts, one_sync, ctx):
    ctx = _ctx(ctx)
    if isinstance(A, (CscMatrix, SparseDeviceMatrix)):
        return _lsqr_sparse(A, P, b, x0, opts, one_sync, ctx)
    if isinstance(A, DeviceMatrix):
        dm = A
        m, n = A.m, A.n
        bb = _vec(b) if b is not None else None
    else:
        A = _f64(A)
        m, n = A.shape
        bb = _vec(b)
        if bb.size != m:
            raise DimensionMismatch("rmatvec: length mismatch")
        dm = DeviceMatrix.from_numpy(A, bb, ctx=ctx)
        bb = None
    M = _f64(P.M if isinstance(P, Preconditioner) else P)
    if M.shape != (n, n):
        raise DimensionMismatch("tri_upper_matvec")
    x0 = _vec(x0)
    if x0.size != n:
        raise DimensionMismatch("matvec: x has wrong length")
    co, keep = _opts(opts, one_sync, n)
    maxit = max(int(co.maxit), 0)
    est = np.zeros(maxit + 2)
    err = np.zeros(maxit + 2)
    tru = np.zeros(maxit + 2)
    x = np.zeros(n)
    rep = C.Report()
    _check(C.lib.slq_lsqr(ctx.handle, dm.handle, _d(M), _d(bb), _d(x0), ct.byref(co), _d(x), ct.byref(rep),
                          _d(est), _d(err), _d(tru)))
    del keep
    return x, _report(rep, est, err, tru)


def _lsqr_sparse(A, P, b, x0, opts, one_sync, ctx):
    if isinstance(A, CscMatrix):
        bb = _vec(b)
        if bb.size != A.rows:
            raise DimensionMismatch("rmatvec(csc): length mismatch")
        dm = SparseDeviceMatrix.from_csc(A, bb, ctx=ctx)
        bb = None
    else:
        dm = A
        bb = _vec(b) if b is not None else None
    n = dm.n
    M = _f64(P.M if isinstance(P, Preconditioner) else P)
    if M.shape != (n, n):
        raise DimensionMismatch("tri_upper_matvec")
    x0 = _vec(x0)
    if x0.size != n:
        raise DimensionMismatch("matvec(csc): length mismatch")
    co, keep = _opts(opts, one_sync, n)
    maxit = max(int(co.maxit), 0)
    est, err, tru = np.zeros(maxit + 2), np.zeros(maxit + 2), np.zeros(maxit + 2)
    x = np.zeros(n)
    rep = C.Report()
    _check(C.lib.slq_lsqr_sparse(ctx.handle, dm.handle, _d(M), _d(bb), _d(x0), ct.byref(co), _d(x), ct.byref(rep),
                                 _d(est), _d(err), _d(tru)))
    del keep
    return x, _report(rep, est, err, tru)


def lsqr(A, P, b, x0, opts: SolveOptions | None = None, ctx=None):
    """lsqr.hpp:175-180 / :193-202 -- preconditioned LSQR (standard variant)."""
    return _lsqr(A, P, b, x0, opts, False, ctx)


def lsqr_one_sync(A, P, b, x0, opts: SolveOptions | None = None, ctx=None):
    """lsqr.hpp:185-189 / :203-212 -- one reduction per iteration."""
    return _lsqr(A, P, b, x0, opts, True, ctx)


# --------------------------------------------------------- gradient family


@dataclass
class GradientParams:
    """gradient.hpp:20-24"""

    alpha: float = 1.0
    beta: float = 0.0
    eta_hat: float = 0.0


def hbm_params(eta_hat: float) -> GradientParams:
    """gradient.hpp:27-34: alpha = (1 - eta^2)^2, beta = eta^2 (rate sqrt(beta))."""
    g = C.GradientParams()
    _check(C.lib.slq_hbm_params(float(eta_hat), ct.byref(g)))
    return GradientParams(g.alpha, g.beta, g.eta_hat)


def gd_params(eta_hat: float) -> GradientParams:
    """gradient.hpp:46-48: plain gradient descent, alpha = gd_step_size(eta_hat), beta = 0."""
    g = C.GradientParams()
    _check(C.lib.slq_gd_params(float(eta_hat), ct.byref(g)))
    return GradientParams(g.alpha, g.beta, g.eta_hat)


def gd_step_size(eta_hat: float) -> float:
    """gradient.hpp:37-44"""
    return gd_params(eta_hat).alpha


def gradient_descent_hbm(A, P, b, x0, params: GradientParams, opts: SolveOptions | None = None, ctx=None):
    """gradient.hpp:56-126 -- heavy-ball (beta > 0) / gradient descent (beta = 0)
    on the preconditioned problem; one HBM pass over A per iteration.  Raises
    Divergence when ||M^T A^T r|| grows by 1e6 over its first value."""
    ctx = _ctx(ctx)
    sparse = isinstance(A, (CscMatrix, SparseDeviceMatrix))
    if isinstance(A, CscMatrix):
        bb = _vec(b)
        if bb.size != A.rows:
            raise DimensionMismatch("rmatvec(csc): length mismatch")
        dm, bb = SparseDeviceMatrix.from_csc(A, bb, ctx=ctx), None
    elif isinstance(A, (DeviceMatrix, SparseDeviceMatrix)):
        dm = A
        bb = _vec(b) if b is not None else None
    else:
        A = _f64(A)
        bb = _vec(b)
        if bb.size != A.shape[0]:
            raise DimensionMismatch("rmatvec: length mismatch")
        dm, bb = DeviceMatrix.from_numpy(A, bb, ctx=ctx), None
    n = dm.n
    M = _f64(P.M if isinstance(P, Preconditioner) else P)
    if M.shape != (n, n):
        raise DimensionMismatch("tri_upper_matvec")
    x0 = _vec(x0)
    if x0.size != n:
        raise DimensionMismatch("matvec: x has wrong length")
    co, keep = _opts(opts, False, n)
    maxit = max(int(co.maxit), 0)
    est, err, tru = np.zeros(maxit + 2), np.zeros(maxit + 2), np.zeros(maxit + 2)
    x = np.zeros(n)
    rep = C.Report()
    gp = C.GradientParams(float(params.alpha), float(params.beta), float(params.eta_hat))
    fn = C.lib.slq_gradient_descent_hbm_sparse if sparse else C.lib.slq_gradient_descent_hbm
    _check(fn(ctx.handle, dm.handle, _d(M), _d(bb), _d(x0), ct.byref(gp), ct.byref(co), _d(x), ct.byref(rep),
              _d(est), _d(err), _d(tru)))
    del keep
    return x, _report(rep, est, err, tru)


# ------------------------------------------------------------ distributed


def partition_rows(m: int, p: int) -> RowPartition:
    """distsim.hpp:31-42"""
    out = np.zeros(p + 1 if p >= 1 else 1, np.int64)
    _check(C.lib.slq_partition_rows(m, p, _i(out)))
    return RowPartition(m, [int(v) for v in out])


# ---------------------------------------------------------- whole pipeline


def solve(A, d, zeta, seed, opts: SolveOptions | None = None, b=None, one_sync=True, ctx=None):
    """Sketch -> precondition -> LSQR on the device (the paper's Alg. 1):
    generate_sparse_sign + apply + sketch_vector + build_preconditioner +
    initial_guess + lsqr (sketch.hpp:178,297,304; preconditioner.hpp:35,48;
    lsqr.hpp:175).  ``A`` is a DeviceMatrix (this rank's rows; b stored with
    it) or a host array (then ``b`` is required).  Returns (x, report, phase_times)."""
    ctx = _ctx(ctx)
    sparse = isinstance(A, (CscMatrix, SparseDeviceMatrix))
    if isinstance(A, CscMatrix):
        A = SparseDeviceMatrix.from_csc(A, b, ctx=ctx)
    elif not sparse and not isinstance(A, DeviceMatrix):
        A = DeviceMatrix.from_numpy(A, b, ctx=ctx)
    co, keep = _opts(opts, one_sync, A.n)
    maxit = max(int(co.maxit), 0)
    est = np.zeros(maxit + 2)
    x = np.zeros(A.n)
    rep = C.Report()
    pt = C.PhaseTimes()
    fn = C.lib.slq_solve_sparse if sparse else C.lib.slq_solve
    _check(fn(ctx.handle, A.handle, d, zeta, seed & (2**64 - 1), ct.byref(co), _d(x), ct.byref(rep), ct.byref(pt),
              _d(est)))
    del keep
    return x, _report(rep, est, None, None), pt.as_dict()
