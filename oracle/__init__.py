"""oracle -- CPU checker for the sketch-and-precondition hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference`` arm) import
this package; the product (``paper_2506_03070_b200``) never does.

Two backends with one numpy-facing API:

* ``C``   -- ``_build/liboracle.so``: the plain-C restatement in
  ``sketchlsq_oracle.c`` (each function cites the reference file:line).
* ``REF`` -- ``_ref/libsketchlsq_ref.so``: the unmodified reference headers
  (``/root/reference/proj/include/sketchlsq``) compiled in place by
  ``oracle/Makefile`` behind the thin ``ref_shim.cpp``.

Matrices are numpy float64 arrays in the reference's column-major layout
(``dense_matrix.hpp:14-35``); we accept any 2-D array and pass ``np.asfortranarray``.
"""
from __future__ import annotations

import ctypes as ct
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
C_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
REF_LIB_PATH = os.path.join(_HERE, "_ref", "libsketchlsq_ref.so")

_i64 = ct.c_int64
_u64 = ct.c_uint64
_dp = ct.POINTER(ct.c_double)
_ip = ct.POINTER(ct.c_int64)

TERMINATION = {0: "tolerance", 1: "maxiter", 2: "breakdown"}

STATUS = {
    0: None,
    1: "InvalidSparsity",
    2: "InvalidDims",
    3: "DimensionMismatch",
    4: "RankDeficient",
    5: "SingularTriangular",
    11: "InvalidDistortion",
    12: "Divergence",
    13: "NegativeArgument",
    14: "InvalidResidual",
    15: "UnsupportedFormat",
    8: "OOM",
    99: "Error",
}


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str = ""):
        self.code = code
        self.kind = STATUS.get(code, "Error")
        super().__init__(f"{self.kind}: {what}")


def build(quiet: bool = True) -> None:
    """Compile the restatement (and the reference shim when headers exist)."""
    import subprocess

    out = subprocess.run(["make", "-C", _HERE], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


def _d(a):
    return a.ctypes.data_as(_dp) if a is not None else None


def _i(a):
    return a.ctypes.data_as(_ip) if a is not None else None


def _f(a):
    return np.asfortranarray(a, dtype=np.float64)


def _col(a):
    return np.ascontiguousarray(a, dtype=np.float64).reshape(-1)


@dataclass
class Report:
    iterations: int
    termination: str
    residual_estimate: np.ndarray
    iterates_error: np.ndarray = field(default_factory=lambda: np.zeros(0))
    residual_true: np.ndarray = field(default_factory=lambda: np.zeros(0))
    sync_count: int = 0
    broadcasts: int = 0
    init_reductions: int = 0
    init_broadcasts: int = 0
    wall_time: float = 0.0


class _RefReport(ct.Structure):
    _fields_ = [
        ("iterations", ct.c_int64),
        ("termination", ct.c_int32),
        ("pad", ct.c_int32),
        ("sync_count", ct.c_int64),
        ("broadcasts", ct.c_int64),
        ("init_reductions", ct.c_int64),
        ("init_broadcasts", ct.c_int64),
        ("wall_time", ct.c_double),
        ("n_estimate", ct.c_int64),
        ("n_true", ct.c_int64),
        ("n_err", ct.c_int64),
    ]


class _OrcReport(ct.Structure):
    _fields_ = [
        ("iterations", ct.c_long),
        ("termination", ct.c_int),
        ("n_estimate", ct.c_long),
        ("n_true", ct.c_long),
        ("n_err", ct.c_long),
    ]


class _Base:
    lib: ct.CDLL

    def _check(self, code, what=""):
        if code != 0:
            raise OracleError(code, what)


class COracle(_Base):
    """The plain-C restatement (sketchlsq_oracle.c)."""

    def __init__(self, path: str = C_LIB_PATH):
        if not os.path.exists(path):
            build()
        self.lib = ct.CDLL(path)
        L = self.lib
        L.orc_mix64.restype = _u64
        L.orc_mix64.argtypes = [_u64]
        L.orc_rng_stream.restype = _u64
        L.orc_rng_stream.argtypes = [_u64, _u64]
        L.orc_rng_seed.restype = _u64
        L.orc_rng_seed.argtypes = [_u64]
        L.orc_next_u64.restype = _u64
        L.orc_next_u64.argtypes = [ct.POINTER(_u64)]
        L.orc_uniform_below.restype = _u64
        L.orc_uniform_below.argtypes = [ct.POINTER(_u64), _u64]
        L.orc_sparse_sign_block.argtypes = [_i64, _i64, _u64, _i64, _i64, _ip, _dp, _ip, _ip, _ip]
        L.orc_rejection_sample_columns.argtypes = [_i64, _i64, _i64, _u64, _ip, _ip, _ip]
        L.orc_spmm_csc_dense.argtypes = [_i64, _i64, _ip, _dp, _ip, _dp, _i64, _dp]
        L.orc_csc_matvec.argtypes = [_i64, _i64, _ip, _dp, _ip, _dp, _dp]
        L.orc_csc_rmatvec.argtypes = [_i64, _i64, _ip, _dp, _ip, _dp, _dp]
        L.orc_lsqr_csc.argtypes = [_i64, _i64, _ip, _dp, _ip, _dp, _dp, _dp, ct.c_double, ct.c_long, ct.c_int,
                                   _dp, ct.c_int, _dp, ct.POINTER(_OrcReport), _dp, _dp, _dp]
        L.orc_spmm_csc_csc.argtypes = [_i64, _ip, _dp, _ip, _i64, _ip, _dp, _ip, _dp]
        L.orc_matvec.argtypes = [_dp, _i64, _i64, _dp, _dp]
        L.orc_rmatvec.argtypes = [_dp, _i64, _i64, _dp, _dp]
        L.orc_tri_upper_matvec.argtypes = [_dp, _i64, _dp, _dp]
        L.orc_tri_upper_rmatvec.argtypes = [_dp, _i64, _dp, _dp]
        L.orc_householder_qr.argtypes = [_dp, _i64, _i64, _dp, _dp, _ip]
        L.orc_tri_inverse.argtypes = [_dp, _i64, _dp, _ip]
        L.orc_initial_guess.argtypes = [_dp, _dp, _i64, _i64, _dp, _dp]
        L.orc_lsqr.argtypes = [_dp, _i64, _i64, _dp, _dp, _dp, ct.c_double, ct.c_long, ct.c_int,
                               _dp, ct.c_int, _dp, ct.POINTER(_OrcReport), _dp, _dp, _dp]
        L.orc_partition_rows.argtypes = [_i64, ct.c_int, _ip]
        L.orc_hbm_params.argtypes = [ct.c_double, _dp, _dp]
        L.orc_gd_params.argtypes = [ct.c_double, _dp, _dp]
        L.orc_gd_hbm.argtypes = [_dp, _i64, _i64, _dp, _dp, _dp, ct.c_double, ct.c_double, ct.c_double, ct.c_long,
                                 _dp, ct.c_int, _dp, ct.POINTER(_OrcReport), _dp, _dp, _dp]
        L.orc_gd_hbm_csc.argtypes = [_i64, _i64, _ip, _dp, _ip, _dp, _dp, _dp, ct.c_double, ct.c_double,
                                     ct.c_double, ct.c_long, _dp, ct.c_int, _dp, ct.POINTER(_OrcReport), _dp, _dp,
                                     _dp]
        L.orc_gen_dense.argtypes = [_i64, _i64, ct.c_double, _u64, _dp]
        L.orc_gen_rhs.argtypes = [_dp, _i64, _i64, ct.c_double, _u64, _dp, _dp]

    # rng.hpp
    def rng_draws(self, seed: int, stream: int | None, k: int) -> np.ndarray:
        st = _u64(self.lib.orc_rng_seed(seed) if stream is None else self.lib.orc_rng_stream(seed, stream))
        return np.array([self.lib.orc_next_u64(ct.byref(st)) for _ in range(k)], dtype=np.uint64)

    def uniform_below(self, seed: int, stream: int, bound: int, k: int) -> np.ndarray:
        st = _u64(self.lib.orc_rng_stream(seed, stream))
        return np.array([self.lib.orc_uniform_below(ct.byref(st), bound) for _ in range(k)], dtype=np.uint64)

    # sketch.hpp
    def generate_sparse_sign(self, d, m, zeta, seed, col_begin=0):
        rows = np.zeros(m * zeta, np.int64)
        vals = np.zeros(m * zeta, np.float64)
        colptr = np.zeros(m + 1, np.int64)
        cr = np.zeros(1, np.int64)
        rr = np.zeros(1, np.int64)
        self._check(self.lib.orc_sparse_sign_block(d, zeta, seed, col_begin, col_begin + m, _i(rows),
                                                   _d(vals), _i(colptr), _i(cr), _i(rr)))
        return rows, vals, colptr, (int(cr[0]), int(rr[0]))

    def rejection_sample_columns(self, d, m, zeta, seed):
        C = np.zeros(m * zeta, np.int64)
        cr = np.zeros(1, np.int64)
        rr = np.zeros(1, np.int64)
        self._check(self.lib.orc_rejection_sample_columns(d, m, zeta, seed, _i(C), _i(cr), _i(rr)))
        return C, (int(cr[0]), int(rr[0]))

    def spmm(self, d, rows, vals, colptr, A):
        A = _f(A)
        m, n = A.shape
        Y = np.zeros((d, n), order="F")
        self._check(self.lib.orc_spmm_csc_dense(d, m, _i(rows), _d(vals), _i(colptr), _d(A), n, _d(Y)))
        return Y

    def csc_matvec(self, d, rows, vals, colptr, x):
        x = _col(x)
        y = np.zeros(d)
        self._check(self.lib.orc_csc_matvec(d, x.size, _i(rows), _d(vals), _i(colptr), _d(x), _d(y)))
        return y

    def spmm_csc(self, d, srows, svals, scolptr, m, n, arows, avals, acolptr):
        """Y = S A for CSC S (d x m) and CSC A (m x n): csc_matrix.hpp:123-136"""
        Y = np.zeros((d, n), order="F")
        self._check(self.lib.orc_spmm_csc_csc(d, _i(srows), _d(svals), _i(scolptr), n, _i(arows), _d(avals),
                                              _i(acolptr), _d(Y)))
        return Y

    def sketch_apply_csc(self, d, zeta, seed, m, n, arows, avals, acolptr, b=None):
        rows, vals, colptr, _ = self.generate_sparse_sign(d, m, zeta, seed)
        Y = self.spmm_csc(d, rows, vals, colptr, m, n, arows, avals, acolptr)
        Sb = self.csc_matvec(d, rows, vals, colptr, b) if b is not None else None
        return Y, Sb

    def csc_matvec_A(self, m, n, arows, avals, acolptr, x):
        """y = A x for CSC A (m x n): csc_matrix.hpp:71-82"""
        y = np.zeros(m)
        self._check(self.lib.orc_csc_matvec(m, n, _i(arows), _d(avals), _i(acolptr), _d(_col(x)), _d(y)))
        return y

    def csc_rmatvec_A(self, m, n, arows, avals, acolptr, y):
        """x = A^T y for CSC A: csc_matrix.hpp:85-96"""
        x = np.zeros(n)
        self._check(self.lib.orc_csc_rmatvec(m, n, _i(arows), _d(avals), _i(acolptr), _d(_col(y)), _d(x)))
        return x

    def lsqr_csc(self, m, n, arows, avals, acolptr, M, b, x0, eps=1e-10, maxit=100, one_sync=False, x_star=None,
                 track_true=False):
        M = _f(M)
        x = np.zeros(n)
        rep = _OrcReport()
        est = np.zeros(max(maxit, 1) + 1)
        err = np.zeros(max(maxit, 1) + 2)
        tru = np.zeros(max(maxit, 1) + 2)
        xs = _col(x_star) if x_star is not None else None
        self._check(self.lib.orc_lsqr_csc(m, n, _i(arows), _d(avals), _i(acolptr), _d(M), _d(_col(b)),
                                          _d(_col(x0)), eps, maxit, int(one_sync), _d(xs), int(track_true),
                                          _d(x), ct.byref(rep), _d(est), _d(err), _d(tru)))
        return x, Report(rep.iterations, TERMINATION[rep.termination], est[: rep.n_estimate].copy(),
                         err[: rep.n_err].copy(), tru[: rep.n_true].copy())

    def sketch_apply(self, d, zeta, seed, A, b=None):
        A = _f(A)
        rows, vals, colptr, _ = self.generate_sparse_sign(d, A.shape[0], zeta, seed)
        Y = self.spmm(d, rows, vals, colptr, A)
        Sb = self.csc_matvec(d, rows, vals, colptr, b) if b is not None else None
        return Y, Sb

    # dense_matrix.hpp / triangular.hpp
    def matvec(self, A, x):
        A = _f(A)
        y = np.zeros(A.shape[0])
        self.lib.orc_matvec(_d(A), A.shape[0], A.shape[1], _d(_col(x)), _d(y))
        return y

    def rmatvec(self, A, x):
        A = _f(A)
        y = np.zeros(A.shape[1])
        self.lib.orc_rmatvec(_d(A), A.shape[0], A.shape[1], _d(_col(x)), _d(y))
        return y

    def apply_M(self, M, v):
        M = _f(M)
        y = np.zeros(M.shape[0])
        self.lib.orc_tri_upper_matvec(_d(M), M.shape[0], _d(_col(v)), _d(y))
        return y

    def apply_Mt(self, M, v):
        M = _f(M)
        y = np.zeros(M.shape[0])
        self.lib.orc_tri_upper_rmatvec(_d(M), M.shape[0], _d(_col(v)), _d(y))
        return y

    # qr.hpp / triangular.hpp / preconditioner.hpp
    def householder_qr(self, Y, want_q=True):
        Y = _f(Y)
        d, n = Y.shape
        Q = np.zeros((d, n), order="F") if want_q else None
        R = np.zeros((n, n), order="F")
        bad = np.zeros(1, np.int64)
        self._check(self.lib.orc_householder_qr(_d(Y), d, n, _d(Q), _d(R), _i(bad)), f"column {bad[0]}")
        return Q, R

    def tri_inverse(self, R):
        R = _f(R)
        n = R.shape[0]
        M = np.zeros((n, n), order="F")
        bad = np.zeros(1, np.int64)
        self._check(self.lib.orc_tri_inverse(_d(R), n, _d(M), _i(bad)), f"diag {bad[0]}")
        return M

    def build_preconditioner(self, Y):
        Q, R = self.householder_qr(Y)
        return self.tri_inverse(R), Q

    def initial_guess(self, M, Q, Sb):
        M, Q = _f(M), _f(Q)
        x0 = np.zeros(M.shape[0])
        self._check(self.lib.orc_initial_guess(_d(M), _d(Q), Q.shape[0], Q.shape[1], _d(_col(Sb)), _d(x0)))
        return x0

    # lsqr.hpp
    def lsqr(self, A, M, b, x0, eps=1e-10, maxit=100, one_sync=False, x_star=None, track_true=False):
        A, M = _f(A), _f(M)
        m, n = A.shape
        x = np.zeros(n)
        rep = _OrcReport()
        est = np.zeros(max(maxit, 1) + 1)
        err = np.zeros(max(maxit, 1) + 2)
        tru = np.zeros(max(maxit, 1) + 2)
        xs = _col(x_star) if x_star is not None else None
        self._check(self.lib.orc_lsqr(_d(A), m, n, _d(M), _d(_col(b)), _d(_col(x0)), eps, maxit,
                                      int(one_sync), _d(xs), int(track_true), _d(x), ct.byref(rep),
                                      _d(est), _d(err), _d(tru)))
        return x, Report(rep.iterations, TERMINATION[rep.termination], est[: rep.n_estimate].copy(),
                         err[: rep.n_err].copy(), tru[: rep.n_true].copy())

    # gradient.hpp
    def gradient_params(self, eta, hbm=True):
        a, b = np.zeros(1), np.zeros(1)
        self._check((self.lib.orc_hbm_params if hbm else self.lib.orc_gd_params)(eta, _d(a), _d(b)))
        return float(a[0]), float(b[0])

    def gd_hbm(self, A, M, b, x0, alpha, beta, eps=1e-10, maxit=100, x_star=None, track_true=False):
        A, M = _f(A), _f(M)
        m, n = A.shape
        x = np.zeros(n)
        rep = _OrcReport()
        est, err, tru = np.zeros(maxit + 1), np.zeros(maxit + 2), np.zeros(maxit + 2)
        xs = _col(x_star) if x_star is not None else None
        self._check(self.lib.orc_gd_hbm(_d(A), m, n, _d(M), _d(_col(b)), _d(_col(x0)), alpha, beta, eps, maxit,
                                        _d(xs), int(track_true), _d(x), ct.byref(rep), _d(est), _d(err), _d(tru)))
        return x, Report(rep.iterations, TERMINATION[rep.termination], est[: rep.n_estimate].copy(),
                         err[: rep.n_err].copy(), tru[: rep.n_true].copy())

    def gd_hbm_csc(self, m, n, arows, avals, acolptr, M, b, x0, alpha, beta, eps=1e-10, maxit=100, x_star=None,
                   track_true=False):
        M = _f(M)
        x = np.zeros(n)
        rep = _OrcReport()
        est, err, tru = np.zeros(maxit + 1), np.zeros(maxit + 2), np.zeros(maxit + 2)
        xs = _col(x_star) if x_star is not None else None
        self._check(self.lib.orc_gd_hbm_csc(m, n, _i(arows), _d(avals), _i(acolptr), _d(M), _d(_col(b)),
                                            _d(_col(x0)), alpha, beta, eps, maxit, _d(xs), int(track_true), _d(x),
                                            ct.byref(rep), _d(est), _d(err), _d(tru)))
        return x, Report(rep.iterations, TERMINATION[rep.termination], est[: rep.n_estimate].copy(),
                         err[: rep.n_err].copy(), tru[: rep.n_true].copy())

    # distsim.hpp
    def partition_rows(self, m, p):
        out = np.zeros(p + 1, np.int64)
        self._check(self.lib.orc_partition_rows(m, p, _i(out)))
        return out

    # problems.hpp (harness)
    def gen_dense(self, m, n, cond, seed):
        A = np.zeros((m, n), order="F")
        self._check(self.lib.orc_gen_dense(m, n, cond, seed, _d(A)))
        return A

    def gen_rhs(self, A, rho, seed):
        A = _f(A)
        m, n = A.shape
        b = np.zeros(m)
        xs = np.zeros(n)
        self._check(self.lib.orc_gen_rhs(_d(A), m, n, rho, seed, _d(b), _d(xs)))
        return b, xs


class RefOracle(_Base):
    """The reference headers themselves, compiled by oracle/Makefile."""

    def __init__(self, path: str = REF_LIB_PATH):
        if not os.path.exists(path):
            build()
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = ct.CDLL(path)
        L = self.lib
        L.ref_last_error.restype = ct.c_char_p
        L.ref_rng_draws.argtypes = [_u64, _i64, _i64, ct.POINTER(_u64)]
        L.ref_uniform_below.argtypes = [_u64, _u64, _u64, _i64, ct.POINTER(_u64)]
        L.ref_generate_sparse_sign.argtypes = [_i64, _i64, _i64, _i64, _u64, _ip, _dp, _ip, _ip]
        L.ref_rejection_sample_columns.argtypes = [_i64, _i64, _i64, _u64, _ip, _ip]
        L.ref_sketch_apply.argtypes = [_i64, _i64, _i64, _u64, _dp, _i64, _dp, _dp, _dp]
        L.ref_sketch_apply_csc.argtypes = [_i64, _i64, _i64, _u64, _i64, _ip, _dp, _ip, _dp]
        L.ref_householder_qr.argtypes = [_dp, _i64, _i64, _dp, _dp]
        L.ref_tri_inverse.argtypes = [_dp, _i64, _dp]
        L.ref_build_preconditioner.argtypes = [_dp, _i64, _i64, _dp, _dp, _dp, _dp, _dp]
        L.ref_lsqr.argtypes = [_dp, _i64, _i64, _dp, _dp, _dp, ct.c_double, _i64, ct.c_int, _dp,
                               ct.c_int, ct.c_int, _dp, ct.POINTER(_RefReport), _dp, _dp, _dp]
        L.ref_partition_rows.argtypes = [_i64, ct.c_int, _ip]
        L.ref_embedding.argtypes = [_i64, _i64, _i64, ct.c_double, ct.c_double, _dp]
        L.ref_distortion.argtypes = [_i64, _i64, _u64, _dp, _i64, _i64, _dp, _dp]
        L.ref_metric_scalars.argtypes = [ct.c_double] * 5 + [_dp]
        L.ref_mm_write_csc.argtypes = [ct.c_char_p, _i64, _i64, _ip, _dp, _ip]
        L.ref_mm_write_dense.argtypes = [ct.c_char_p, _dp, _i64, _i64]
        L.ref_mm_read_csc.argtypes = [ct.c_char_p, _ip, _ip, _dp, _ip]
        L.ref_mm_read_dense.argtypes = [ct.c_char_p, _ip, _dp]
        L.ref_gradient_params.argtypes = [ct.c_double, ct.c_int, _dp]
        L.ref_gradient_descent_hbm.argtypes = [ct.c_int, _dp, _i64, _i64, _ip, _dp, _ip, _dp, _dp, _dp, ct.c_double,
                                               ct.c_double, ct.c_double, _i64, _dp, ct.c_int, ct.c_int, _dp,
                                               ct.POINTER(_RefReport), _dp, _dp, _dp]
        L.ref_lsqr_csc.argtypes = [_i64, _i64, _ip, _dp, _ip, _dp, _dp, _dp, ct.c_double, _i64, ct.c_int, _dp,
                                   ct.c_int, ct.c_int, _dp, ct.POINTER(_RefReport), _dp, _dp, _dp]
        L.ref_dist_generate_sparse_sign.argtypes = [_i64, _i64, _i64, _u64, ct.c_int, _ip, _dp, _ip]
        L.ref_dist_sketch_apply.argtypes = [_i64, _i64, _i64, _u64, _dp, _i64, _dp, ct.c_int, _dp, _dp]
        L.ref_gen_dense.argtypes = [_i64, _i64, ct.c_double, _u64, _dp]
        L.ref_gen_rhs.argtypes = [_dp, _i64, _i64, ct.c_double, _u64, _dp, _dp]
        L.ref_solve_timed.argtypes = [_dp, _i64, _i64, _dp, _i64, _i64, _u64, ct.c_double, _i64,
                                      ct.c_int, _dp, ct.POINTER(_RefReport), _dp]

    def _check(self, code, what=""):
        if code != 0:
            raise OracleError(code, self.lib.ref_last_error().decode())

    def rng_draws(self, seed, stream, k):
        out = np.zeros(k, np.uint64)
        self.lib.ref_rng_draws(seed, -1 if stream is None else stream, k,
                               out.ctypes.data_as(ct.POINTER(_u64)))
        return out

    def uniform_below(self, seed, stream, bound, k):
        out = np.zeros(k, np.uint64)
        self.lib.ref_uniform_below(seed, stream, bound, k, out.ctypes.data_as(ct.POINTER(_u64)))
        return out

    def generate_sparse_sign(self, d, m, zeta, seed, col_begin=0):
        rows = np.zeros(m * zeta, np.int64)
        vals = np.zeros(m * zeta, np.float64)
        colptr = np.zeros(m + 1, np.int64)
        st = np.zeros(2, np.int64)
        self._check(self.lib.ref_generate_sparse_sign(d, col_begin, m, zeta, seed, _i(rows), _d(vals),
                                                      _i(colptr), _i(st)))
        return rows, vals, colptr, (int(st[0]), int(st[1]))

    def rejection_sample_columns(self, d, m, zeta, seed):
        C = np.zeros(m * zeta, np.int64)
        st = np.zeros(2, np.int64)
        self._check(self.lib.ref_rejection_sample_columns(d, m, zeta, seed, _i(C), _i(st)))
        return C, (int(st[0]), int(st[1]))

    def sketch_apply(self, d, zeta, seed, A, b=None):
        A = _f(A)
        m, n = A.shape
        Y = np.zeros((d, n), order="F")
        Sb = np.zeros(d) if b is not None else None
        self._check(self.lib.ref_sketch_apply(d, m, zeta, seed, _d(A), n,
                                              _d(_col(b)) if b is not None else None, _d(Y), _d(Sb)))
        return Y, Sb

    def householder_qr(self, Y, want_q=True):
        Y = _f(Y)
        d, n = Y.shape
        Q = np.zeros((d, n), order="F") if want_q else None
        R = np.zeros((n, n), order="F")
        self._check(self.lib.ref_householder_qr(_d(Y), d, n, _d(Q), _d(R)))
        return Q, R

    def tri_inverse(self, R):
        R = _f(R)
        n = R.shape[0]
        M = np.zeros((n, n), order="F")
        self._check(self.lib.ref_tri_inverse(_d(R), n, _d(M)))
        return M

    def build_preconditioner(self, Y, Sb=None):
        Y = _f(Y)
        d, n = Y.shape
        M = np.zeros((n, n), order="F")
        Q = np.zeros((d, n), order="F")
        x0 = np.zeros(n) if Sb is not None else None
        bt = np.zeros(1)
        self._check(self.lib.ref_build_preconditioner(_d(Y), d, n, _d(_col(Sb)) if Sb is not None else None,
                                                      _d(M), _d(Q), _d(x0), _d(bt)))
        return M, Q, x0, float(bt[0])

    def lsqr(self, A, M, b, x0, eps=1e-10, maxit=100, one_sync=False, x_star=None, track_true=False,
             workers=0):
        A, M = _f(A), _f(M)
        m, n = A.shape
        x = np.zeros(n)
        rep = _RefReport()
        est = np.zeros(max(maxit, 1) + 1)
        err = np.zeros(max(maxit, 1) + 2)
        tru = np.zeros(max(maxit, 1) + 2)
        xs = _col(x_star) if x_star is not None else None
        self._check(self.lib.ref_lsqr(_d(A), m, n, _d(M), _d(_col(b)), _d(_col(x0)), eps, maxit,
                                      int(one_sync), _d(xs), int(track_true), workers, _d(x),
                                      ct.byref(rep), _d(est), _d(err), _d(tru)))
        return x, Report(rep.iterations, TERMINATION[rep.termination], est[: rep.n_estimate].copy(),
                         err[: rep.n_err].copy(), tru[: rep.n_true].copy(), rep.sync_count,
                         rep.broadcasts, rep.init_reductions, rep.init_broadcasts, rep.wall_time)

    def partition_rows(self, m, p):
        out = np.zeros(p + 1, np.int64)
        self._check(self.lib.ref_partition_rows(m, p, _i(out)))
        return out

    def gradient_params(self, eta, hbm=True):
        out = np.zeros(2)
        self._check(self.lib.ref_gradient_params(eta, int(hbm), _d(out)))
        return float(out[0]), float(out[1])

    def embedding(self, m, n, d, eps, x):
        """embedding.hpp: [rate, kappa, iterations_for, lambert_w(x), balance_real, plan d, iters, kappa]"""
        out = np.zeros(8)
        self._check(self.lib.ref_embedding(m, n, d, eps, x, _d(out)))
        return out

    def distortion(self, d, zeta, seed, U, b=None):
        U = _f(U)
        out = np.zeros(3)
        self._check(self.lib.ref_distortion(d, zeta, seed, _d(U), U.shape[0], U.shape[1],
                                            _d(_col(b)) if b is not None else None, _d(out)))
        return tuple(float(v) for v in out)

    def metric_scalars(self, x, ratio, eta, res_hat, res_star):
        out = np.zeros(3)
        self._check(self.lib.ref_metric_scalars(x, ratio, eta, res_hat, res_star, _d(out)))
        return tuple(float(v) for v in out)

    def mm_write_csc(self, path, m, n, rows, vals, colptr):
        self._check(self.lib.ref_mm_write_csc(path.encode(), m, n, _i(rows), _d(vals), _i(colptr)))

    def mm_write_dense(self, path, A):
        A = _f(A)
        self._check(self.lib.ref_mm_write_dense(path.encode(), _d(A), A.shape[0], A.shape[1]))

    def mm_read_csc(self, path):
        dims = np.zeros(3, np.int64)
        self._check(self.lib.ref_mm_read_csc(path.encode(), _i(dims), None, None, None))
        rows, vals, cp = np.zeros(dims[2], np.int64), np.zeros(dims[2]), np.zeros(dims[1] + 1, np.int64)
        self._check(self.lib.ref_mm_read_csc(path.encode(), _i(dims), _i(rows), _d(vals), _i(cp)))
        return int(dims[0]), int(dims[1]), rows, vals, cp

    def mm_read_dense(self, path):
        dims = np.zeros(2, np.int64)
        self._check(self.lib.ref_mm_read_dense(path.encode(), _i(dims), None))
        A = np.zeros((dims[0], dims[1]), order="F")
        self._check(self.lib.ref_mm_read_dense(path.encode(), _i(dims), _d(A)))
        return A

    def gd_hbm(self, A, M, b, x0, alpha, beta, eps=1e-10, maxit=100, x_star=None, track_true=False, workers=0,
               csc=None):
        """gradient.hpp:56-126; csc = (m, n, rows, vals, colptr) selects the CscMatrix overload."""
        M = _f(M)
        if csc is not None:
            m, n, rows, vals, colptr = csc
            Ad = None
        else:
            Ad = _f(A)
            (m, n), rows, vals, colptr = Ad.shape, None, None, None
        x = np.zeros(n)
        rep = _RefReport()
        est, err, tru = np.zeros(maxit + 1), np.zeros(maxit + 2), np.zeros(maxit + 2)
        xs = _col(x_star) if x_star is not None else None
        self._check(self.lib.ref_gradient_descent_hbm(int(csc is not None), _d(Ad), m, n, _i(rows), _d(vals),
                                                      _i(colptr), _d(M), _d(_col(b)), _d(_col(x0)), alpha, beta,
                                                      eps, maxit, _d(xs), int(track_true), workers, _d(x),
                                                      ct.byref(rep), _d(est), _d(err), _d(tru)))
        return x, Report(rep.iterations, TERMINATION[rep.termination], est[: rep.n_estimate].copy(),
                         err[: rep.n_err].copy(), tru[: rep.n_true].copy(), rep.sync_count,
                         rep.broadcasts, rep.init_reductions, rep.init_broadcasts, rep.wall_time)

    def sketch_apply_csc(self, d, zeta, seed, m, n, arows, avals, acolptr):
        Y = np.zeros((d, n), order="F")
        self._check(self.lib.ref_sketch_apply_csc(d, m, zeta, seed, n, _i(arows), _d(avals), _i(acolptr), _d(Y)))
        return Y

    def lsqr_csc(self, m, n, arows, avals, acolptr, M, b, x0, eps=1e-10, maxit=100, one_sync=False, x_star=None,
                 track_true=False, workers=0):
        M = _f(M)
        x = np.zeros(n)
        rep = _RefReport()
        est = np.zeros(max(maxit, 1) + 1)
        err = np.zeros(max(maxit, 1) + 2)
        tru = np.zeros(max(maxit, 1) + 2)
        xs = _col(x_star) if x_star is not None else None
        self._check(self.lib.ref_lsqr_csc(m, n, _i(arows), _d(avals), _i(acolptr), _d(M), _d(_col(b)),
                                          _d(_col(x0)), eps, maxit, int(one_sync), _d(xs), int(track_true), workers,
                                          _d(x), ct.byref(rep), _d(est), _d(err), _d(tru)))
        return x, Report(rep.iterations, TERMINATION[rep.termination], est[: rep.n_estimate].copy(),
                         err[: rep.n_err].copy(), tru[: rep.n_true].copy(), rep.sync_count,
                         rep.broadcasts, rep.init_reductions, rep.init_broadcasts, rep.wall_time)

    def dist_generate_sparse_sign(self, d, m, zeta, seed, p):
        rows = np.zeros(m * zeta, np.int64)
        vals = np.zeros(m * zeta)
        colptr = np.zeros(m + 1, np.int64)
        self._check(self.lib.ref_dist_generate_sparse_sign(d, m, zeta, seed, p, _i(rows), _d(vals), _i(colptr)))
        return rows, vals, colptr

    def dist_sketch_apply(self, d, zeta, seed, A, b, p):
        A = _f(A)
        m, n = A.shape
        Y = np.zeros((d, n), order="F")
        Sb = np.zeros(d)
        self._check(self.lib.ref_dist_sketch_apply(d, m, zeta, seed, _d(A), n, _d(_col(b)), p, _d(Y), _d(Sb)))
        return Y, Sb

    def gen_dense(self, m, n, cond, seed):
        A = np.zeros((m, n), order="F")
        self._check(self.lib.ref_gen_dense(m, n, cond, seed, _d(A)))
        return A

    def gen_rhs(self, A, rho, seed):
        A = _f(A)
        m, n = A.shape
        b = np.zeros(m)
        xs = np.zeros(n)
        self._check(self.lib.ref_gen_rhs(_d(A), m, n, rho, seed, _d(b), _d(xs)))
        return b, xs

    def solve_timed(self, A, b, d, zeta, seed, eps, maxit, workers):
        """Reference pipeline timed phase by phase (see ref_shim.cpp:ref_solve_timed)."""
        A = _f(A)
        m, n = A.shape
        x = np.zeros(n)
        rep = _RefReport()
        times = np.zeros(6)
        self._check(self.lib.ref_solve_timed(_d(A), m, n, _d(_col(b)), d, zeta, seed, eps, maxit, workers,
                                             _d(x), ct.byref(rep), _d(times)))
        names = ["generate", "apply", "precond", "x0", "lsqr", "distribute"]
        return x, Report(rep.iterations, TERMINATION[rep.termination], np.zeros(0)), dict(zip(names, times))


_c = None
_ref = None


def C() -> COracle:
    global _c
    if _c is None:
        _c = COracle()
    return _c


def REF() -> RefOracle:
    global _ref
    if _ref is None:
        _ref = RefOracle()
    return _ref


def ref_available() -> bool:
    return os.path.exists(REF_LIB_PATH)
