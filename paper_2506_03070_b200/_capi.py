"""ctypes binding of include/slq_b200.h (the C-ABI of libslq_b200.so).

The library is built in-tree (``make -C paper_2506_03070_b200`` or
``__graft_entry__.build()``).  There is no fallback: if the shared object is
missing this module raises on import.
"""
from __future__ import annotations

import ctypes as ct
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libslq_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the sm_100a library first "
        "(python -c 'import __graft_entry__ as g; g.build()' or make -C paper_2506_03070_b200)"
    )

lib = ct.CDLL(LIB_PATH)

i64 = ct.c_int64
u64 = ct.c_uint64
dp = ct.POINTER(ct.c_double)
ip = ct.POINTER(ct.c_int64)
vp = ct.c_void_p


class RejectionStats(ct.Structure):
    _fields_ = [("columns_resampled", i64), ("resample_rounds", i64)]


BIDIAG_CB = ct.CFUNCTYPE(None, vp, i64, ct.c_double, ct.c_double)


class SolveOpts(ct.Structure):
    _fields_ = [
        ("eps", ct.c_double),
        ("maxit", i64),
        ("x_star", dp),
        ("track_true_residual", ct.c_int32),
        ("one_sync", ct.c_int32),
        ("backward_tol", ct.c_double),
        ("a_norm_est", ct.c_double),
        ("on_bidiag", BIDIAG_CB),
        ("on_bidiag_user", vp),
    ]


HostCollective = ct.CFUNCTYPE(ct.c_int, ct.c_void_p, ct.POINTER(ct.c_double), ct.c_int64)


class HostComm(ct.Structure):
    _fields_ = [("allreduce_sum", HostCollective), ("reduce_sum_root", HostCollective),
                ("broadcast_root", HostCollective), ("user", ct.c_void_p)]


class Report(ct.Structure):
    _fields_ = [
        ("iterations", i64),
        ("termination", ct.c_int32),
        ("pad0", ct.c_int32),
        ("sync_count", i64),
        ("broadcasts", i64),
        ("init_reductions", i64),
        ("init_broadcasts", i64),
        ("wall_time", ct.c_double),
        ("n_estimate", i64),
        ("n_err", i64),
        ("n_true", i64),
        ("backward_error", ct.c_double),
    ]


class GradientParams(ct.Structure):
    _fields_ = [("alpha", ct.c_double), ("beta", ct.c_double), ("eta_hat", ct.c_double)]


class PhaseTimes(ct.Structure):
    _fields_ = [
        ("generate", ct.c_double),
        ("apply", ct.c_double),
        ("reduce", ct.c_double),
        ("qr", ct.c_double),
        ("inverse", ct.c_double),
        ("x0", ct.c_double),
        ("lsqr", ct.c_double),
        ("total", ct.c_double),
        ("lsqr_per_iteration", ct.c_double),
        ("nccl_calls", i64),
        ("kernel_launches", i64),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_SIGS = {
    "slq_last_error": (ct.c_char_p, []),
    "slq_version": (ct.c_char_p, []),
    "slq_solve_opts_default": (None, [ct.POINTER(SolveOpts)]),
    "slq_ctx_create": (ct.c_int, [ct.c_int, ct.POINTER(vp)]),
    "slq_ctx_destroy": (ct.c_int, [vp]),
    "slq_ctx_set_stream": (ct.c_int, [vp, vp]),
    "slq_ctx_synchronize": (ct.c_int, [vp]),
    "slq_ctx_kernel_launches": (i64, [vp]),
    "slq_comm_unique_id": (ct.c_int, [ct.c_char_p]),
    "slq_ctx_init_comm": (ct.c_int, [vp, ct.c_char_p, ct.c_int, ct.c_int]),
    "slq_partition_rows": (ct.c_int, [i64, ct.c_int, ip]),
    "slq_generate_sparse_sign": (ct.c_int, [vp, i64, i64, i64, i64, u64, ip, dp, ip, ct.POINTER(RejectionStats)]),
    "slq_rejection_sample_columns": (ct.c_int, [vp, i64, i64, i64, u64, ip, ct.POINTER(RejectionStats)]),
    "slq_dense_upload": (ct.c_int, [vp, dp, i64, i64, i64, dp, i64, ct.POINTER(vp)]),
    "slq_dense_create": (ct.c_int, [vp, i64, i64, i64, ct.POINTER(vp), ct.POINTER(vp), ip]),
    "slq_dense_wrap": (ct.c_int, [vp, vp, i64, i64, i64, i64, ct.POINTER(vp)]),
    "slq_dense_set_rhs": (ct.c_int, [vp, dp]),
    "slq_dense_free": (ct.c_int, [vp]),
    "slq_dense_ld": (i64, [vp]),
    "slq_sketch_apply": (ct.c_int, [vp, vp, i64, i64, u64, ct.c_int, dp, dp]),
    "slq_spmm_csc_dense": (ct.c_int, [vp, i64, i64, ip, dp, ip, dp, i64, i64, dp]),
    "slq_householder_qr": (ct.c_int, [vp, dp, i64, i64, i64, dp, dp]),
    "slq_tri_inverse": (ct.c_int, [vp, dp, i64, dp]),
    "slq_build_preconditioner": (ct.c_int, [vp, dp, i64, i64, i64, dp, dp, dp, dp, dp]),
    "slq_initial_guess": (ct.c_int, [vp, dp, dp, i64, i64, dp, dp]),
    "slq_tri_upper_matvec": (ct.c_int, [vp, dp, i64, dp, dp, ct.c_int]),
    "slq_ctx_set_host_comm": (ct.c_int, [vp, ct.POINTER(HostComm), ct.c_int, ct.c_int]),
    "slq_dense_matvec": (ct.c_int, [vp, vp, dp, dp]),
    "slq_dense_rmatvec": (ct.c_int, [vp, vp, dp, dp, dp]),
    "slq_sparse_matvec": (ct.c_int, [vp, vp, dp, dp]),
    "slq_sparse_rmatvec": (ct.c_int, [vp, vp, dp, dp, dp]),
    "slq_lsqr": (ct.c_int, [vp, vp, dp, dp, dp, ct.POINTER(SolveOpts), dp, ct.POINTER(Report), dp, dp, dp]),
    "slq_solve": (ct.c_int, [vp, vp, i64, i64, u64, ct.POINTER(SolveOpts), dp, ct.POINTER(Report),
                             ct.POINTER(PhaseTimes), dp]),
    "slq_sparse_upload_csc": (ct.c_int, [vp, i64, i64, ip, ip, dp, dp, i64, ct.POINTER(vp)]),
    "slq_sparse_create_csr": (ct.c_int, [vp, i64, i64, i64, i64, ct.c_int, ct.POINTER(vp), ct.POINTER(vp),
                                         ct.POINTER(vp), ct.POINTER(vp), ct.POINTER(vp)]),
    "slq_sparse_set_rhs": (ct.c_int, [vp, dp]),
    "slq_sparse_fill_random": (ct.c_int, [vp, i64, u64, dp]),
    "slq_sparse_free": (ct.c_int, [vp]),
    "slq_sparse_prepare": (ct.c_int, [vp, vp]),
    "slq_debug_check_guards": (ct.c_int, [ct.POINTER(i64)]),
    "slq_debug_guard_selftest": (ct.c_int, [ct.POINTER(ct.c_int)]),
    "slq_spmm_csc_csc": (ct.c_int, [vp, i64, i64, ip, dp, ip, i64, ip, ip, dp, dp]),
    "slq_sketch_apply_sparse": (ct.c_int, [vp, vp, i64, i64, u64, dp, dp]),
    "slq_lsqr_sparse": (ct.c_int, [vp, vp, dp, dp, dp, ct.POINTER(SolveOpts), dp, ct.POINTER(Report), dp, dp, dp]),
    "slq_solve_sparse": (ct.c_int, [vp, vp, i64, i64, u64, ct.POINTER(SolveOpts), dp, ct.POINTER(Report),
                                    ct.POINTER(PhaseTimes), dp]),
    "slq_hbm_params": (ct.c_int, [ct.c_double, ct.POINTER(GradientParams)]),
    "slq_gd_params": (ct.c_int, [ct.c_double, ct.POINTER(GradientParams)]),
    "slq_gradient_descent_hbm": (ct.c_int, [vp, vp, dp, dp, dp, ct.POINTER(GradientParams), ct.POINTER(SolveOpts), dp,
                                            ct.POINTER(Report), dp, dp, dp]),
    "slq_gradient_descent_hbm_sparse": (ct.c_int, [vp, vp, dp, dp, dp, ct.POINTER(GradientParams),
                                                   ct.POINTER(SolveOpts), dp, ct.POINTER(Report), dp, dp, dp]),
    "slq_time_kernels": (ct.c_int, [vp, vp, i64, i64, u64, ct.c_int, dp]),
    "slq_time_sparse_pass": (ct.c_int, [vp, vp, ct.c_int, dp]),
    "slq_solve_host": (ct.c_int, [vp, dp, i64, i64, i64, dp, i64, i64, i64, u64, ct.POINTER(SolveOpts), dp,
                                  ct.POINTER(Report), ct.POINTER(PhaseTimes), dp]),
}

for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = sorted(_SIGS)
