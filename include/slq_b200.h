/*
 * slq_b200.h -- C-ABI of the B200-native sketch-and-precondition LSQ solver.
 *
 * This is the drop-in boundary for the reference's hot path (the header-only
 * C++ library `sketchlsq`, /root/reference/proj/include/sketchlsq/).  The
 * reference has no FFI of its own; each entry point below states which
 * reference function it replaces (file:line).  Plain pointers and sizes only:
 * host buffers are caller-owned, device buffers are context-owned.  Every call
 * returns an slq_status; the message of the last failure on the calling
 * thread is available from slq_last_error().  Status codes map one-to-one to
 * the reference exception types (errors.hpp:9-76).
 *
 * Layout conventions (reference: dense_matrix.hpp:14-35, csc_matrix.hpp:19-60):
 *   dense host matrices are column-major with leading dimension lda >= rows;
 *   CSC uses int64 row indices / col pointers and fp64 values.
 * Device-resident dense matrices (slq_dense) are row-major [A | b] with a
 * padded leading dimension.
 */
#ifndef SLQ_B200_H
#define SLQ_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SLQ_OK = 0,
    SLQ_INVALID_SPARSITY = 1,    /* InvalidSparsity   errors.hpp:31  */
    SLQ_INVALID_DIMS = 2,        /* InvalidDims       errors.hpp:46  */
    SLQ_DIMENSION_MISMATCH = 3,  /* DimensionMismatch errors.hpp:26  */
    SLQ_RANK_DEFICIENT = 4,      /* RankDeficient     errors.hpp:16  */
    SLQ_SINGULAR_TRIANGULAR = 5, /* SingularTriangular errors.hpp:21 */
    SLQ_CUDA = 6,
    SLQ_NCCL = 7,
    SLQ_OOM = 8,
    SLQ_UNSUPPORTED = 9,
    SLQ_INVALID_ARG = 10,
    SLQ_INVALID_DISTORTION = 11, /* InvalidDistortion errors.hpp:39 */
    SLQ_DIVERGENCE = 12          /* Divergence        errors.hpp:64 */
} slq_status;

typedef enum { SLQ_TERM_TOLERANCE = 0, SLQ_TERM_MAXITER = 1, SLQ_TERM_BREAKDOWN = 2 } slq_termination;

/* ------------------------------------------------------------ context -- */

typedef struct slq_ctx slq_ctx;

const char* slq_last_error(void);
const char* slq_version(void);

/* One context per device per thread.  All work is issued on the context's
 * stream (its own, unless slq_ctx_set_stream adopts a caller stream). */
int slq_ctx_create(int device, slq_ctx** out);
int slq_ctx_destroy(slq_ctx* ctx);
int slq_ctx_set_stream(slq_ctx* ctx, void* cuda_stream);
int slq_ctx_synchronize(slq_ctx* ctx);
/* Number of kernels this context launched so far (instrumentation). */
int64_t slq_ctx_kernel_launches(const slq_ctx* ctx);

/* Multi-GPU (one process per GPU).  Replaces the reference's in-process
 * WorkerPool (distsim.hpp:77-146): rank 0 creates the id, the caller ships
 * it to the other ranks, every rank calls slq_ctx_init_comm.  Collectives
 * (ncclReduce / ncclBroadcast / ncclAllReduce over NVLink) are then issued
 * inside slq_solve. */
int slq_comm_unique_id(unsigned char id_out[128]);
int slq_ctx_init_comm(slq_ctx* ctx, const unsigned char id[128], int rank, int nranks);

/* Host-side collectives (an alternative to NCCL, for tests and for callers
 * that bring their own transport): in-place operations on host buffers of
 * `count` doubles, called by the library with the stream synchronized (each
 * call is a host round trip; the iteration graphs are not used).  Every rank
 * calls them in the same order; return 0 on success.  reduce_sum_root needs
 * the sum on rank 0 only; broadcast_root copies rank 0's buffer to all. */
typedef struct {
    int (*allreduce_sum)(void* user, double* buf, int64_t count);
    int (*reduce_sum_root)(void* user, double* buf, int64_t count);
    int (*broadcast_root)(void* user, double* buf, int64_t count);
    void* user;
} slq_host_comm;
int slq_ctx_set_host_comm(slq_ctx* ctx, const slq_host_comm* comm, int rank, int nranks);

/* Diagnostics: with SLQ_GUARD=1 in the environment, the library's device
 * scratch buffers are allocated with 64 KB guard bands (0xA5) on both sides;
 * this call synchronizes the device and reports how many bands were found
 * overwritten (live buffers now + buffers released since the process began).
 * Without SLQ_GUARD it reports 0. */
int slq_debug_check_guards(int64_t* corrupted);
/* Self-test of that mechanism (SLQ_GUARD=1 only): plants one out-of-bounds
 * write behind a scratch buffer and reports whether the release check saw it. */
int slq_debug_guard_selftest(int* detected);

/* distsim.hpp:31-42 partition_rows: boundaries[0..p] */
int slq_partition_rows(int64_t m, int p, int64_t* boundaries);

/* ------------------------------------------------------------ sketch --- */

typedef struct {
    int64_t columns_resampled; /* sketch.hpp:65-68 RejectionStats */
    int64_t resample_rounds;
} slq_rejection_stats;

/* sketch.hpp:178-194 generate_sparse_sign (col_begin = 0, ncols = m) and
 * sketch.hpp:149-173 detail::sparse_sign_block (any global column window, the
 * unit of distsim.hpp:346-361 dist_generate_sparse_sign).  Outputs the
 * reference CSC layout into host buffers: row_indices[ncols*zeta],
 * values[ncols*zeta], col_pointers[ncols+1].  Bit-exact with the reference.
 * stats may be NULL. */
int slq_generate_sparse_sign(slq_ctx* ctx, int64_t d, int64_t col_begin, int64_t ncols,
                             int64_t zeta, uint64_t seed, int64_t* row_indices, double* values,
                             int64_t* col_pointers, slq_rejection_stats* stats);

/* sketch.hpp:105-124 rejection_sample_columns: out[m*zeta] */
int slq_rejection_sample_columns(slq_ctx* ctx, int64_t d, int64_t m, int64_t zeta, uint64_t seed,
                                 int64_t* out, slq_rejection_stats* stats);

/* ------------------------------------------------ device dense matrix -- */

typedef struct slq_dense slq_dense;

/* Uploads rows [0, m) of a host column-major A (and optional b) as this
 * rank's row block, whose first row is global row row_begin (sketch columns
 * are keyed by global row id, distsim.hpp:346-361).  Replaces distribute()
 * (distsim.hpp:215-233).  Converts to the device layout on the GPU. */
int slq_dense_upload(slq_ctx* ctx, const double* A, int64_t m, int64_t n, int64_t lda,
                     const double* b, int64_t row_begin, slq_dense** out);
/* Allocates a device block and returns its row-major storage so the caller
 * (e.g. a device-side generator) can fill it in place: element (i, j) at
 * dev[i*ld + j], b in column n, columns > n zero. */
int slq_dense_create(slq_ctx* ctx, int64_t m, int64_t n, int64_t row_begin, slq_dense** out,
                     double** dev_ptr, int64_t* ld);
/* Wraps caller-owned device storage with the same layout (not freed). */
int slq_dense_wrap(slq_ctx* ctx, double* dev_ptr, int64_t m, int64_t n, int64_t ld,
                   int64_t row_begin, slq_dense** out);
int slq_dense_set_rhs(slq_dense* A, const double* b_host);
int slq_dense_free(slq_dense* A);
int64_t slq_dense_ld(const slq_dense* A);

/* sketch.hpp:297 apply(SparseSignSketch, DenseMatrix) -> csc_matrix.hpp:103-120
 * and sketch.hpp:304 sketch_vector -> csc_matrix.hpp:71-82, fused: the sparse
 * sign sketch (d, zeta, seed) is generated on the device for this rank's rows
 * and applied to [A | b] in one pass.  Y (d x n, column-major, ldy = d) and
 * Sb (d) are host outputs; either may be NULL.  exact != 0 forces the
 * reference's serial accumulation order (bit-identical Y on one GPU);
 * exact == 0 (and slq_solve) runs the FP64 tensor-core tile gather, whose
 * sums differ from the serial order by rounding only (~1e-15 relative). */
int slq_sketch_apply(slq_ctx* ctx, const slq_dense* A, int64_t d, int64_t zeta, uint64_t seed,
                     int exact, double* Y, double* Sb);

/* csc_matrix.hpp:103-120 spmm(csc, dense) for a caller-given CSC S (d x m)
 * and host column-major A (m x n, lda): Y = S A (column-major d x n).
 * Same accumulation order as the reference (bit-identical).  A sparse-sign S
 * (all |values| equal) runs the sketch gather; any other values the general
 * kernel (row-sorted entries, one thread per Y entry).  The entries are
 * validated on the device (SLQ_INVALID_ARG for a row out of range). */
int slq_spmm_csc_dense(slq_ctx* ctx, int64_t d, int64_t m, const int64_t* row_indices,
                       const double* values, const int64_t* col_pointers, const double* A,
                       int64_t n, int64_t lda, double* Y);

/* ------------------------------------------------ device sparse matrix -- */

/* A row block of a sparse A in CSR on the device (int64 row pointers, int32
 * column indices, fp64 values).  Replaces the CscMatrix operand of
 * sketch.hpp:298, csc_matrix.hpp:71-136 and lsqr.hpp:198-212, and its row
 * distribution csc_row_block / distribute (csc_matrix.hpp:139-152,
 * distsim.hpp:235-246). */
typedef struct slq_sparse slq_sparse;

/* From the reference's host CSC layout (col_pointers[n+1], row_indices[nnz]
 * int64, values[nnz] fp64) of this rank's rows [0, m), first row = global
 * row row_begin; b (m, may be NULL) is the right-hand side of these rows. */
int slq_sparse_upload_csc(slq_ctx* ctx, int64_t m, int64_t n, const int64_t* col_pointers,
                          const int64_t* row_indices, const double* values, const double* b,
                          int64_t row_begin, slq_sparse** out);
/* Allocates the device CSR (with bulk-copy slack) for the caller to fill in
 * place: row_ptr[m+1], col_idx[nnz] (sorted within rows), values[nnz],
 * b[m] when with_b. */
int slq_sparse_create_csr(slq_ctx* ctx, int64_t m, int64_t n, int64_t nnz, int64_t row_begin, int with_b,
                          slq_sparse** out, int64_t** row_ptr, int32_t** col_idx, double** values,
                          double** b);
int slq_sparse_set_rhs(slq_sparse* A, const double* b_host);
/* Benchmark harness: fills A (created with
 * nnz = m * nnz_per_row) with nnz_per_row distinct random columns per row,
 * drawn by the reference's rejection sampler keyed by global row id, values
 * +-col_scale[col] (host array of n, NULL = +-1). */
int slq_sparse_fill_random(slq_sparse* A, int64_t nnz_per_row, uint64_t seed, const double* col_scale);
int slq_sparse_free(slq_sparse* A);
/* (Re)builds the row-blocked CSC copy of A that the LSQR / gradient solves
 * stream for A^T u (the first solve on A builds it implicitly and keeps it
 * with the matrix).  Call it after rewriting the CSR arrays of a matrix from
 * slq_sparse_create_csr in place once a solve has run on it.  No reference
 * counterpart: part of the device representation, like the CSC -> CSR
 * conversion of slq_sparse_upload_csc. */
int slq_sparse_prepare(slq_ctx* ctx, slq_sparse* A);

/* sketch.hpp:298 + :304 for a sparse operand: Y = S A (d x n, column-major)
 * and Sb, bit-identical to spmm(csc, csc) / matvec(csc) on one GPU. */
int slq_sketch_apply_sparse(slq_ctx* ctx, const slq_sparse* A, int64_t d, int64_t zeta, uint64_t seed,
                            double* Y, double* Sb);

/* csc_matrix.hpp:123-136 spmm(csc, csc): Y = S A for a caller CSC S (d x m;
 * sparse-sign or arbitrary values, as slq_spmm_csc_dense) and a host CSC A
 * (m x n); reference order (bit-identical). */
int slq_spmm_csc_csc(slq_ctx* ctx, int64_t d, int64_t m, const int64_t* s_rows, const double* s_vals,
                     const int64_t* s_colptr, int64_t n, const int64_t* a_colptr, const int64_t* a_rows,
                     const double* a_vals, double* Y);

/* ------------------------------------------------------ preconditioner -- */

/* qr.hpp:21-89 householder_qr.  Y d x n column-major (ldy >= d); Q (d x n,
 * may be NULL) and R (n x n) column-major.  SLQ_RANK_DEFICIENT when a column
 * norm falls below 1e-12 * max|Y|. */
int slq_householder_qr(slq_ctx* ctx, const double* Y, int64_t d, int64_t n, int64_t ldy, double* Q,
                       double* R);

/* triangular.hpp:14-33 tri_inverse.  SLQ_SINGULAR_TRIANGULAR on a zero diagonal. */
int slq_tri_inverse(slq_ctx* ctx, const double* R, int64_t n, double* M);

/* preconditioner.hpp:35-44 build_preconditioner and, when Sb and x0 are
 * given, preconditioner.hpp:48-53 initial_guess (x0 = M Q^T Sb).  Q may be
 * NULL (it is then never formed).  build_time: seconds (QR + inverse). */
int slq_build_preconditioner(slq_ctx* ctx, const double* Y, int64_t d, int64_t n, int64_t ldy,
                             const double* Sb, double* M, double* Q, double* x0,
                             double* build_time);

/* preconditioner.hpp:48-53 initial_guess: x0 = M (Q^T Sb) for a given
 * preconditioner (M n x n, Q d x n, column-major). */
int slq_initial_guess(slq_ctx* ctx, const double* M, const double* Q, int64_t d, int64_t n, const double* Sb,
                      double* x0);

/* triangular.hpp:36-61 tri_upper_matvec (trans = 0: y = R x) and
 * tri_upper_rmatvec (trans = 1: y = R^T x); preconditioner.hpp:55-56
 * apply_M / apply_Mt are these with R = M. */
int slq_tri_upper_matvec(slq_ctx* ctx, const double* R, int64_t n, const double* x, double* y, int trans);

/* ------------------------------------------------- operator products -- */

/* The Op concept of the reference (operators.hpp:15-51 SerialOperator;
 * distsim.hpp:283-331 dist_matvec / dist_rmatvec / dist_rmatvec_and_norm):
 * one HBM pass of the device operand each.  Host vectors in and out.
 *   matvec:  y[m] = A x[n]   (this rank's rows; no communication)
 *   rmatvec: z[n] = A^T y[m] and, when ynorm2 != NULL, *ynorm2 = ||y||^2 --
 *            fused (the one-synchronization product of lsqr.hpp:120-127);
 *            with a communicator both are summed over ranks (one allreduce). */
int slq_dense_matvec(slq_ctx* ctx, const slq_dense* A, const double* x, double* y);
int slq_dense_rmatvec(slq_ctx* ctx, const slq_dense* A, const double* y, double* z, double* ynorm2);
int slq_sparse_matvec(slq_ctx* ctx, const slq_sparse* A, const double* x, double* y);
int slq_sparse_rmatvec(slq_ctx* ctx, const slq_sparse* A, const double* y, double* z, double* ynorm2);

/* ---------------------------------------------------------------- LSQR -- */

typedef struct {
    double eps;              /* lsqr.hpp:15 stop when phi_bar <= eps * beta_1 */
    int64_t maxit;           /* lsqr.hpp:16 */
    const double* x_star;    /* lsqr.hpp:17 record ||A (x_star - x_t)|| (host, n) or NULL */
    int32_t track_true_residual; /* lsqr.hpp:18 record ||b - A x_t|| */
    int32_t one_sync;        /* lsqr_one_sync (lsqr.hpp:185) vs lsqr (lsqr.hpp:175) */
    /* extension (off by default): also stop when the backward error
     * ||A^T r|| / (||A|| ||r||) is <= backward_tol.  The device triggers on
     * the Paige-Saunders estimate alpha_{t+1} |c_t| <= trigger (initially
     * backward_tol); the host then measures the backward error with one
     * direct A^T r pass (a_norm_est = ||A||_2, 1 if 0) and accepts
     * (termination Tolerance, report.backward_error set) or resumes with a
     * trigger tightened by the measured ratio.  a_norm_est > 0 alone only
     * reports the backward error at exit. */
    double backward_tol;
    double a_norm_est;
    /* lsqr.hpp:21 on_bidiag hook: called after each iteration with the
     * recomputed norms of u_{t+1} and v_{t+1}; forces a host sync per step. */
    void (*on_bidiag)(void* user, int64_t t, double u_norm, double v_norm);
    void* on_bidiag_user;
} slq_solve_opts;

void slq_solve_opts_default(slq_solve_opts* o);

typedef struct {
    int64_t iterations;        /* solve_report.hpp:38 */
    int32_t termination;       /* slq_termination, solve_report.hpp:11 */
    int32_t pad0;
    int64_t sync_count;        /* reductions (allreduce calls) solve_report.hpp:42 */
    int64_t broadcasts;
    int64_t init_reductions;
    int64_t init_broadcasts;
    double wall_time;          /* seconds, solve_report.hpp:47 */
    int64_t n_estimate;        /* entries written to residual_estimate */
    int64_t n_err;             /* entries written to iterates_error */
    int64_t n_true;            /* entries written to residual_true */
    double backward_error;     /* ||A^T r||/(||A|| ||r||) at exit when computed, else -1 */
} slq_report;

/* lsqr.hpp:175-212 lsqr / lsqr_one_sync over a device matrix (serial operator
 * on one GPU, the row-partitioned DistOperator of distsim.hpp:413-450 when
 * the context has a communicator).  M (n x n upper, column-major), x0 (n) and
 * b (this rank's rows; NULL = use the b stored with A) are host buffers.
 * History buffers (host, may be NULL) need maxit+1 (estimate) and maxit+2
 * (error / true) entries. */
int slq_lsqr(slq_ctx* ctx, const slq_dense* A, const double* M, const double* b, const double* x0,
             const slq_solve_opts* opts, double* x_out, slq_report* report,
             double* residual_estimate, double* iterates_error, double* residual_true);

/* lsqr.hpp:198-202 / :208-212 -- LSQR over a sparse operand (arguments as slq_lsqr). */
int slq_lsqr_sparse(slq_ctx* ctx, const slq_sparse* A, const double* M, const double* b, const double* x0,
                    const slq_solve_opts* opts, double* x_out, slq_report* report,
                    double* residual_estimate, double* iterates_error, double* residual_true);

/* -------------------------------------------------- gradient family --- */

typedef struct {
    double alpha;   /* gradient.hpp:20-24 GradientParams */
    double beta;
    double eta_hat;
} slq_gradient_params;

/* gradient.hpp:27-34 hbm_params: alpha = (1-eta^2)^2, beta = eta^2.
 * SLQ_INVALID_DISTORTION unless 0 <= eta_hat < 1. */
int slq_hbm_params(double eta_hat, slq_gradient_params* out);
/* gradient.hpp:37-48 gd_params: alpha = (1-eta^2)^2 / (1+eta^2), beta = 0. */
int slq_gd_params(double eta_hat, slq_gradient_params* out);

/* gradient.hpp:56-115 gradient_descent_hbm over a device matrix (arguments as
 * slq_lsqr; opts->one_sync / backward_tol / on_bidiag are ignored).  Heavy
 * ball x_t = x_{t-1} + alpha M M^T A^T r_{t-1} + beta (x_{t-1} - x_{t-2});
 * stops when ||M^T A^T r|| <= eps times its first value.  One HBM pass over A
 * per iteration (r_t and A^T r_t from the same sweep) and one n-vector
 * allreduce with a communicator.  SLQ_DIVERGENCE when ||M^T A^T r|| grows by
 * 1e6 (gradient.hpp:82-85). */
int slq_gradient_descent_hbm(slq_ctx* ctx, const slq_dense* A, const double* M, const double* b,
                             const double* x0, const slq_gradient_params* params,
                             const slq_solve_opts* opts, double* x_out, slq_report* report,
                             double* residual_estimate, double* iterates_error, double* residual_true);
/* gradient.hpp:117-122 -- the CscMatrix overload, over a sparse operand. */
int slq_gradient_descent_hbm_sparse(slq_ctx* ctx, const slq_sparse* A, const double* M, const double* b,
                                    const double* x0, const slq_gradient_params* params,
                                    const slq_solve_opts* opts, double* x_out, slq_report* report,
                                    double* residual_estimate, double* iterates_error,
                                    double* residual_true);

/* ---------------------------------------------------- whole pipeline --- */

typedef struct {
    double generate, apply, reduce, qr, inverse, x0, lsqr, total; /* seconds (CUDA events) */
    double lsqr_per_iteration;
    int64_t nccl_calls;
    int64_t kernel_launches;
} slq_phase_times;

/* The paper's Alg. 1 end to end on the device-resident A (this rank's row
 * block): sparse-sign sketch (d, zeta, seed) -> S[A b] -> (NCCL reduce) ->
 * QR / M = R^-1 / x0 on rank 0 -> (NCCL broadcast) -> LSQR.  Equivalent to
 * the reference sequence generate_sparse_sign, apply, sketch_vector,
 * build_preconditioner, initial_guess, lsqr[_one_sync]
 * (sketch.hpp:178,297,304; preconditioner.hpp:35,48; lsqr.hpp:175,185). */
int slq_solve(slq_ctx* ctx, const slq_dense* A, int64_t d, int64_t zeta, uint64_t seed,
              const slq_solve_opts* opts, double* x_out, slq_report* report,
              slq_phase_times* times, double* residual_estimate);

/* slq_solve for a sparse operand (BASELINE config C4). */
int slq_solve_sparse(slq_ctx* ctx, const slq_sparse* A, int64_t d, int64_t zeta, uint64_t seed,
                     const slq_solve_opts* opts, double* x_out, slq_report* report,
                     slq_phase_times* times, double* residual_estimate);

/* Kernel timing for the roofline report (CUDA events on the context stream):
 * out[0] = seconds per K4 fused LSQR pass launch (average over reps),
 * out[1] = seconds for the sketch (K1 generate + K2 apply) of A,
 * out[2] = seconds for K1 generation alone,
 * out[3] = seconds for QR + R^-1 + x0 of the resulting d x n sketch. */
int slq_time_kernels(slq_ctx* ctx, const slq_dense* A, int64_t d, int64_t zeta, uint64_t seed, int reps,
                     double* out);

/* Benchmark helper (no reference counterpart): average device seconds of one
 * K4s launch -- the sparse LSQR pass u_hat = A p + c u, z = A^T u_hat,
 * ||u_hat||^2 -- over `reps` launches on the context stream (CUDA events). */
int slq_time_sparse_pass(slq_ctx* ctx, const slq_sparse* A, int reps, double* seconds);

/* slq_solve from host buffers: upload (column-major A, lda) + solve + free. */
int slq_solve_host(slq_ctx* ctx, const double* A, int64_t m, int64_t n, int64_t lda,
                   const double* b, int64_t row_begin, int64_t d, int64_t zeta, uint64_t seed,
                   const slq_solve_opts* opts, double* x_out, slq_report* report,
                   slq_phase_times* times, double* residual_estimate);

#ifdef __cplusplus
}
#endif

#endif /* SLQ_B200_H */
