/*
 * sketchlsq_oracle.c -- CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the
 * B200 product in paper_2506_03070_b200/.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it; the product path never does.
 *
 * It restates, in plain sequential C (IEEE double, no FMA contraction:
 * build with -ffp-contract=off), the algorithms of the reference header
 * library `sketchlsq` (/root/reference/proj/include/sketchlsq/).  Every
 * function cites the reference file:line it follows.  Parity of this
 * restatement is pinned against the compiled reference (oracle/_ref) and
 * against the known-answer vectors of SURVEY.md Appendix A
 * (tests/golden/, tests/test_oracle.py).
 *
 * Status codes mirror the reference exception types (errors.hpp:9-76).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OK 0
#define E_INVALID_SPARSITY 1
#define E_INVALID_DIMS 2
#define E_DIMENSION_MISMATCH 3
#define E_RANK_DEFICIENT 4
#define E_SINGULAR_TRIANGULAR 5
#define E_OOM 8
#define E_INVALID_DISTORTION 11
#define E_DIVERGENCE 12

typedef int64_t idx;

/* ---------------------------------------------------------------- RNG */

/* rng.hpp:11-16 -- splitmix64 finalizer */
uint64_t orc_mix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* rng.hpp:29 -- Rng(seed) */
uint64_t orc_rng_seed(uint64_t seed) { return orc_mix64(seed); }

/* rng.hpp:32-33 -- Rng(seed, stream) */
uint64_t orc_rng_stream(uint64_t seed, uint64_t stream) {
    return orc_mix64(orc_mix64(seed) ^ (0x6a09e667f3bcc909ULL + stream));
}

/* rng.hpp:35-41 -- Weyl step then the same finalizer body */
uint64_t orc_next_u64(uint64_t* state) {
    *state += 0x9e3779b97f4a7c15ULL;
    uint64_t z = *state;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* rng.hpp:44-53 -- Lemire multiply-shift with rejection */
uint64_t orc_uniform_below(uint64_t* state, uint64_t bound) {
    for (;;) {
        uint64_t x = orc_next_u64(state);
        unsigned __int128 prod = (unsigned __int128)x * bound;
        uint64_t lo = (uint64_t)prod;
        if (lo >= bound || lo >= (0 - bound) % bound) return (uint64_t)(prod >> 64);
    }
}

/* rng.hpp:56-58 */
double orc_uniform01(uint64_t* state) { return (double)(orc_next_u64(state) >> 11) * 0x1.0p-53; }

/* rng.hpp:61 */
double orc_uniform_sym(uint64_t* state) { return 2.0 * orc_uniform01(state) - 1.0; }

/* rng.hpp:64 */
double orc_sign(uint64_t* state) { return (orc_next_u64(state) & 1u) ? 1.0 : -1.0; }

/* rng.hpp:67-82 -- Box-Muller with a cached spare (state carried by caller) */
typedef struct { uint64_t s; int have_spare; double spare; } orc_normal_state;
static double orc_normal(orc_normal_state* g) {
    if (g->have_spare) { g->have_spare = 0; return g->spare; }
    double u, v, s;
    do {
        u = orc_uniform_sym(&g->s);
        v = orc_uniform_sym(&g->s);
        s = u * u + v * v;
    } while (s >= 1.0 || s == 0.0);
    double f = sqrt(-2.0 * log(s) / s);
    g->spare = v * f;
    g->have_spare = 1;
    return u * f;
}

/* ------------------------------------------------------ sparse sign */

static void sort_idx(idx* a, idx n) { /* insertion sort == std::sort result on distinct-or-equal keys */
    for (idx i = 1; i < n; ++i) {
        idx v = a[i], j = i - 1;
        while (j >= 0 && a[j] > v) { a[j + 1] = a[j]; --j; }
        a[j + 1] = v;
    }
}

/* sketch.hpp:75-94 -- draw zeta, sort, redraw left-to-right duplicates,
 * re-sort, repeat.  Returns 1 when any redraw happened. */
int orc_rejection_sample_one(idx d, idx zeta, uint64_t* st, idx* out, idx* rounds) {
    for (idx i = 0; i < zeta; ++i) out[i] = (idx)orc_uniform_below(st, (uint64_t)d);
    sort_idx(out, zeta);
    int resampled = 0;
    for (;;) {
        idx bad = 0;
        for (idx i = 1; i < zeta; ++i) {
            if (out[i] == out[i - 1]) {
                out[i] = (idx)orc_uniform_below(st, (uint64_t)d);
                ++bad;
            }
        }
        if (bad == 0) break;
        resampled = 1;
        if (rounds) ++(*rounds);
        sort_idx(out, zeta);
    }
    return resampled;
}

/* sketch.hpp:105-124 */
int orc_rejection_sample_columns(idx d, idx m, idx zeta, uint64_t seed, idx* C,
                                 idx* cols_resampled, idx* rounds_total) {
    if (zeta > d || zeta < 1) return E_INVALID_SPARSITY;
    for (idx j = 0; j < m; ++j) {
        uint64_t st = orc_rng_stream(seed, 2 * (uint64_t)j);
        idx rounds = 0;
        int r = orc_rejection_sample_one(d, zeta, &st, C + j * zeta, &rounds);
        if (cols_resampled) *cols_resampled += r;
        if (rounds_total) *rounds_total += rounds;
    }
    return OK;
}

/* sketch.hpp:149-173 (block of global columns [col_begin, col_end));
 * sketch.hpp:178-189 (generate_sparse_sign == block [0, m)). */
int orc_sparse_sign_block(idx d, idx zeta, uint64_t seed, idx col_begin, idx col_end,
                          idx* row_indices, double* values, idx* col_pointers,
                          idx* cols_resampled, idx* rounds_total) {
    if (zeta > d || zeta < 1) return E_INVALID_SPARSITY;
    const double val = 1.0 / sqrt((double)zeta);
    col_pointers[0] = 0;
    for (idx j = 0; j < col_end - col_begin; ++j) {
        uint64_t gj = (uint64_t)(col_begin + j);
        uint64_t ist = orc_rng_stream(seed, 2 * gj);
        uint64_t vst = orc_rng_stream(seed, 2 * gj + 1);
        idx rounds = 0;
        int r = orc_rejection_sample_one(d, zeta, &ist, row_indices + j * zeta, &rounds);
        if (cols_resampled) *cols_resampled += r;
        if (rounds_total) *rounds_total += rounds;
        for (idx i = 0; i < zeta; ++i) values[j * zeta + i] = orc_sign(&vst) * val;
        col_pointers[j + 1] = (j + 1) * zeta;
    }
    return OK;
}

/* ---------------------------------------------------- CSC products */

/* csc_matrix.hpp:103-120 -- Y = S A, A column-major m x n; order: column j
 * of A, then k ascending, then nonzeros of S column k in storage order. */
int orc_spmm_csc_dense(idx d, idx m, const idx* rows, const double* vals, const idx* colptr,
                       const double* A, idx n, double* Y) {
    memset(Y, 0, sizeof(double) * (size_t)(d * n));
    for (idx j = 0; j < n; ++j) {
        const double* aj = A + j * m;
        double* yj = Y + j * d;
        for (idx k = 0; k < m; ++k) {
            const double akj = aj[k];
            if (akj == 0.0) continue;
            for (idx p = colptr[k]; p < colptr[k + 1]; ++p) yj[rows[p]] += vals[p] * akj;
        }
    }
    return OK;
}

/* csc_matrix.hpp:71-82 -- y = S x */
int orc_csc_matvec(idx d, idx m, const idx* rows, const double* vals, const idx* colptr,
                   const double* x, double* y) {
    memset(y, 0, sizeof(double) * (size_t)d);
    for (idx j = 0; j < m; ++j) {
        const double xj = x[j];
        if (xj == 0.0) continue;
        for (idx p = colptr[j]; p < colptr[j + 1]; ++p) y[rows[p]] += vals[p] * xj;
    }
    return OK;
}

/* csc_matrix.hpp:85-96 -- x = S^T y (per-column dot) */
int orc_csc_rmatvec(idx d, idx m, const idx* rows, const double* vals, const idx* colptr,
                    const double* y, double* x) {
    (void)d;
    for (idx j = 0; j < m; ++j) {
        double s = 0.0;
        for (idx p = colptr[j]; p < colptr[j + 1]; ++p) s += vals[p] * y[rows[p]];
        x[j] = s;
    }
    return OK;
}

/* csc_matrix.hpp:123-136 -- Y = S A for CSC A (m x n) */
int orc_spmm_csc_csc(idx d, const idx* srows, const double* svals, const idx* scolptr,
                     idx n, const idx* arows, const double* avals, const idx* acolptr, double* Y) {
    memset(Y, 0, sizeof(double) * (size_t)(d * n));
    for (idx j = 0; j < n; ++j) {
        double* yj = Y + j * d;
        for (idx q = acolptr[j]; q < acolptr[j + 1]; ++q) {
            const idx k = arows[q];
            const double akj = avals[q];
            for (idx p = scolptr[k]; p < scolptr[k + 1]; ++p) yj[srows[p]] += svals[p] * akj;
        }
    }
    return OK;
}

/* ---------------------------------------------------- dense BLAS-2 */

/* dense_matrix.hpp:53-67 -- y = A x (column-axpy order, zero x_j skipped) */
void orc_matvec(const double* A, idx m, idx n, const double* x, double* y) {
    memset(y, 0, sizeof(double) * (size_t)m);
    for (idx j = 0; j < n; ++j) {
        const double xj = x[j];
        if (xj == 0.0) continue;
        const double* aj = A + j * m;
        for (idx i = 0; i < m; ++i) y[i] += aj[i] * xj;
    }
}

/* dense_matrix.hpp:70-84 -- y = A^T x (sequential dot per column) */
void orc_rmatvec(const double* A, idx m, idx n, const double* x, double* y) {
    for (idx j = 0; j < n; ++j) {
        const double* aj = A + j * m;
        double s = 0.0;
        for (idx i = 0; i < m; ++i) s += aj[i] * x[i];
        y[j] = s;
    }
}

/* vector_ops.hpp:31-35 */
static double norm2(const double* x, idx n) {
    double s = 0.0;
    for (idx i = 0; i < n; ++i) s += x[i] * x[i];
    return sqrt(s);
}

/* triangular.hpp:36-47 -- y = R x, upper triangle only */
void orc_tri_upper_matvec(const double* R, idx n, const double* x, double* y) {
    memset(y, 0, sizeof(double) * (size_t)n);
    for (idx j = 0; j < n; ++j) {
        const double xj = x[j];
        if (xj == 0.0) continue;
        const double* rj = R + j * n;
        for (idx i = 0; i <= j; ++i) y[i] += rj[i] * xj;
    }
}

/* triangular.hpp:50-61 -- y = R^T x */
void orc_tri_upper_rmatvec(const double* R, idx n, const double* x, double* y) {
    for (idx j = 0; j < n; ++j) {
        const double* rj = R + j * n;
        double s = 0.0;
        for (idx i = 0; i <= j; ++i) s += rj[i] * x[i];
        y[j] = s;
    }
}

/* ------------------------------------------------------------- QR */

/* qr.hpp:21-89 -- thin Householder QR of column-major d x n Y.
 * Q (d x n) may be NULL; R (n x n) must not be.  rank column returned in
 * *bad_col on E_RANK_DEFICIENT. */
int orc_householder_qr(const double* Y, idx d, idx n, double* Q, double* R, idx* bad_col) {
    if (d < n) return E_DIMENSION_MISMATCH;
    double mx = 0.0;
    for (idx i = 0; i < d * n; ++i) mx = fmax(mx, fabs(Y[i]));
    const double rank_tol = 1e-12 * mx;
    double* W = (double*)malloc(sizeof(double) * (size_t)(d * n));
    double* tau = (double*)calloc((size_t)n, sizeof(double));
    if (!W || !tau) { free(W); free(tau); return E_OOM; }
    memcpy(W, Y, sizeof(double) * (size_t)(d * n));
    for (idx k = 0; k < n; ++k) {
        double* wk = W + k * d;
        double sigma = 0.0;
        for (idx i = k + 1; i < d; ++i) sigma += wk[i] * wk[i];
        const double x0 = wk[k];
        const double normx = sqrt(x0 * x0 + sigma);
        if (normx < rank_tol || normx == 0.0) {
            if (bad_col) *bad_col = k;
            free(W); free(tau);
            return E_RANK_DEFICIENT;
        }
        const double beta = (x0 > 0.0) ? -normx : normx;
        const double v0 = x0 - beta;
        for (idx i = k + 1; i < d; ++i) wk[i] /= v0;
        tau[k] = (beta - x0) / beta;
        wk[k] = beta;
        for (idx j = k + 1; j < n; ++j) {
            double* wj = W + j * d;
            double s = wj[k];
            for (idx i = k + 1; i < d; ++i) s += wk[i] * wj[i];
            s *= tau[k];
            wj[k] -= s;
            for (idx i = k + 1; i < d; ++i) wj[i] -= s * wk[i];
        }
    }
    memset(R, 0, sizeof(double) * (size_t)(n * n));
    for (idx j = 0; j < n; ++j)
        for (idx i = 0; i <= j; ++i) R[j * n + i] = W[j * d + i];
    if (Q) {
        memset(Q, 0, sizeof(double) * (size_t)(d * n));
        for (idx j = 0; j < n; ++j) Q[j * d + j] = 1.0;
        for (idx k = n - 1; k >= 0; --k) {
            const double* wk = W + k * d;
            const double t = tau[k];
            for (idx j = 0; j < n; ++j) {
                double* qj = Q + j * d;
                double s = qj[k];
                for (idx i = k + 1; i < d; ++i) s += wk[i] * qj[i];
                s *= t;
                qj[k] -= s;
                for (idx i = k + 1; i < d; ++i) qj[i] -= s * wk[i];
            }
        }
    }
    for (idx k = 0; k < n; ++k) {
        if (R[k * n + k] < 0.0) {
            for (idx j = k; j < n; ++j) R[j * n + k] = -R[j * n + k];
            if (Q)
                for (idx i = 0; i < d; ++i) Q[k * d + i] = -Q[k * d + i];
        }
    }
    free(W);
    free(tau);
    return OK;
}

/* triangular.hpp:14-33 -- explicit inverse by column back-substitution */
int orc_tri_inverse(const double* R, idx n, double* M, idx* bad_diag) {
    for (idx i = 0; i < n; ++i)
        if (R[i * n + i] == 0.0) {
            if (bad_diag) *bad_diag = i;
            return E_SINGULAR_TRIANGULAR;
        }
    memset(M, 0, sizeof(double) * (size_t)(n * n));
    for (idx j = 0; j < n; ++j) {
        double* mj = M + j * n;
        mj[j] = 1.0 / R[j * n + j];
        for (idx i = j - 1; i >= 0; --i) {
            double s = 0.0;
            for (idx k = i + 1; k <= j; ++k) s += R[k * n + i] * mj[k];
            mj[i] = -s / R[i * n + i];
        }
    }
    return OK;
}

/* preconditioner.hpp:48-53 -- x0 = M (Q^T Sb) */
int orc_initial_guess(const double* M, const double* Q, idx d, idx n, const double* Sb, double* x0) {
    double* t = (double*)malloc(sizeof(double) * (size_t)n);
    if (!t) return E_OOM;
    orc_rmatvec(Q, d, n, Sb, t);
    orc_tri_upper_matvec(M, n, t, x0);
    free(t);
    return OK;
}

/* ------------------------------------------------------------ LSQR */

enum { TERM_TOLERANCE = 0, TERM_MAXITER = 1, TERM_BREAKDOWN = 2 };

typedef struct {
    long iterations;
    int termination;
    long n_estimate;   /* entries written to residual_estimate */
    long n_true;       /* entries written to residual_true */
    long n_err;        /* entries written to iterates_error */
} orc_lsqr_report;

/* The Op surface of operators.hpp:15-51 (SerialOperator<DenseMatrix> and
 * SerialOperator<CscMatrix>): only matvec / rmatvec differ. */
typedef struct {
    idx m, n;
    int csc;
    const double* A;        /* dense column-major */
    const idx* rows;        /* CSC */
    const double* vals;
    const idx* colptr;
} orc_op;

static void op_matvec(const orc_op* op, const double* x, double* y) {
    if (op->csc) orc_csc_matvec(op->m, op->n, op->rows, op->vals, op->colptr, x, y);
    else orc_matvec(op->A, op->m, op->n, x, y);
}

static void op_rmatvec(const orc_op* op, const double* y, double* x) {
    if (op->csc) orc_csc_rmatvec(op->m, op->n, op->rows, op->vals, op->colptr, y, x);
    else orc_rmatvec(op->A, op->m, op->n, y, x);
}

static void record(const orc_op* op, idx m, idx n, const double* b, const double* x,
                   const double* x_star, int track_true, double* err_hist, double* true_hist,
                   orc_lsqr_report* rep, double* wm, double* wn) {
    /* lsqr.hpp:26-37 + operators.hpp:37-42 */
    if (x_star) {
        for (idx j = 0; j < n; ++j) wn[j] = x_star[j] - x[j];
        op_matvec(op, wn, wm);
        err_hist[rep->n_err++] = norm2(wm, m);
    }
    if (track_true) {
        op_matvec(op, x, wm);
        for (idx i = 0; i < m; ++i) wm[i] = b[i] + (-1.0) * wm[i];
        true_hist[rep->n_true++] = norm2(wm, m);
    }
}

/* lsqr.hpp:50-168 (lsqr_impl), serial operator operators.hpp:15-51.
 * one_sync selects lsqr.hpp:120-127 vs lsqr.hpp:128-132. */
static int lsqr_op(const orc_op* op, const double* M, const double* b, const double* x0,
                   double eps, long maxit, int one_sync, const double* x_star, int track_true,
                   double* x_out, orc_lsqr_report* rep, double* est_hist, double* err_hist,
                   double* true_hist) {
    const idx m = op->m, n = op->n;
    memset(rep, 0, sizeof(*rep));
    double* u = (double*)malloc(sizeof(double) * (size_t)m);
    double* uh = (double*)malloc(sizeof(double) * (size_t)m);
    double* wm = (double*)malloc(sizeof(double) * (size_t)m);
    double* v = (double*)malloc(sizeof(double) * (size_t)n);
    double* w = (double*)malloc(sizeof(double) * (size_t)n);
    double* tn = (double*)malloc(sizeof(double) * (size_t)n);
    double* tn2 = (double*)malloc(sizeof(double) * (size_t)n);
    double* wn = (double*)malloc(sizeof(double) * (size_t)n);
    if (!u || !uh || !wm || !v || !w || !tn || !tn2 || !wn) return E_OOM;
    double* x = x_out;
    memcpy(x, x0, sizeof(double) * (size_t)n);

    op_matvec(op, x0, wm);
    for (idx i = 0; i < m; ++i) u[i] = b[i] + (-1.0) * wm[i];
    const double beta1 = norm2(u, m);
    record(op, m, n, b, x, x_star, track_true, err_hist, true_hist, rep, wm, wn);
    int status = OK;
    if (beta1 == 0.0) { rep->termination = TERM_TOLERANCE; rep->iterations = 0; goto done; }
    for (idx i = 0; i < m; ++i) u[i] *= 1.0 / beta1;
    op_rmatvec(op, u, tn);
    orc_tri_upper_rmatvec(M, n, tn, v);
    double alpha = norm2(v, n);
    if (alpha == 0.0) { rep->termination = TERM_TOLERANCE; rep->iterations = 0; goto done; }
    for (idx j = 0; j < n; ++j) v[j] *= 1.0 / alpha;
    orc_tri_upper_matvec(M, n, v, w);
    double phi_bar = beta1, rho_bar = alpha;

    rep->termination = TERM_MAXITER;
    rep->iterations = maxit;
    for (long t = 1; t <= maxit; ++t) {
        orc_tri_upper_matvec(M, n, v, tn);
        op_matvec(op, tn, uh);
        for (idx i = 0; i < m; ++i) uh[i] += -alpha * u[i];
        double beta;
        if (one_sync) {
            op_rmatvec(op, uh, tn);
            beta = norm2(uh, m);
        } else {
            beta = norm2(uh, m);
        }
        double beta_term = -1.0;
        if (beta < 1e-300) beta_term = 0.0;
        if (beta_term < 0.0) {
            if (one_sync) {
                for (idx j = 0; j < n; ++j) tn[j] *= 1.0 / beta;
                for (idx i = 0; i < m; ++i) uh[i] *= 1.0 / beta;
            } else {
                for (idx i = 0; i < m; ++i) uh[i] *= 1.0 / beta;
                op_rmatvec(op, uh, tn);
            }
            memcpy(u, uh, sizeof(double) * (size_t)m);
            orc_tri_upper_rmatvec(M, n, tn, tn2);          /* v_hat = M^T z */
            for (idx j = 0; j < n; ++j) tn2[j] += -beta * v[j];
            const double alpha_next = norm2(tn2, n);
            if (alpha_next < 1e-300) beta_term = beta;
            else {
                for (idx j = 0; j < n; ++j) v[j] = tn2[j] * (1.0 / alpha_next);
                alpha = alpha_next;
                const double rho = hypot(rho_bar, beta);
                const double c = rho_bar / rho;
                const double s = beta / rho;
                const double theta = s * alpha;
                rho_bar = -c * alpha;
                const double phi = c * phi_bar;
                phi_bar = s * phi_bar;
                for (idx j = 0; j < n; ++j) x[j] += (phi / rho) * w[j];
                orc_tri_upper_matvec(M, n, v, tn2);
                for (idx j = 0; j < n; ++j) w[j] = tn2[j] + (-theta / rho) * w[j];
                est_hist[rep->n_estimate++] = phi_bar;
                record(op, m, n, b, x, x_star, track_true, err_hist, true_hist, rep, wm, wn);
                if (phi_bar <= eps * beta1) {
                    rep->termination = TERM_TOLERANCE;
                    rep->iterations = t;
                    break;
                }
                continue;
            }
        }
        /* lsqr.hpp:101-111 -- final rotation with the vanished quantity as 0 */
        {
            const double rho = hypot(rho_bar, beta_term);
            const double c = rho_bar / rho;
            const double phi = c * phi_bar;
            phi_bar = (beta_term / rho) * phi_bar;
            for (idx j = 0; j < n; ++j) x[j] += (phi / rho) * w[j];
            est_hist[rep->n_estimate++] = phi_bar;
            record(op, m, n, b, x, x_star, track_true, err_hist, true_hist, rep, wm, wn);
            rep->termination = TERM_BREAKDOWN;
            rep->iterations = t;
            break;
        }
    }
done:
    free(u); free(uh); free(wm); free(v); free(w); free(tn); free(tn2); free(wn);
    return status;
}

int orc_lsqr(const double* A, idx m, idx n, const double* M, const double* b, const double* x0,
             double eps, long maxit, int one_sync, const double* x_star, int track_true,
             double* x_out, orc_lsqr_report* rep, double* est_hist, double* err_hist,
             double* true_hist) {
    orc_op op = {m, n, 0, A, NULL, NULL, NULL};
    return lsqr_op(&op, M, b, x0, eps, maxit, one_sync, x_star, track_true, x_out, rep, est_hist,
                   err_hist, true_hist);
}

/* lsqr.hpp:198-202 / :208-212 -- CscMatrix overloads (SerialOperator<CscMatrix>) */
int orc_lsqr_csc(idx m, idx n, const idx* rows, const double* vals, const idx* colptr,
                 const double* M, const double* b, const double* x0, double eps, long maxit,
                 int one_sync, const double* x_star, int track_true, double* x_out,
                 orc_lsqr_report* rep, double* est_hist, double* err_hist, double* true_hist) {
    orc_op op = {m, n, 1, NULL, rows, vals, colptr};
    return lsqr_op(&op, M, b, x0, eps, maxit, one_sync, x_star, track_true, x_out, rep, est_hist,
                   err_hist, true_hist);
}

/* ------------------------------------------------- gradient family */

/* gradient.hpp:27-48 hbm_params / gd_step_size: alpha, beta from eta_hat. */
int orc_hbm_params(double eta, double* alpha, double* beta) {
    if (!(eta >= 0.0 && eta < 1.0)) return E_INVALID_DISTORTION;
    const double e2 = eta * eta;
    *alpha = (1.0 - e2) * (1.0 - e2);
    *beta = e2;
    return OK;
}
int orc_gd_params(double eta, double* alpha, double* beta) {
    if (!(eta >= 0.0 && eta < 1.0)) return E_INVALID_DISTORTION;
    const double e2 = eta * eta;
    *alpha = (1.0 - e2) * (1.0 - e2) / (1.0 + e2);
    *beta = 0.0;
    return OK;
}

/* gradient.hpp:56-115 gradient_descent_hbm (heavy ball; beta = 0 is plain
 * gradient descent) over the serial operator:
 *   h = M^T A^T r_{t-1}; metric = ||h||; Divergence if metric > 1e6 metric_1;
 *   x_t = (1+beta) x_{t-1} - beta x_{t-2} + alpha M h; r_t = b - A x_t;
 *   stop when metric <= eps metric_1. */
static int gd_op(const orc_op* op, const double* M, const double* b, const double* x0, double alpha,
                 double beta, double eps, long maxit, const double* x_star, int track_true, double* x_out,
                 orc_lsqr_report* rep, double* est_hist, double* err_hist, double* true_hist) {
    const idx m = op->m, n = op->n;
    memset(rep, 0, sizeof(*rep));
    double* r = (double*)malloc(sizeof(double) * (size_t)m);
    double* wm = (double*)malloc(sizeof(double) * (size_t)m);
    double* xp = (double*)malloc(sizeof(double) * (size_t)n);
    double* xn = (double*)malloc(sizeof(double) * (size_t)n);
    double* tn = (double*)malloc(sizeof(double) * (size_t)n);
    double* h = (double*)malloc(sizeof(double) * (size_t)n);
    double* g = (double*)malloc(sizeof(double) * (size_t)n);
    double* wn = (double*)malloc(sizeof(double) * (size_t)n);
    if (!r || !wm || !xp || !xn || !tn || !h || !g || !wn) return E_OOM;
    double* x = x_out;
    memcpy(x, x0, sizeof(double) * (size_t)n);
    memcpy(xp, x0, sizeof(double) * (size_t)n);
    op_matvec(op, x, wm);
    for (idx i = 0; i < m; ++i) r[i] = b[i] + (-1.0) * wm[i];
    record(op, m, n, b, x, x_star, track_true, err_hist, true_hist, rep, wm, wn);
    int status = OK;
    double metric0 = -1.0;
    rep->termination = TERM_MAXITER;
    rep->iterations = maxit;
    for (long t = 1; t <= maxit; ++t) {
        op_rmatvec(op, r, tn);
        orc_tri_upper_rmatvec(M, n, tn, h);
        const double metric = norm2(h, n);
        if (metric0 < 0.0) metric0 = metric;
        if (metric > 1e6 * metric0) { status = E_DIVERGENCE; break; }
        orc_tri_upper_matvec(M, n, h, g);
        for (idx j = 0; j < n; ++j) {
            double v = x[j];
            v *= 1.0 + beta;          /* scal(1 + beta, x_next) */
            v += -beta * xp[j];       /* axpy(-beta, x_prev, x_next) */
            v += alpha * g[j];        /* axpy(alpha, g, x_next) */
            xn[j] = v;
        }
        memcpy(xp, x, sizeof(double) * (size_t)n);
        memcpy(x, xn, sizeof(double) * (size_t)n);
        op_matvec(op, x, wm);
        for (idx i = 0; i < m; ++i) r[i] = b[i] + (-1.0) * wm[i];
        est_hist[rep->n_estimate++] = metric;
        record(op, m, n, b, x, x_star, track_true, err_hist, true_hist, rep, wm, wn);
        if (metric <= eps * metric0) {
            rep->termination = TERM_TOLERANCE;
            rep->iterations = t;
            break;
        }
    }
    free(r); free(wm); free(xp); free(xn); free(tn); free(h); free(g); free(wn);
    return status;
}

int orc_gd_hbm(const double* A, idx m, idx n, const double* M, const double* b, const double* x0, double alpha,
               double beta, double eps, long maxit, const double* x_star, int track_true, double* x_out,
               orc_lsqr_report* rep, double* est_hist, double* err_hist, double* true_hist) {
    orc_op op = {m, n, 0, A, NULL, NULL, NULL};
    return gd_op(&op, M, b, x0, alpha, beta, eps, maxit, x_star, track_true, x_out, rep, est_hist, err_hist,
                 true_hist);
}

/* gradient.hpp:117-122 -- CscMatrix overload */
int orc_gd_hbm_csc(idx m, idx n, const idx* rows, const double* vals, const idx* colptr, const double* M,
                   const double* b, const double* x0, double alpha, double beta, double eps, long maxit,
                   const double* x_star, int track_true, double* x_out, orc_lsqr_report* rep,
                   double* est_hist, double* err_hist, double* true_hist) {
    orc_op op = {m, n, 1, NULL, rows, vals, colptr};
    return gd_op(&op, M, b, x0, alpha, beta, eps, maxit, x_star, track_true, x_out, rep, est_hist, err_hist,
                 true_hist);
}

/* ----------------------------------------------------- partitioning */

/* distsim.hpp:31-42 */
int orc_partition_rows(idx m, int p, idx* boundaries) {
    if (p < 1 || (idx)p > m) return E_INVALID_DIMS;
    const idx stride = m / p;
    for (int k = 0; k < p; ++k) boundaries[k] = stride * k;
    boundaries[p] = m;
    return OK;
}

/* ------------------------------------------------ problem generators */

/* problems.hpp:45-66 -- A = U diag(s) V^T, U/V = Q factors of Gaussians */
int orc_gen_dense(idx m, idx n, double cond, uint64_t seed, double* A) {
    if (cond < 1.0) return E_INVALID_DIMS;
    double* G = (double*)malloc(sizeof(double) * (size_t)(m * n));
    double* U = (double*)malloc(sizeof(double) * (size_t)(m * n));
    double* H = (double*)malloc(sizeof(double) * (size_t)(n * n));
    double* V = (double*)malloc(sizeof(double) * (size_t)(n * n));
    double* R = (double*)malloc(sizeof(double) * (size_t)(n * n));
    if (!G || !U || !H || !V || !R) return E_OOM;
    orc_normal_state g = {orc_rng_stream(seed, 0), 0, 0.0};
    for (idx i = 0; i < m * n; ++i) G[i] = orc_normal(&g);
    int st = orc_householder_qr(G, m, n, U, R, NULL);
    orc_normal_state g2 = {orc_rng_stream(seed, 1), 0, 0.0};
    for (idx i = 0; i < n * n; ++i) H[i] = orc_normal(&g2);
    if (st == OK) st = orc_householder_qr(H, n, n, V, R, NULL);
    if (st == OK) {
        for (idx j = 0; j < n; ++j) {
            const double s = (n == 1) ? 1.0 : pow(10.0, -log10(cond) * (double)j / (double)(n - 1));
            for (idx i = 0; i < m; ++i) U[j * m + i] *= s;
        }
        /* matmul(U, transpose(V)) -- dense_matrix.hpp:87-103 order */
        memset(A, 0, sizeof(double) * (size_t)(m * n));
        for (idx j = 0; j < n; ++j) {
            double* cj = A + j * m;
            for (idx k = 0; k < n; ++k) {
                const double bkj = V[k * n + j]; /* V^T(k, j) = V(j, k) */
                if (bkj == 0.0) continue;
                const double* ak = U + k * m;
                for (idx i = 0; i < m; ++i) cj[i] += ak[i] * bkj;
            }
        }
    }
    free(G); free(U); free(H); free(V); free(R);
    return st;
}

/* eigen_sym.hpp:85-120 -- Cholesky solve (harness for gen_rhs) */
static int chol_solve(const double* Gm, idx n, const double* b, double* y) {
    double* L = (double*)calloc((size_t)(n * n), sizeof(double));
    if (!L) return E_OOM;
    for (idx j = 0; j < n; ++j) {
        double s = Gm[j * n + j];
        for (idx k = 0; k < j; ++k) s -= L[k * n + j] * L[k * n + j];
        if (s <= 0.0) { free(L); return E_INVALID_DIMS; }
        L[j * n + j] = sqrt(s);
        for (idx i = j + 1; i < n; ++i) {
            double t = Gm[j * n + i];
            for (idx k = 0; k < j; ++k) t -= L[k * n + i] * L[k * n + j];
            L[j * n + i] = t / L[j * n + j];
        }
    }
    memcpy(y, b, sizeof(double) * (size_t)n);
    for (idx i = 0; i < n; ++i) {
        double s = y[i];
        for (idx k = 0; k < i; ++k) s -= L[k * n + i] * y[k];
        y[i] = s / L[i * n + i];
    }
    for (idx i = n - 1; i >= 0; --i) {
        double s = y[i];
        for (idx k = i + 1; k < n; ++k) s -= L[i * n + k] * y[k];
        y[i] = s / L[i * n + i];
    }
    free(L);
    return OK;
}

/* problems.hpp:137-167 -- b with ||b|| = 1 and ||b - A x*|| = rho */
int orc_gen_rhs(const double* A, idx m, idx n, double rho, uint64_t seed, double* b, double* x_star) {
    if (!(rho >= 0.0 && rho < 1.0)) return E_INVALID_DIMS;
    uint64_t st = orc_rng_stream(seed, 0);
    double* w = (double*)malloc(sizeof(double) * (size_t)n);
    double* p = (double*)malloc(sizeof(double) * (size_t)m);
    for (idx j = 0; j < n; ++j) w[j] = orc_uniform_sym(&st);
    orc_matvec(A, m, n, w, p);
    const double pn = norm2(p, m);
    if (pn == 0.0) { free(w); free(p); return E_RANK_DEFICIENT; }
    const double range_norm = sqrt(1.0 - rho * rho);
    for (idx j = 0; j < n; ++j) x_star[j] = w[j] * (range_norm / pn);
    for (idx i = 0; i < m; ++i) b[i] = p[i] * (range_norm / pn);
    int status = OK;
    if (rho != 0.0) {
        double* Gm = (double*)malloc(sizeof(double) * (size_t)(n * n));
        /* matmul_at_b(A, A) -- dense_matrix.hpp:106-122 */
        for (idx j = 0; j < n; ++j)
            for (idx i = 0; i < n; ++i) {
                double s = 0.0;
                for (idx k = 0; k < m; ++k) s += A[i * m + k] * A[j * m + k];
                Gm[j * n + i] = s;
            }
        double* z = (double*)malloc(sizeof(double) * (size_t)m);
        double* atz = (double*)malloc(sizeof(double) * (size_t)n);
        double* y = (double*)malloc(sizeof(double) * (size_t)n);
        for (idx i = 0; i < m; ++i) z[i] = orc_uniform_sym(&st);
        for (int pass = 0; pass < 2 && status == OK; ++pass) {
            orc_rmatvec(A, m, n, z, atz);
            status = chol_solve(Gm, n, atz, y);
            orc_matvec(A, m, n, y, p);
            for (idx i = 0; i < m; ++i) z[i] += -1.0 * p[i];
        }
        const double zn = norm2(z, m);
        if (status == OK && zn == 0.0) status = E_INVALID_DIMS;
        if (status == OK)
            for (idx i = 0; i < m; ++i) b[i] += (rho / zn) * z[i];
        free(Gm); free(z); free(atz); free(y);
    }
    free(w); free(p);
    return status;
}
