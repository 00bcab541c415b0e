// ref_shim.cpp -- extern "C" entry points over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY (checker + CPU baseline).  Compiled by
// oracle/Makefile directly from /root/reference/proj/include into
// oracle/_ref/libsketchlsq_ref.so; no reference source is copied into this
// repository.  Used by tests/ to pin the C restatement (oracle/sketchlsq_oracle.c)
// and to generate tests/golden/, and by bench.py as the `--impl reference`
// arm / cpu_baseline (kind "reference").
//
// Every function is a thin marshal: column-major double buffers in, the
// reference call, buffers out.  Exceptions become the status codes of
// include/slq_b200.h (errors.hpp:9-76).
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "sketchlsq/distsim.hpp"
#include "sketchlsq/embedding.hpp"
#include "sketchlsq/gradient.hpp"
#include "sketchlsq/matrix_market.hpp"
#include "sketchlsq/metrics.hpp"
#include "sketchlsq/lsqr.hpp"
#include "sketchlsq/preconditioner.hpp"
#include "sketchlsq/problems.hpp"
#include "sketchlsq/sketch.hpp"

using namespace sketchlsq;

namespace {

thread_local std::string g_err;

int map_exc() {
    try {
        throw;
    } catch (const InvalidSparsity& e) { g_err = e.what(); return 1; }
    catch (const InvalidDims& e) { g_err = e.what(); return 2; }
    catch (const DimensionMismatch& e) { g_err = e.what(); return 3; }
    catch (const RankDeficient& e) { g_err = e.what(); return 4; }
    catch (const SingularTriangular& e) { g_err = e.what(); return 5; }
    catch (const InvalidDistortion& e) { g_err = e.what(); return 11; }
    catch (const Divergence& e) { g_err = e.what(); return 12; }
    catch (const NegativeArgument& e) { g_err = e.what(); return 13; }
    catch (const InvalidResidual& e) { g_err = e.what(); return 14; }
    catch (const UnsupportedFormat& e) { g_err = e.what(); return 15; }
    catch (const std::exception& e) { g_err = e.what(); return 99; }
}

DenseMatrix wrap(const double* p, index_t r, index_t c) {
    return DenseMatrix(r, c, std::vector<double>(p, p + r * c));
}

void put(const DenseMatrix& M, double* out) {
    std::memcpy(out, M.data().data(), sizeof(double) * M.data().size());
}

double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// rng.hpp:29-64 -- k draws of next_u64 from Rng(seed) (stream < 0) or Rng(seed, stream)
void ref_rng_draws(uint64_t seed, int64_t stream, int64_t k, uint64_t* out) {
    if (stream < 0) {
        Rng r(seed);
        for (int64_t i = 0; i < k; ++i) out[i] = r.next_u64();
    } else {
        Rng r(seed, static_cast<uint64_t>(stream));
        for (int64_t i = 0; i < k; ++i) out[i] = r.next_u64();
    }
}

void ref_uniform_below(uint64_t seed, uint64_t stream, uint64_t bound, int64_t k, uint64_t* out) {
    Rng r(seed, stream);
    for (int64_t i = 0; i < k; ++i) out[i] = r.uniform_below(bound);
}

// sketch.hpp:178 generate_sparse_sign (col_begin == 0 && ncols == m) or
// sketch.hpp:149 sparse_sign_block for a general global column window.
int ref_generate_sparse_sign(int64_t d, int64_t col_begin, int64_t ncols, int64_t zeta,
                             uint64_t seed, int64_t* rows, double* vals, int64_t* colptr,
                             int64_t* stats2) {
    try {
        RejectionStats st;
        CscMatrix S;
        if (col_begin == 0) {
            S = generate_sparse_sign(d, ncols, zeta, seed, &st).matrix;
        } else {
            if (zeta > d || zeta < 1) throw InvalidSparsity("need 1 <= zeta <= d");
            S = detail::sparse_sign_block(d, zeta, seed, col_begin, col_begin + ncols, &st);
        }
        std::memcpy(rows, S.row_indices.data(), sizeof(int64_t) * S.row_indices.size());
        std::memcpy(vals, S.values.data(), sizeof(double) * S.values.size());
        std::memcpy(colptr, S.col_pointers.data(), sizeof(int64_t) * S.col_pointers.size());
        if (stats2) {
            stats2[0] = st.columns_resampled;
            stats2[1] = st.resample_rounds;
        }
        return 0;
    } catch (...) { return map_exc(); }
}

// sketch.hpp:105
int ref_rejection_sample_columns(int64_t d, int64_t m, int64_t zeta, uint64_t seed, int64_t* out,
                                 int64_t* stats2) {
    try {
        RejectionStats st;
        auto C = rejection_sample_columns(d, m, zeta, seed, &st);
        std::memcpy(out, C.data(), sizeof(int64_t) * C.size());
        if (stats2) {
            stats2[0] = st.columns_resampled;
            stats2[1] = st.resample_rounds;
        }
        return 0;
    } catch (...) { return map_exc(); }
}

// sketch.hpp:297 apply(SparseSignSketch, DenseMatrix) and sketch.hpp:304 sketch_vector
int ref_sketch_apply(int64_t d, int64_t m, int64_t zeta, uint64_t seed, const double* A, int64_t n,
                     const double* b, double* Y, double* Sb) {
    try {
        SparseSignSketch S = generate_sparse_sign(d, m, zeta, seed);
        if (A) put(apply(S, wrap(A, m, n)), Y);
        if (b) {
            Vector sb = sketch_vector(S, Vector(b, b + m));
            std::memcpy(Sb, sb.data(), sizeof(double) * sb.size());
        }
        return 0;
    } catch (...) { return map_exc(); }
}

// sketch.hpp:298 apply(SparseSignSketch, CscMatrix) -> csc_matrix.hpp:123
int ref_sketch_apply_csc(int64_t d, int64_t m, int64_t zeta, uint64_t seed, int64_t n,
                         const int64_t* arows, const double* avals, const int64_t* acolptr,
                         double* Y) {
    try {
        SparseSignSketch S = generate_sparse_sign(d, m, zeta, seed);
        CscMatrix A(m, n);
        const int64_t nnz = acolptr[n];
        A.row_indices.assign(arows, arows + nnz);
        A.values.assign(avals, avals + nnz);
        A.col_pointers.assign(acolptr, acolptr + n + 1);
        put(apply(S, A), Y);
        return 0;
    } catch (...) { return map_exc(); }
}

// qr.hpp:21
int ref_householder_qr(const double* Y, int64_t d, int64_t n, double* Q, double* R) {
    try {
        QrResult qr = householder_qr(wrap(Y, d, n));
        if (Q) put(qr.Q, Q);
        put(qr.R, R);
        return 0;
    } catch (...) { return map_exc(); }
}

// triangular.hpp:14
int ref_tri_inverse(const double* R, int64_t n, double* M) {
    try {
        put(tri_inverse(wrap(R, n, n)), M);
        return 0;
    } catch (...) { return map_exc(); }
}

// preconditioner.hpp:35 + preconditioner.hpp:48
int ref_build_preconditioner(const double* Y, int64_t d, int64_t n, const double* Sb, double* M,
                             double* Q, double* x0, double* build_time) {
    try {
        Preconditioner P = build_preconditioner(wrap(Y, d, n));
        put(P.M, M);
        if (Q) put(P.Q, Q);
        if (build_time) *build_time = P.build_time;
        if (Sb && x0) {
            Vector g = initial_guess(P, Vector(Sb, Sb + d));
            std::memcpy(x0, g.data(), sizeof(double) * g.size());
        }
        return 0;
    } catch (...) { return map_exc(); }
}

struct ref_report {
    int64_t iterations;
    int32_t termination;
    int32_t pad;
    int64_t sync_count, broadcasts, init_reductions, init_broadcasts;
    double wall_time;
    int64_t n_estimate, n_true, n_err;
};

static void fill(const SolveReport& r, ref_report* out, double* est, double* err, double* tru) {
    out->iterations = r.iterations;
    out->termination = static_cast<int32_t>(r.termination);
    out->sync_count = r.sync_count;
    out->broadcasts = r.broadcasts;
    out->init_reductions = r.init_reductions;
    out->init_broadcasts = r.init_broadcasts;
    out->wall_time = r.wall_time;
    out->n_estimate = static_cast<int64_t>(r.residual_estimate.size());
    out->n_true = static_cast<int64_t>(r.residual_true.size());
    out->n_err = static_cast<int64_t>(r.iterates_error.size());
    if (est) std::memcpy(est, r.residual_estimate.data(), sizeof(double) * r.residual_estimate.size());
    if (err) std::memcpy(err, r.iterates_error.data(), sizeof(double) * r.iterates_error.size());
    if (tru) std::memcpy(tru, r.residual_true.data(), sizeof(double) * r.residual_true.size());
}

// lsqr.hpp:193-207 (serial overloads); workers > 0 selects the reference's
// distributed backend: WorkerPool + distribute + dist_operator (distsim.hpp:79,215,453).
int ref_lsqr(const double* A, int64_t m, int64_t n, const double* M, const double* b,
             const double* x0, double eps, int64_t maxit, int one_sync, const double* x_star,
             int track_true, int workers, double* x_out, ref_report* rep, double* est,
             double* err, double* tru) {
    try {
        DenseMatrix Am = wrap(A, m, n);
        Preconditioner P;
        P.M = wrap(M, n, n);
        P.Q = DenseMatrix(0, 0);
        Vector bv(b, b + m), xv(x0, x0 + n), xs;
        SolveOptions o;
        o.eps = eps;
        o.maxit = maxit;
        if (x_star) {
            xs.assign(x_star, x_star + n);
            o.x_star = &xs;
        }
        o.track_true_residual = track_true != 0;
        std::pair<Vector, SolveReport> res;
        if (workers <= 0) {
            res = one_sync ? lsqr_one_sync(Am, P, bv, xv, o) : lsqr(Am, P, bv, xv, o);
        } else {
            WorkerPool pool(workers);
            auto dA = distribute(Am, pool);
            DistributedVector db = distribute(bv, pool);
            auto op = dist_operator(dA);
            res = one_sync ? lsqr_one_sync(op, P, db, xv, o) : lsqr(op, P, db, xv, o);
        }
        std::memcpy(x_out, res.first.data(), sizeof(double) * n);
        fill(res.second, rep, est, err, tru);
        return 0;
    } catch (...) { return map_exc(); }
}

// lsqr.hpp:198-202 / :208-212 (CscMatrix overloads); workers > 0: DistOperator<CscMatrix>
int ref_lsqr_csc(int64_t m, int64_t n, const int64_t* rows, const double* vals, const int64_t* colptr,
                 const double* M, const double* b, const double* x0, double eps, int64_t maxit, int one_sync,
                 const double* x_star, int track_true, int workers, double* x_out, ref_report* rep, double* est,
                 double* err, double* tru) {
    try {
        CscMatrix A(m, n);
        const int64_t nnz = colptr[n];
        A.row_indices.assign(rows, rows + nnz);
        A.values.assign(vals, vals + nnz);
        A.col_pointers.assign(colptr, colptr + n + 1);
        Preconditioner P;
        P.M = wrap(M, n, n);
        Vector bv(b, b + m), xv(x0, x0 + n), xs;
        SolveOptions o;
        o.eps = eps;
        o.maxit = maxit;
        if (x_star) {
            xs.assign(x_star, x_star + n);
            o.x_star = &xs;
        }
        o.track_true_residual = track_true != 0;
        std::pair<Vector, SolveReport> res;
        if (workers <= 0) {
            res = one_sync ? lsqr_one_sync(A, P, bv, xv, o) : lsqr(A, P, bv, xv, o);
        } else {
            WorkerPool pool(workers);
            auto dA = distribute(A, pool);
            DistributedVector db = distribute(bv, pool);
            auto op = dist_operator(dA);
            res = one_sync ? lsqr_one_sync(op, P, db, xv, o) : lsqr(op, P, db, xv, o);
        }
        std::memcpy(x_out, res.first.data(), sizeof(double) * n);
        fill(res.second, rep, est, err, tru);
        return 0;
    } catch (...) { return map_exc(); }
}

// gradient.hpp:27-48 hbm_params / gd_params (out: alpha, beta)
int ref_gradient_params(double eta, int hbm, double* out) {
    try {
        const GradientParams g = hbm ? hbm_params(eta) : gd_params(eta);
        out[0] = g.alpha;
        out[1] = g.beta;
        return 0;
    } catch (...) { return map_exc(); }
}

// gradient.hpp:56-126 gradient_descent_hbm, dense (csc == 0: A column-major m x n)
// or CSC (rows / vals / colptr), serial operator or WorkerPool(workers).
int ref_gradient_descent_hbm(int csc, const double* A, int64_t m, int64_t n, const int64_t* rows, const double* vals,
                             const int64_t* colptr, const double* M, const double* b, const double* x0, double alpha,
                             double beta, double eps, int64_t maxit, const double* x_star, int track_true, int workers,
                             double* x_out, ref_report* rep, double* est, double* err, double* tru) {
    try {
        Preconditioner P;
        P.M = wrap(M, n, n);
        Vector bv(b, b + m), xv(x0, x0 + n), xs;
        SolveOptions o;
        o.eps = eps;
        o.maxit = maxit;
        if (x_star) {
            xs.assign(x_star, x_star + n);
            o.x_star = &xs;
        }
        o.track_true_residual = track_true != 0;
        const GradientParams gp{alpha, beta, 0.0};
        std::pair<Vector, SolveReport> res;
        auto run = [&](const auto& Am) {
            if (workers <= 0) return gradient_descent_hbm(Am, P, bv, xv, gp, o);
            WorkerPool pool(workers);
            auto dA = distribute(Am, pool);
            DistributedVector db = distribute(bv, pool);
            auto op = dist_operator(dA);
            return gradient_descent_hbm(op, P, db, xv, gp, o);
        };
        if (csc) {
            CscMatrix Ac(m, n);
            const int64_t nnz = colptr[n];
            Ac.row_indices.assign(rows, rows + nnz);
            Ac.values.assign(vals, vals + nnz);
            Ac.col_pointers.assign(colptr, colptr + n + 1);
            res = run(Ac);
        } else {
            res = run(wrap(A, m, n));
        }
        std::memcpy(x_out, res.first.data(), sizeof(double) * n);
        fill(res.second, rep, est, err, tru);
        return 0;
    } catch (...) { return map_exc(); }
}

// embedding.hpp:20-98 -- out: [rate, kappa, iterations_for, lambert_w(x), balance_real, plan.d,
// plan.predicted_iters, plan.predicted_kappa]
int ref_embedding(int64_t m, int64_t n, int64_t d, double eps, double x, double* out) {
    try {
        const RateEstimate r = estimate_rate(n, d);
        out[0] = r.rate_per_iter;
        out[1] = r.kappa;
        out[2] = static_cast<double>(iterations_for(eps, n, d));
        out[3] = lambert_w(x);
        out[4] = balance_dimension_real(m, n, eps);
        const DimensionPlan p = select_embedding_dim(m, n, eps);
        out[5] = static_cast<double>(p.d);
        out[6] = static_cast<double>(p.predicted_iters);
        out[7] = p.predicted_kappa;
        return 0;
    } catch (...) { return map_exc(); }
}

// metrics.hpp:66-78 distortion of the sparse sign sketch (d, zeta, seed) on
// range(U) [+ span(b)]: out = [eta, sigma_min, sigma_max]
int ref_distortion(int64_t d, int64_t zeta, uint64_t seed, const double* U, int64_t m, int64_t n, const double* b,
                   double* out) {
    try {
        SparseSignSketch S = generate_sparse_sign(d, m, zeta, seed);
        Vector bv;
        if (b) bv.assign(b, b + m);
        const DistortionReport r = distortion(S, wrap(U, m, n), b ? &bv : nullptr);
        out[0] = r.eta;
        out[1] = r.sigma_min;
        out[2] = r.sigma_max;
        return 0;
    } catch (...) { return map_exc(); }
}

// metrics.hpp:122-150 scalar helpers: out = [mp_pdf(x, ratio), cond_bound(eta), fwd_err(res_hat, res_star)]
int ref_metric_scalars(double x, double ratio, double eta, double res_hat, double res_star, double* out) {
    try {
        out[0] = marchenko_pastur_pdf(x, ratio);
        out[1] = cond_bound(eta);
        out[2] = forward_error_from_residuals(res_hat, res_star);
        return 0;
    } catch (...) { return map_exc(); }
}

// matrix_market.hpp:140-166 writers
int ref_mm_write_csc(const char* path, int64_t m, int64_t n, const int64_t* rows, const double* vals,
                     const int64_t* colptr) {
    try {
        CscMatrix A(m, n);
        const int64_t nnz = colptr[n];
        A.row_indices.assign(rows, rows + nnz);
        A.values.assign(vals, vals + nnz);
        A.col_pointers.assign(colptr, colptr + n + 1);
        mm::write_csc(path, A);
        return 0;
    } catch (...) { return map_exc(); }
}
int ref_mm_write_dense(const char* path, const double* A, int64_t m, int64_t n) {
    try {
        mm::write_dense(path, wrap(A, m, n));
        return 0;
    } catch (...) { return map_exc(); }
}
// matrix_market.hpp:64-128 readers: call with out buffers NULL to get the sizes (dims[0..2] = rows, cols, nnz)
int ref_mm_read_csc(const char* path, int64_t* dims, int64_t* rows, double* vals, int64_t* colptr) {
    try {
        CscMatrix A = mm::read_csc(path);
        dims[0] = A.rows;
        dims[1] = A.cols;
        dims[2] = A.nnz();
        if (rows) {
            std::memcpy(rows, A.row_indices.data(), sizeof(int64_t) * A.row_indices.size());
            std::memcpy(vals, A.values.data(), sizeof(double) * A.values.size());
            std::memcpy(colptr, A.col_pointers.data(), sizeof(int64_t) * A.col_pointers.size());
        }
        return 0;
    } catch (...) { return map_exc(); }
}
int ref_mm_read_dense(const char* path, int64_t* dims, double* out) {
    try {
        DenseMatrix A = mm::read_dense(path);
        dims[0] = A.rows();
        dims[1] = A.cols();
        if (out) put(A, out);
        return 0;
    } catch (...) { return map_exc(); }
}

// distsim.hpp:31
int ref_partition_rows(int64_t m, int p, int64_t* boundaries) {
    try {
        RowPartition part = partition_rows(m, p);
        std::memcpy(boundaries, part.boundaries.data(), sizeof(int64_t) * part.boundaries.size());
        return 0;
    } catch (...) { return map_exc(); }
}

// distsim.hpp:346 + distsim.hpp:364 -- generation across p workers, assembled
int ref_dist_generate_sparse_sign(int64_t d, int64_t m, int64_t zeta, uint64_t seed, int p,
                                  int64_t* rows, double* vals, int64_t* colptr) {
    try {
        WorkerPool pool(p);
        RowPartition part = partition_rows(m, p);
        CscMatrix S = assemble(dist_generate_sparse_sign(d, zeta, seed, part, pool));
        std::memcpy(rows, S.row_indices.data(), sizeof(int64_t) * S.row_indices.size());
        std::memcpy(vals, S.values.data(), sizeof(double) * S.values.size());
        std::memcpy(colptr, S.col_pointers.data(), sizeof(int64_t) * S.col_pointers.size());
        return 0;
    } catch (...) { return map_exc(); }
}

// distsim.hpp:383 / :399 -- partitioned S A and S b with tree reduction
int ref_dist_sketch_apply(int64_t d, int64_t m, int64_t zeta, uint64_t seed, const double* A,
                          int64_t n, const double* b, int p, double* Y, double* Sb) {
    try {
        WorkerPool pool(p);
        auto dA = distribute(wrap(A, m, n), pool);
        DistSparseSketch S = dist_generate_sparse_sign(d, zeta, seed, dA.partition, pool);
        put(dist_sketch_apply(S, dA), Y);
        if (b) {
            Vector sb = dist_sketch_apply(S, distribute(Vector(b, b + m), pool));
            std::memcpy(Sb, sb.data(), sizeof(double) * sb.size());
        }
        return 0;
    } catch (...) { return map_exc(); }
}

// problems.hpp:45 / :137 -- harness generators
int ref_gen_dense(int64_t m, int64_t n, double cond, uint64_t seed, double* A) {
    try {
        put(gen_dense(m, n, cond, seed), A);
        return 0;
    } catch (...) { return map_exc(); }
}

int ref_gen_rhs(const double* A, int64_t m, int64_t n, double rho, uint64_t seed, double* b,
                double* x_star) {
    try {
        RhsResult r = gen_rhs(wrap(A, m, n), rho, seed);
        std::memcpy(b, r.b.data(), sizeof(double) * m);
        std::memcpy(x_star, r.x_star.data(), sizeof(double) * n);
        return 0;
    } catch (...) { return map_exc(); }
}

// Timed end-to-end reference pipeline (the CPU baseline of bench.py).
// workers == 0: serial path (generate_sparse_sign, apply, sketch_vector,
// build_preconditioner, initial_guess, lsqr_one_sync over SerialOperator).
// workers  > 0: the reference's own parallel backend on `workers` threads
// (distribute, dist_generate_sparse_sign, dist_sketch_apply, serial QR,
// lsqr_one_sync over DistOperator).  LSQR runs with eps / maxit as given.
// times[0..5] = generate, apply(S A and S b), precond build, x0, lsqr, distribute.
int ref_solve_timed(const double* A, int64_t m, int64_t n, const double* b, int64_t d,
                    int64_t zeta, uint64_t seed, double eps, int64_t maxit, int workers,
                    double* x_out, ref_report* rep, double* times) {
    try {
        DenseMatrix Am = wrap(A, m, n);
        Vector bv(b, b + m);
        SolveOptions o;
        o.eps = eps;
        o.maxit = maxit;
        if (workers <= 0) {
            double t0 = now();
            SparseSignSketch S = generate_sparse_sign(d, m, zeta, seed);
            double t1 = now();
            DenseMatrix Y = apply(S, Am);
            Vector sb = sketch_vector(S, bv);
            double t2 = now();
            Preconditioner P = build_preconditioner(Y);
            double t3 = now();
            Vector x0 = initial_guess(P, sb);
            double t4 = now();
            auto res = lsqr_one_sync(Am, P, bv, x0, o);
            double t5 = now();
            std::memcpy(x_out, res.first.data(), sizeof(double) * n);
            fill(res.second, rep, nullptr, nullptr, nullptr);
            double tt[6] = {t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4, 0.0};
            std::memcpy(times, tt, sizeof(tt));
        } else {
            WorkerPool pool(workers);
            double tA = now();
            auto dA = distribute(Am, pool);
            DistributedVector db = distribute(bv, pool);
            double t0 = now();
            DistSparseSketch S = dist_generate_sparse_sign(d, zeta, seed, dA.partition, pool);
            double t1 = now();
            DenseMatrix Y = dist_sketch_apply(S, dA);
            Vector sb = dist_sketch_apply(S, db);
            double t2 = now();
            Preconditioner P = build_preconditioner(Y);
            double t3 = now();
            Vector x0 = initial_guess(P, sb);
            double t4 = now();
            auto op = dist_operator(dA);
            auto res = lsqr_one_sync(op, P, db, x0, o);
            double t5 = now();
            std::memcpy(x_out, res.first.data(), sizeof(double) * n);
            fill(res.second, rep, nullptr, nullptr, nullptr);
            double tt[6] = {t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4, t0 - tA};
            std::memcpy(times, tt, sizeof(tt));
        }
        return 0;
    } catch (...) { return map_exc(); }
}

}  // extern "C"
