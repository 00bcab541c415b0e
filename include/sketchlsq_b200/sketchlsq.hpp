// sketchlsq_b200/sketchlsq.hpp -- header-only C++ drop-in for the hot path of
// the reference library `sketchlsq` (/root/reference/proj/include/sketchlsq),
// implemented on top of the C-ABI in slq_b200.h (link -lslq_b200).
//
// Replace
//     #include "sketchlsq/sketch.hpp"
//     #include "sketchlsq/preconditioner.hpp"
//     #include "sketchlsq/lsqr.hpp"
// with
//     #include "sketchlsq_b200/sketchlsq.hpp"
// and the same calls (same names, argument meaning, value semantics and
// exception types) run on the B200.  Types mirror dense_matrix.hpp:18-50,
// csc_matrix.hpp:19-60, sketch.hpp:20-68, qr.hpp:15-18,
// preconditioner.hpp:15-30, lsqr.hpp:14-22, solve_report.hpp:11-49,
// gradient.hpp:20-126, distsim.hpp:21-42.  Define SKETCHLSQ_B200_NAMESPACE to place the mirror in
// another namespace (default: sketchlsq, i.e. a true drop-in).
#pragma once

#include <cmath>
#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "slq_b200.h"

#ifndef SKETCHLSQ_B200_NAMESPACE
#define SKETCHLSQ_B200_NAMESPACE sketchlsq
#endif

namespace SKETCHLSQ_B200_NAMESPACE {

using index_t = std::int64_t;
using Vector = std::vector<double>;

// errors.hpp:9-76
struct Error : std::runtime_error {
    explicit Error(const std::string& w) : std::runtime_error(w) {}
};
struct RankDeficient : Error { using Error::Error; };
struct SingularTriangular : Error { using Error::Error; };
struct DimensionMismatch : Error { using Error::Error; };
struct InvalidSparsity : Error { using Error::Error; };
struct InvalidDims : Error { using Error::Error; };
struct InvalidDistortion : Error { using Error::Error; };
struct Divergence : Error { using Error::Error; };
struct DeviceError : Error { using Error::Error; };

namespace b200 {

inline void check(int st) {
    if (st == SLQ_OK) return;
    const std::string msg = slq_last_error();
    switch (st) {
        case SLQ_INVALID_SPARSITY: throw InvalidSparsity(msg);
        case SLQ_INVALID_DIMS: throw InvalidDims(msg);
        case SLQ_DIMENSION_MISMATCH: throw DimensionMismatch(msg);
        case SLQ_RANK_DEFICIENT: throw RankDeficient(msg);
        case SLQ_SINGULAR_TRIANGULAR: throw SingularTriangular(msg);
        case SLQ_INVALID_DISTORTION: throw InvalidDistortion(msg);
        case SLQ_DIVERGENCE: throw Divergence(msg);
        default: throw DeviceError(msg);
    }
}

// One context per thread on device 0 unless set_device() is called first.
struct Ctx {
    slq_ctx* h = nullptr;
    int device = 0;
    ~Ctx() {
        if (h) slq_ctx_destroy(h);
    }
};
inline Ctx& tls() {
    thread_local Ctx c;
    return c;
}
inline void set_device(int device) {
    Ctx& c = tls();
    if (c.h && c.device != device) {
        slq_ctx_destroy(c.h);
        c.h = nullptr;
    }
    c.device = device;
}
inline slq_ctx* ctx() {
    Ctx& c = tls();
    if (!c.h) check(slq_ctx_create(c.device, &c.h));
    return c.h;
}

}  // namespace b200

// dense_matrix.hpp:18-50 -- column-major
class DenseMatrix {
public:
    DenseMatrix() = default;
    DenseMatrix(index_t r, index_t c) : rows_(r), cols_(c), data_(static_cast<std::size_t>(r * c), 0.0) {}
    DenseMatrix(index_t r, index_t c, std::vector<double> d) : rows_(r), cols_(c), data_(std::move(d)) {}
    index_t rows() const { return rows_; }
    index_t cols() const { return cols_; }
    double& operator()(index_t i, index_t j) { return data_[static_cast<std::size_t>(j * rows_ + i)]; }
    double operator()(index_t i, index_t j) const { return data_[static_cast<std::size_t>(j * rows_ + i)]; }
    double* col(index_t j) { return data_.data() + j * rows_; }
    const double* col(index_t j) const { return data_.data() + j * rows_; }
    std::vector<double>& data() { return data_; }
    const std::vector<double>& data() const { return data_; }
    static DenseMatrix identity(index_t n) {
        DenseMatrix I(n, n);
        for (index_t i = 0; i < n; ++i) I(i, i) = 1.0;
        return I;
    }

private:
    index_t rows_ = 0, cols_ = 0;
    std::vector<double> data_;
};

// csc_matrix.hpp:19-60
struct CscMatrix {
    index_t rows = 0, cols = 0;
    std::vector<double> values;
    std::vector<index_t> row_indices;
    std::vector<index_t> col_pointers;
    CscMatrix() : col_pointers{0} {}
    CscMatrix(index_t r, index_t c) : rows(r), cols(c), col_pointers(static_cast<std::size_t>(c) + 1, 0) {}
    index_t nnz() const { return static_cast<index_t>(values.size()); }
};

// sketch.hpp:20-68
struct SketchParams {
    index_t d = 0;
    index_t zeta = 8;
    std::uint64_t seed = 0;
    void validate(index_t m, index_t n) const {
        if (!(n < d && d <= m)) throw InvalidDims("SketchParams: need n < d <= m");
        if (!(1 <= zeta && zeta <= d)) throw InvalidSparsity("SketchParams: need 1 <= zeta <= d");
    }
};
struct SparseSignSketch {
    CscMatrix matrix;
    index_t zeta = 0;
    std::uint64_t seed = 0;
};
struct RejectionStats {
    index_t columns_resampled = 0;
    index_t resample_rounds = 0;
};

namespace detail {
// sketch.hpp:149-173
inline CscMatrix sparse_sign_block(index_t d, index_t zeta, std::uint64_t seed, index_t col_begin, index_t col_end,
                                   RejectionStats* stats = nullptr) {
    const index_t mb = col_end - col_begin;
    CscMatrix S(d, mb);
    S.values.resize(static_cast<std::size_t>(mb * zeta));
    S.row_indices.resize(static_cast<std::size_t>(mb * zeta));
    slq_rejection_stats st{0, 0};
    b200::check(slq_generate_sparse_sign(b200::ctx(), d, col_begin, mb, zeta, seed, S.row_indices.data(),
                                         S.values.data(), S.col_pointers.data(), &st));
    if (stats) {
        stats->columns_resampled += st.columns_resampled;
        stats->resample_rounds += st.resample_rounds;
    }
    return S;
}
}  // namespace detail

// sketch.hpp:178-194
inline SparseSignSketch generate_sparse_sign(index_t d, index_t m, index_t zeta, std::uint64_t seed,
                                             RejectionStats* stats = nullptr) {
    if (zeta > d || zeta < 1) throw InvalidSparsity("generate_sparse_sign: need 1 <= zeta <= d");
    return SparseSignSketch{detail::sparse_sign_block(d, zeta, seed, 0, m, stats), zeta, seed};
}
inline SparseSignSketch generate_sparse_sign(const SketchParams& p, index_t m, RejectionStats* stats = nullptr) {
    return generate_sparse_sign(p.d, m, p.zeta, p.seed, stats);
}

// sketch.hpp:105-124
inline std::vector<index_t> rejection_sample_columns(index_t d, index_t m, index_t zeta, std::uint64_t seed,
                                                     RejectionStats* stats = nullptr) {
    std::vector<index_t> C(static_cast<std::size_t>(m * zeta));
    slq_rejection_stats st{0, 0};
    b200::check(slq_rejection_sample_columns(b200::ctx(), d, m, zeta, seed, C.data(), &st));
    if (stats) {
        stats->columns_resampled += st.columns_resampled;
        stats->resample_rounds += st.resample_rounds;
    }
    return C;
}

// sketch.hpp:297 -> csc_matrix.hpp:103-120 (bit-identical accumulation order)
inline DenseMatrix apply(const SparseSignSketch& s, const DenseMatrix& A) {
    if (s.matrix.cols != A.rows()) throw DimensionMismatch("spmm: inner dimensions disagree");
    DenseMatrix Y(s.matrix.rows, A.cols());
    b200::check(slq_spmm_csc_dense(b200::ctx(), s.matrix.rows, s.matrix.cols, s.matrix.row_indices.data(),
                                   s.matrix.values.data(), s.matrix.col_pointers.data(), A.data().data(), A.cols(),
                                   A.rows() > 0 ? A.rows() : 1, Y.data().data()));
    return Y;
}
// sketch.hpp:304 -> csc_matrix.hpp:71-82
inline Vector sketch_vector(const SparseSignSketch& s, const Vector& b) {
    if (static_cast<index_t>(b.size()) != s.matrix.cols) throw DimensionMismatch("matvec(csc): length mismatch");
    DenseMatrix B(static_cast<index_t>(b.size()), 1, b);
    DenseMatrix Y = apply(s, B);
    return Vector(Y.data().begin(), Y.data().end());
}

// qr.hpp:15-89
struct QrResult {
    DenseMatrix Q;
    DenseMatrix R;
};
inline QrResult householder_qr(const DenseMatrix& Y) {
    const index_t d = Y.rows(), n = Y.cols();
    if (d < n) throw DimensionMismatch("householder_qr: need rows >= cols");
    QrResult out{DenseMatrix(d, n), DenseMatrix(n, n)};
    b200::check(slq_householder_qr(b200::ctx(), Y.data().data(), d, n, d > 0 ? d : 1, out.Q.data().data(),
                                   out.R.data().data()));
    return out;
}

// triangular.hpp:14-61
inline DenseMatrix tri_inverse(const DenseMatrix& R) {
    const index_t n = R.rows();
    if (R.cols() != n) throw DimensionMismatch("tri_inverse: matrix not square");
    DenseMatrix M(n, n);
    b200::check(slq_tri_inverse(b200::ctx(), R.data().data(), n, M.data().data()));
    return M;
}
inline Vector tri_upper_matvec(const DenseMatrix& R, const Vector& x) {
    if (static_cast<index_t>(x.size()) != R.rows()) throw DimensionMismatch("tri_upper_matvec");
    Vector y(x.size());
    b200::check(slq_tri_upper_matvec(b200::ctx(), R.data().data(), R.rows(), x.data(), y.data(), 0));
    return y;
}
inline Vector tri_upper_rmatvec(const DenseMatrix& R, const Vector& x) {
    if (static_cast<index_t>(x.size()) != R.rows()) throw DimensionMismatch("tri_upper_rmatvec");
    Vector y(x.size());
    b200::check(slq_tri_upper_matvec(b200::ctx(), R.data().data(), R.rows(), x.data(), y.data(), 1));
    return y;
}

// preconditioner.hpp:15-56
struct Preconditioner {
    DenseMatrix M;
    DenseMatrix Q;
    double build_time = 0.0;
    index_t d = 0;
    index_t n() const { return M.rows(); }
    static Preconditioner identity(index_t n) {
        Preconditioner P;
        P.M = DenseMatrix::identity(n);
        P.Q = DenseMatrix::identity(n);
        P.d = n;
        return P;
    }
};
inline Preconditioner build_preconditioner(const DenseMatrix& Y) {
    const index_t d = Y.rows(), n = Y.cols();
    if (d < n) throw DimensionMismatch("householder_qr: need rows >= cols");
    Preconditioner P;
    P.M = DenseMatrix(n, n);
    P.Q = DenseMatrix(d, n);
    P.d = d;
    b200::check(slq_build_preconditioner(b200::ctx(), Y.data().data(), d, n, d > 0 ? d : 1, nullptr,
                                         P.M.data().data(), P.Q.data().data(), nullptr, &P.build_time));
    return P;
}
inline Vector initial_guess(const Preconditioner& P, const Vector& Sb) {
    if (static_cast<index_t>(Sb.size()) != P.Q.rows())
        throw DimensionMismatch("initial_guess: Sb length does not match sketch dimension");
    Vector x0(static_cast<std::size_t>(P.n()));
    b200::check(slq_initial_guess(b200::ctx(), P.M.data().data(), P.Q.data().data(), P.Q.rows(), P.n(), Sb.data(),
                                  x0.data()));
    return x0;
}
inline Vector apply_M(const Preconditioner& P, const Vector& v) { return tri_upper_matvec(P.M, v); }
inline Vector apply_Mt(const Preconditioner& P, const Vector& v) { return tri_upper_rmatvec(P.M, v); }

// solve_report.hpp:11-49
enum class Termination { Tolerance, MaxIter, Breakdown };
inline std::string to_string(Termination t) {
    switch (t) {
        case Termination::Tolerance: return "tolerance";
        case Termination::MaxIter: return "maxiter";
        case Termination::Breakdown: return "breakdown";
    }
    return "unknown";
}
struct SolveReport {
    std::vector<double> iterates_error, residual_estimate, residual_true;
    long iterations = 0;
    Termination termination = Termination::MaxIter;
    long sync_count = 0, broadcasts = 0, init_reductions = 0, init_broadcasts = 0;
    double wall_time = 0.0;
    double reductions_per_iteration() const {
        return iterations > 0 ? static_cast<double>(sync_count - init_reductions) / iterations : 0.0;
    }
    double broadcasts_per_iteration() const {
        return iterations > 0 ? static_cast<double>(broadcasts - init_broadcasts) / iterations : 0.0;
    }
};

// lsqr.hpp:14-22
struct SolveOptions {
    double eps = 1e-10;
    long maxit = 100;
    const Vector* x_star = nullptr;
    bool track_true_residual = false;
    std::function<void(long t, double u_norm, double v_norm)> on_bidiag;
};

namespace detail {
inline void bidiag_trampoline(void* user, int64_t t, double un, double vn) {
    (*static_cast<std::function<void(long, double, double)>*>(user))(static_cast<long>(t), un, vn);
}
inline std::pair<Vector, SolveReport> lsqr_device(const DenseMatrix& A, const Preconditioner& P, const Vector& b,
                                                  const Vector& x0, const SolveOptions& o, bool one_sync) {
    const index_t m = A.rows(), n = A.cols();
    if (static_cast<index_t>(b.size()) != m) throw DimensionMismatch("rmatvec: length mismatch");
    if (static_cast<index_t>(x0.size()) != n) throw DimensionMismatch("matvec: length mismatch");
    if (P.M.rows() != n) throw DimensionMismatch("tri_upper_matvec");
    slq_dense* dA = nullptr;
    b200::check(slq_dense_upload(b200::ctx(), A.data().data(), m, n, m > 0 ? m : 1, b.data(), 0, &dA));
    slq_solve_opts so;
    slq_solve_opts_default(&so);
    so.eps = o.eps;
    so.maxit = o.maxit;
    so.x_star = o.x_star ? o.x_star->data() : nullptr;
    so.track_true_residual = o.track_true_residual ? 1 : 0;
    so.one_sync = one_sync ? 1 : 0;
    std::function<void(long, double, double)> hook = o.on_bidiag;
    if (hook) {
        so.on_bidiag = &bidiag_trampoline;
        so.on_bidiag_user = &hook;
    }
    const std::size_t cap = static_cast<std::size_t>(o.maxit > 0 ? o.maxit : 0) + 2;
    Vector x(static_cast<std::size_t>(n)), est(cap), err(cap), tru(cap);
    slq_report r;
    const int st = slq_lsqr(b200::ctx(), dA, P.M.data().data(), nullptr, x0.data(), &so, x.data(), &r, est.data(),
                            err.data(), tru.data());
    slq_dense_free(dA);
    b200::check(st);
    SolveReport rep;
    rep.residual_estimate.assign(est.begin(), est.begin() + r.n_estimate);
    rep.iterates_error.assign(err.begin(), err.begin() + r.n_err);
    rep.residual_true.assign(tru.begin(), tru.begin() + r.n_true);
    rep.iterations = static_cast<long>(r.iterations);
    rep.termination = static_cast<Termination>(r.termination);
    rep.sync_count = static_cast<long>(r.sync_count);
    rep.broadcasts = static_cast<long>(r.broadcasts);
    rep.init_reductions = static_cast<long>(r.init_reductions);
    rep.init_broadcasts = static_cast<long>(r.init_broadcasts);
    rep.wall_time = r.wall_time;
    return {std::move(x), std::move(rep)};
}
}  // namespace detail

// lsqr.hpp:193-212 (DenseMatrix overloads)
inline std::pair<Vector, SolveReport> lsqr(const DenseMatrix& A, const Preconditioner& P, const Vector& b,
                                           const Vector& x0, const SolveOptions& opts = {}) {
    return detail::lsqr_device(A, P, b, x0, opts, false);
}
inline std::pair<Vector, SolveReport> lsqr_one_sync(const DenseMatrix& A, const Preconditioner& P, const Vector& b,
                                                    const Vector& x0, const SolveOptions& opts = {}) {
    return detail::lsqr_device(A, P, b, x0, opts, true);
}

// gradient.hpp:20-48
struct GradientParams {
    double alpha = 1.0;
    double beta = 0.0;
    double eta_hat = 0.0;
};
inline GradientParams hbm_params(double eta_hat) {
    slq_gradient_params g;
    b200::check(slq_hbm_params(eta_hat, &g));
    return GradientParams{g.alpha, g.beta, g.eta_hat};
}
inline GradientParams gd_params(double eta_hat) {
    slq_gradient_params g;
    b200::check(slq_gd_params(eta_hat, &g));
    return GradientParams{g.alpha, g.beta, g.eta_hat};
}
inline double gd_step_size(double eta_hat) { return gd_params(eta_hat).alpha; }

// gradient.hpp:56-126 (DenseMatrix overload): one device pass over A per iteration
inline std::pair<Vector, SolveReport> gradient_descent_hbm(const DenseMatrix& A, const Preconditioner& P,
                                                           const Vector& b, const Vector& x0,
                                                           const GradientParams& params,
                                                           const SolveOptions& o = {}) {
    const index_t m = A.rows(), n = A.cols();
    if (static_cast<index_t>(b.size()) != m) throw DimensionMismatch("rmatvec: length mismatch");
    if (static_cast<index_t>(x0.size()) != n) throw DimensionMismatch("matvec: length mismatch");
    if (P.M.rows() != n) throw DimensionMismatch("tri_upper_matvec");
    slq_dense* dA = nullptr;
    b200::check(slq_dense_upload(b200::ctx(), A.data().data(), m, n, m > 0 ? m : 1, b.data(), 0, &dA));
    slq_solve_opts so;
    slq_solve_opts_default(&so);
    so.eps = o.eps;
    so.maxit = o.maxit;
    so.x_star = o.x_star ? o.x_star->data() : nullptr;
    so.track_true_residual = o.track_true_residual ? 1 : 0;
    const slq_gradient_params gp{params.alpha, params.beta, params.eta_hat};
    const std::size_t cap = static_cast<std::size_t>(o.maxit > 0 ? o.maxit : 0) + 2;
    Vector x(static_cast<std::size_t>(n)), est(cap), err(cap), tru(cap);
    slq_report r;
    const int st = slq_gradient_descent_hbm(b200::ctx(), dA, P.M.data().data(), nullptr, x0.data(), &gp, &so,
                                            x.data(), &r, est.data(), err.data(), tru.data());
    slq_dense_free(dA);
    b200::check(st);
    SolveReport rep;
    rep.residual_estimate.assign(est.begin(), est.begin() + r.n_estimate);
    rep.iterates_error.assign(err.begin(), err.begin() + r.n_err);
    rep.residual_true.assign(tru.begin(), tru.begin() + r.n_true);
    rep.iterations = static_cast<long>(r.iterations);
    rep.termination = static_cast<Termination>(r.termination);
    rep.sync_count = static_cast<long>(r.sync_count);
    rep.wall_time = r.wall_time;
    return {std::move(x), std::move(rep)};
}

// distsim.hpp:21-42
struct RowPartition {
    index_t m = 0;
    std::vector<index_t> boundaries;
    int blocks() const { return static_cast<int>(boundaries.size()) - 1; }
    index_t begin(int k) const { return boundaries[static_cast<std::size_t>(k)]; }
    index_t end(int k) const { return boundaries[static_cast<std::size_t>(k) + 1]; }
    index_t size(int k) const { return end(k) - begin(k); }
};
inline RowPartition partition_rows(index_t m, int p) {
    RowPartition part;
    part.m = m;
    part.boundaries.resize(static_cast<std::size_t>(p > 0 ? p : 0) + 1);
    b200::check(slq_partition_rows(m, p, part.boundaries.data()));
    return part;
}

}  // namespace SKETCHLSQ_B200_NAMESPACE
