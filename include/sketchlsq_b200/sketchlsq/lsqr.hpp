// sketchlsq/lsqr.hpp (B200 drop-in) -- preconditioned LSQR (lsqr.hpp:14-212).
//
// Two drop-in levels:
//  * solver level -- the DenseMatrix / CscMatrix overloads run the fused
//    device loop (one HBM pass over A per iteration computing A M v - alpha u,
//    A^T u_hat and ||u_hat||^2 together; M v reused across iterations; the
//    Givens recurrence and the stopping rule on the device; CUDA graphs of 8
//    iterations) through slq_lsqr / slq_lsqr_sparse;
//  * operator level -- the templates over any Op (SerialOperator here, whose
//    products are device passes, or a caller's own backend) run the
//    reference's algorithm (Alg. 2 of the paper, lsqr.hpp:50-168) host-driven,
//    so a custom Op keeps working exactly as with the reference.
// Both stop on phi_bar_{t+1} <= eps beta_1 (lsqr.hpp:163), return Breakdown
// when beta or alpha < 1e-300 after completing the rotation, and record the
// same histories.
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <functional>
#include <memory>
#include <utility>

#include "sketchlsq/device.hpp"
#include "sketchlsq/operators.hpp"
#include "sketchlsq/preconditioner.hpp"
#include "sketchlsq/solve_report.hpp"

namespace sketchlsq {

struct SolveOptions {
    double eps = 1e-10;
    long maxit = 100;
    const Vector* x_star = nullptr;
    bool track_true_residual = false;
    std::function<void(long t, double u_norm, double v_norm)> on_bidiag;
};

namespace detail {

template <class Op>
void record_iterate(const Op& op, const typename Op::VecM& b, const Vector& x, const SolveOptions& opts,
                    SolveReport& rep) {
    if (opts.x_star) {
        Vector e = *opts.x_star;
        axpy(-1.0, x, e);
        rep.iterates_error.push_back(op.error_norm(e));
    }
    if (opts.track_true_residual) rep.residual_true.push_back(op.residual_norm(b, x));
}

// Host-driven LSQR over an Op (operator-level drop-in).  State: u (m-space),
// v, w, x (n-space), the bidiagonalization scalars alpha / beta and the
// rotation scalars rho_bar / phi_bar.
template <class Op>
class LsqrDriver {
public:
    LsqrDriver(const Op& op, const Preconditioner& P, const typename Op::VecM& b, const Vector& x0,
               const SolveOptions& o, bool one_sync)
        : op_(op), P_(P), b_(b), o_(o), one_sync_(one_sync), x_(x0), t0_(std::chrono::steady_clock::now()) {}

    std::pair<Vector, SolveReport> run() {
        // beta_1 u_1 = b - A x0
        u_ = b_;
        op_.axpy(-1.0, op_.matvec(x_), u_);
        beta1_ = op_.norm(u_);
        record_iterate(op_, b_, x_, o_, rep_);
        if (beta1_ == 0.0) return done(Termination::Tolerance, 0);  // x0 solves the system
        op_.scal(1.0 / beta1_, u_);
        // alpha_1 v_1 = M^T A^T u_1
        v_ = apply_Mt(P_, op_.rmatvec(u_));
        alpha_ = norm2(v_);
        if (alpha_ == 0.0) return done(Termination::Tolerance, 0);  // residual orthogonal to range(A M)
        scal(1.0 / alpha_, v_);
        w_ = apply_M(P_, v_);
        phi_bar_ = beta1_;
        rho_bar_ = alpha_;
        std::tie(rep_.init_reductions, rep_.init_broadcasts) = op_.sync_snapshot();

        for (long t = 1; t <= o_.maxit; ++t) {
            // u_hat = A M v_t - alpha_t u_t
            typename Op::VecM uh = op_.matvec(apply_M(P_, v_));
            op_.axpy(-alpha_, u_, uh);
            double beta = 0.0;
            Vector z;
            if (one_sync_) {  // (A^T u_hat, ||u_hat||) in one synchronization
                auto zb = op_.rmatvec_and_norm(uh);
                beta = zb.second;
                if (beta < 1e-300) return breakdown(t, 0.0);
                z = std::move(zb.first);
                scal(1.0 / beta, z);
                op_.scal(1.0 / beta, uh);
            } else {
                beta = op_.norm(uh);
                if (beta < 1e-300) return breakdown(t, 0.0);
                op_.scal(1.0 / beta, uh);
                z = op_.rmatvec(uh);
            }
            u_ = std::move(uh);
            // v_hat = M^T A^T u_{t+1} - beta v_t
            Vector vh = apply_Mt(P_, z);
            axpy(-beta, v_, vh);
            const double alpha_next = norm2(vh);
            if (alpha_next < 1e-300) return breakdown(t, beta);
            scal(1.0 / alpha_next, vh);
            v_ = std::move(vh);
            alpha_ = alpha_next;
            if (o_.on_bidiag) o_.on_bidiag(t, op_.norm_uncounted(u_), norm2(v_));
            rotate(beta);
            rep_.residual_estimate.push_back(phi_bar_);
            record_iterate(op_, b_, x_, o_, rep_);
            if (phi_bar_ <= o_.eps * beta1_) return done(Termination::Tolerance, t);
        }
        return done(Termination::MaxIter, o_.maxit);
    }

private:
    // Givens rotation of step t, then x += (phi/rho) w, w = M v - (theta/rho) w
    void rotate(double beta) {
        const double rho = std::hypot(rho_bar_, beta);
        const double c = rho_bar_ / rho, s = beta / rho;
        const double theta = s * alpha_;
        rho_bar_ = -c * alpha_;
        const double phi = c * phi_bar_;
        phi_bar_ = s * phi_bar_;
        axpy(phi / rho, w_, x_);
        Vector wn = apply_M(P_, v_);
        axpy(-theta / rho, w_, wn);
        w_ = std::move(wn);
    }
    // a vanished beta / alpha ends the bidiagonalization: finish step t's
    // rotation with the vanished quantity as zero, which lands x on the solution
    std::pair<Vector, SolveReport> breakdown(long t, double beta_term) {
        const double rho = std::hypot(rho_bar_, beta_term);
        const double c = rho_bar_ / rho, s = beta_term / rho;
        const double phi = c * phi_bar_;
        phi_bar_ = s * phi_bar_;
        axpy(phi / rho, w_, x_);
        rep_.residual_estimate.push_back(phi_bar_);
        record_iterate(op_, b_, x_, o_, rep_);
        return done(Termination::Breakdown, t);
    }
    std::pair<Vector, SolveReport> done(Termination term, long iters) {
        rep_.termination = term;
        rep_.iterations = iters;
        std::tie(rep_.sync_count, rep_.broadcasts) = op_.sync_snapshot();
        rep_.wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0_).count();
        return {x_, rep_};
    }

    const Op& op_;
    const Preconditioner& P_;
    const typename Op::VecM& b_;
    const SolveOptions& o_;
    bool one_sync_;
    Vector x_, v_, w_;
    typename Op::VecM u_;
    double beta1_ = 0.0, alpha_ = 0.0, phi_bar_ = 0.0, rho_bar_ = 0.0;
    SolveReport rep_;
    std::chrono::steady_clock::time_point t0_;
};

template <class Op>
std::pair<Vector, SolveReport> lsqr_impl(const Op& op, const Preconditioner& P, const typename Op::VecM& b,
                                         const Vector& x0, const SolveOptions& opts, bool one_sync) {
    return LsqrDriver<Op>(op, P, b, x0, opts, one_sync).run();
}

inline void bidiag_trampoline(void* user, int64_t t, double un, double vn) {
    (*static_cast<const std::function<void(long, double, double)>*>(user))(static_cast<long>(t), un, vn);
}

inline slq_solve_opts device_opts(const SolveOptions& o, bool one_sync,
                                  const std::function<void(long, double, double)>* hook) {
    slq_solve_opts so;
    slq_solve_opts_default(&so);
    so.eps = o.eps;
    so.maxit = o.maxit;
    so.x_star = o.x_star ? o.x_star->data() : nullptr;
    so.track_true_residual = o.track_true_residual ? 1 : 0;
    so.one_sync = one_sync ? 1 : 0;
    if (hook && *hook) {
        so.on_bidiag = &bidiag_trampoline;
        so.on_bidiag_user = const_cast<void*>(static_cast<const void*>(hook));
    }
    return so;
}

inline SolveReport device_report(const slq_report& r, const Vector& est, const Vector& err, const Vector& tru) {
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
    return rep;
}

inline void check_shapes(index_t m, index_t n, const Preconditioner& P, const Vector& b, const Vector& x0) {
    if (static_cast<index_t>(b.size()) != m) throw DimensionMismatch("rmatvec: length mismatch");
    if (static_cast<index_t>(x0.size()) != n) throw DimensionMismatch("matvec: length mismatch");
    if (P.M.rows() != n || P.M.cols() != n) throw DimensionMismatch("tri_upper_matvec");
}

// the fused device solver over an uploaded operand (dense or CSR)
template <class Run>
std::pair<Vector, SolveReport> device_solve(index_t n, const SolveOptions& o, Run run) {
    const std::size_t cap = static_cast<std::size_t>(std::max<long>(o.maxit, 0)) + 2;
    Vector x(static_cast<std::size_t>(n)), est(cap), err(cap), tru(cap);
    slq_report r{};
    run(x.data(), &r, est.data(), err.data(), tru.data());
    return {std::move(x), device_report(r, est, err, tru)};
}

inline std::pair<Vector, SolveReport> lsqr_device(const DenseMatrix& A, const Preconditioner& P, const Vector& b,
                                                  const Vector& x0, const SolveOptions& o, bool one_sync) {
    check_shapes(A.rows(), A.cols(), P, b, x0);
    std::unique_ptr<slq_dense, int (*)(slq_dense*)> dA(nullptr, &slq_dense_free);
    slq_dense* h = nullptr;
    b200::check(slq_dense_upload(b200::ctx(), A.data().data(), A.rows(), A.cols(), std::max<index_t>(A.rows(), 1),
                                 b.data(), 0, &h));
    dA.reset(h);
    const slq_solve_opts so = device_opts(o, one_sync, &o.on_bidiag);
    return device_solve(A.cols(), o, [&](double* x, slq_report* r, double* est, double* err, double* tru) {
        b200::check(slq_lsqr(b200::ctx(), dA.get(), P.M.data().data(), nullptr, x0.data(), &so, x, r, est, err, tru));
    });
}

inline std::pair<Vector, SolveReport> lsqr_device(const CscMatrix& A, const Preconditioner& P, const Vector& b,
                                                  const Vector& x0, const SolveOptions& o, bool one_sync) {
    check_shapes(A.rows, A.cols, P, b, x0);
    std::unique_ptr<slq_sparse, int (*)(slq_sparse*)> dA(nullptr, &slq_sparse_free);
    slq_sparse* h = nullptr;
    b200::check(slq_sparse_upload_csc(b200::ctx(), A.rows, A.cols, A.col_pointers.data(), A.row_indices.data(),
                                      A.values.data(), b.data(), 0, &h));
    dA.reset(h);
    const slq_solve_opts so = device_opts(o, one_sync, &o.on_bidiag);
    return device_solve(A.cols, o, [&](double* x, slq_report* r, double* est, double* err, double* tru) {
        b200::check(
            slq_lsqr_sparse(b200::ctx(), dA.get(), P.M.data().data(), nullptr, x0.data(), &so, x, r, est, err, tru));
    });
}

}  // namespace detail

// lsqr.hpp:175-189: over any Op
template <class Op>
std::pair<Vector, SolveReport> lsqr(const Op& op, const Preconditioner& P, const typename Op::VecM& b,
                                    const Vector& x0, const SolveOptions& opts = {}) {
    return detail::lsqr_impl(op, P, b, x0, opts, false);
}
template <class Op>
std::pair<Vector, SolveReport> lsqr_one_sync(const Op& op, const Preconditioner& P, const typename Op::VecM& b,
                                             const Vector& x0, const SolveOptions& opts = {}) {
    return detail::lsqr_impl(op, P, b, x0, opts, true);
}

// lsqr.hpp:193-212: over plain matrices -- the fused device loop
inline std::pair<Vector, SolveReport> lsqr(const DenseMatrix& A, const Preconditioner& P, const Vector& b,
                                           const Vector& x0, const SolveOptions& opts = {}) {
    return detail::lsqr_device(A, P, b, x0, opts, false);
}
inline std::pair<Vector, SolveReport> lsqr(const CscMatrix& A, const Preconditioner& P, const Vector& b,
                                           const Vector& x0, const SolveOptions& opts = {}) {
    return detail::lsqr_device(A, P, b, x0, opts, false);
}
inline std::pair<Vector, SolveReport> lsqr_one_sync(const DenseMatrix& A, const Preconditioner& P, const Vector& b,
                                                    const Vector& x0, const SolveOptions& opts = {}) {
    return detail::lsqr_device(A, P, b, x0, opts, true);
}
inline std::pair<Vector, SolveReport> lsqr_one_sync(const CscMatrix& A, const Preconditioner& P, const Vector& b,
                                                    const Vector& x0, const SolveOptions& opts = {}) {
    return detail::lsqr_device(A, P, b, x0, opts, true);
}

}  // namespace sketchlsq
