// lsqr.cuh -- host side of the K4/K5 LSQR kernels.
#pragma once

#include <memory>
#include <vector>

#include "common.cuh"

namespace slq {

// Preconditioned LSQR (lsqr.hpp:50-168) on device-resident data.
//   A   : this rank's row block (device layout, b in column n unless b_dev given)
//   M   : n x n upper, column-major (device);  Mt: its row-major copy (device)
//   x0  : device n-vector (initial guess);   x: device n-vector (output)
// Histories (host, optional) as in the C-ABI.  With a communicator on ctx the
// partial A^T u / ||u||^2 of every iteration is summed by one ncclAllReduce.
// One HBM pass of the LSQR operator: u_hat = A p + c u (u_in == nullptr: u is
// the right-hand side stored with A), z = A^T u_hat (per-CTA partials in
// part[grid][n+1], the last entry holding ||u_hat||^2).  Dense (lsqr.cu) and
// sparse CSR (sparse.cu) implementations.
struct PassCall {
    const double* p;
    const double* u_in;
    double* u_out;
    const double* coef;  // device scalar c, or nullptr -> c_fixed
    double c_fixed;
    double* part;
    int want_z;
    const int* skip;     // nonzero -> no-op
};

struct PassOp {
    int64_t m = 0, n = 0;
    virtual ~PassOp() = default;
    virtual int grid() const = 0;
    virtual void pass(slq_ctx* ctx, const PassCall& c) const = 0;
    virtual std::vector<uint64_t> key() const = 0;  // identity for the graph cache
    virtual double pass_bytes() const = 0;          // algorithmic bytes of one pass
    // make the main stream wait for data the operator prepares asynchronously
    // (called by every routine before its first pass)
    virtual void ready(slq_ctx*) const {}
};

std::unique_ptr<PassOp> make_dense_op(slq_ctx* ctx, const slq_dense* A);

struct LsqrOut {
    int64_t iterations = 0;
    int termination = SLQ_TERM_MAXITER;
    int64_t n_estimate = 0, n_err = 0, n_true = 0;
    int64_t allreduces = 0, init_allreduces = 0;
    double seconds = 0.0;
    double backward_error = -1.0;
};

// abort (device, may be null): when *abort != 0 at the start the solve is a
// no-op (the preconditioner build failed; the caller reports the error).
void lsqr_dev(slq_ctx* ctx, const PassOp& op, const double* b_dev, const double* M, const double* Mt,
              const double* x0, double* x, const slq_solve_opts& opts, double* est_hist,
              double* err_hist, double* true_hist, LsqrOut& out, const double* abort = nullptr);

// gradient.hpp:56-115 gradient_descent_hbm (alpha, beta from hbm_params /
// gd_params); one fused pass per iteration.  Throws SLQ_DIVERGENCE.
void gd_dev(slq_ctx* ctx, const PassOp& op, const double* b_dev, const double* M, const double* Mt,
            const double* x0, double alpha, double beta, double* x, const slq_solve_opts& opts, double* est_hist,
            double* err_hist, double* true_hist, LsqrOut& out);

// Average seconds per fused-pass launch (K4), timed with CUDA events.
double time_fused_pass(slq_ctx* ctx, const PassOp& op, int reps);

// ||A^T r|| / (a_norm ||r||) for r = b - A x (one fused pass + allreduce);
// b_dev == nullptr: the right-hand side stored with A.
double backward_error_dev(slq_ctx* ctx, const PassOp& op, const double* b_dev, const double* x, double a_norm);

// The Op concept's products over one HBM pass (operators.hpp:15-51,
// distsim.hpp:283-331): y[m + kSparseRowPad] = A x (this rank's rows);
// z[n + 1] = [A^T y | ||y||^2] summed over ranks (one allreduce).  zero_n is
// n + 8 doubles of scratch.
void op_matvec_dev(slq_ctx* ctx, const PassOp& op, const double* x, double* y);
void op_rmatvec_dev(slq_ctx* ctx, const PassOp& op, const double* y, double* z, double* zero_n);

// comm.cu: in-place sum across ranks (no-op without a communicator).
void allreduce_sum(slq_ctx* ctx, double* buf, int64_t count);
void reduce_sum_root(slq_ctx* ctx, double* buf, int64_t count);
void broadcast_root(slq_ctx* ctx, double* buf, int64_t count);

}  // namespace slq

namespace slq {
void comm_unique_id(unsigned char out[128]);
void comm_init(slq_ctx* ctx, const unsigned char id[128], int rank, int nranks);
void comm_destroy(slq_ctx* ctx);
void comm_set_host(slq_ctx* ctx, const slq_host_comm& hc, int rank, int nranks);
}  // namespace slq
