// capi.cu -- the extern "C" boundary (include/slq_b200.h).
//
// Each entry point marshals host buffers, runs the device kernels on the
// context stream and maps slq::Error (thrown by the kernels' host code) to an
// slq_status plus a thread-local message, mirroring the reference's exception
// types (errors.hpp:9-76).
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <unordered_map>
#include <string>
#include <vector>

#include "common.cuh"
#include "lsqr.cuh"
#include "qr.cuh"
#include "sketch.cuh"
#include "sparse.cuh"
#include "spmm_general.cuh"

namespace {

thread_local std::string g_last_error;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return SLQ_OK;
    } catch (const slq::Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return SLQ_OOM;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return SLQ_CUDA;
    }
}

const double kZero = 0.0;  // stands in for the data pointer of an empty vector

void need(bool cond, int code, const char* what) {
    if (!cond) slq::fail(code, what);
}

// ------------------------------------------------------------ kernels

// column-major staging (rows x n, ld = rows_cap) -> row-major A rows [r0, r0+rows)
__global__ void colmajor_to_rows_kernel(const double* src, int64_t rows, int64_t rows_cap, int64_t n,
                                        const double* bsrc, double* A, int64_t ld) {
    __shared__ double tile[32][33];
    const int64_t c0 = static_cast<int64_t>(blockIdx.x) * 32;
    const int64_t r0 = static_cast<int64_t>(blockIdx.y) * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
    for (int k = ty; k < 32; k += 8) {
        const int64_t c = c0 + k, r = r0 + tx;
        double v = 0.0;
        if (r < rows) {
            if (c < n) v = src[c * rows_cap + r];
            else if (c == n && bsrc) v = bsrc[r];
        }
        tile[k][tx] = v;
    }
    __syncthreads();
    for (int k = ty; k < 32; k += 8) {
        const int64_t r = r0 + k, c = c0 + tx;
        if (r < rows && c < ld) A[r * ld + c] = tile[tx][k];
    }
}

__global__ void set_column_kernel(double* A, int64_t m, int64_t ld, int64_t col, const double* v) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < m) A[i * ld + col] = v ? v[i] : 0.0;
}

__global__ void transpose_square_kernel(const double* M, int64_t n, double* Mt) {
    __shared__ double tile[32][33];
    const int64_t c0 = static_cast<int64_t>(blockIdx.x) * 32, r0 = static_cast<int64_t>(blockIdx.y) * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;
    for (int k = ty; k < 32; k += 8)
        if (c0 + k < n && r0 + tx < n) tile[k][tx] = M[(c0 + k) * n + r0 + tx];
    __syncthreads();
    for (int k = ty; k < 32; k += 8)
        if (r0 + k < n && c0 + tx < n) Mt[(r0 + k) * n + c0 + tx] = tile[tx][k];
}

// y_j = Q(:, j)^T v, warp per column (Q column-major d x n)
__global__ void gemv_t_kernel(const double* Q, int64_t d, int64_t n, const double* v, double* y) {
    const int lane = threadIdx.x & 31;
    const int64_t j = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (j >= n) return;
    double s = 0.0;
    for (int64_t i = lane; i < d; i += 32) s += Q[j * d + i] * v[i];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) y[j] = s;
}

__global__ void csc_to_compact_kernel(const int64_t* rows, const double* vals, int64_t nnz, uint32_t* out) {
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e < nnz) out[e] = static_cast<uint32_t>(rows[e]) | (vals[e] < 0.0 ? 0x80000000u : 0u);
}



void transpose_square(slq_ctx* ctx, const double* M, int64_t n, double* Mt) {
    dim3 g(static_cast<unsigned>(slq::ceil_div(n, 32)), static_cast<unsigned>(slq::ceil_div(n, 32)));
    transpose_square_kernel<<<g, dim3(32, 8), 0, ctx->stream>>>(M, n, Mt);
    SLQ_LAUNCH_CHECK(ctx);
}

// Host column-major block (m x n, lda) + optional b -> device layout, in row
// blocks double-buffered over a copy stream.  on_rows(r0, rows), if given, is
// enqueued on the context stream after each block lands (the e2e path sketches
// the block there while the next one is in flight); blocks are then multiples
// of align rows.
void upload_dense(slq_ctx* ctx, const double* A, int64_t m, int64_t n, int64_t lda, const double* b, double* dst,
                  int64_t ld, const std::function<void(int64_t, int64_t)>& on_rows = {}, int64_t align = 32) {
    slq::Workspace& ws = ctx->ws;
    int64_t rows_cap = std::max<int64_t>(32, std::min<int64_t>(m, (int64_t(256) << 20) / (8 * std::max<int64_t>(n + 1, 1))));
    if (const char* e = std::getenv("SLQ_UPLOAD_ROWS")) rows_cap = std::max<int64_t>(1, std::atoll(e));  // diagnostics
    if (align > 1) rows_cap = std::max<int64_t>(align, rows_cap / align * align);
    double* stg[2];
    for (int s = 0; s < 2; ++s) stg[s] = static_cast<double*>(ws.staging[s].ensure(sizeof(double) * rows_cap * (n + 1)));
    cudaStream_t cs;
    SLQ_CUDA_CHECK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    cudaEvent_t copied[2], done[2];
    for (int s = 0; s < 2; ++s) {
        SLQ_CUDA_CHECK(cudaEventCreateWithFlags(&copied[s], cudaEventDisableTiming));
        SLQ_CUDA_CHECK(cudaEventCreateWithFlags(&done[s], cudaEventDisableTiming));
        SLQ_CUDA_CHECK(cudaEventRecord(done[s], ctx->stream));
    }
    int64_t k = 0;
    for (int64_t r0 = 0; r0 < m; r0 += rows_cap, ++k) {
        const int s = static_cast<int>(k & 1);
        const int64_t rows = std::min(rows_cap, m - r0);
        SLQ_CUDA_CHECK(cudaStreamWaitEvent(cs, done[s], 0));
        if (n > 0)
            SLQ_CUDA_CHECK(cudaMemcpy2DAsync(stg[s], sizeof(double) * rows_cap, A + r0, sizeof(double) * lda,
                                             sizeof(double) * rows, n, cudaMemcpyHostToDevice, cs));
        if (b)
            SLQ_CUDA_CHECK(cudaMemcpyAsync(stg[s] + n * rows_cap, b + r0, sizeof(double) * rows,
                                           cudaMemcpyHostToDevice, cs));
        SLQ_CUDA_CHECK(cudaEventRecord(copied[s], cs));
        SLQ_CUDA_CHECK(cudaStreamWaitEvent(ctx->stream, copied[s], 0));
        dim3 g(static_cast<unsigned>(slq::ceil_div(ld, 32)), static_cast<unsigned>(slq::ceil_div(rows, 32)));
        colmajor_to_rows_kernel<<<g, dim3(32, 8), 0, ctx->stream>>>(stg[s], rows, rows_cap, n,
                                                                   b ? stg[s] + n * rows_cap : nullptr,
                                                                   dst + r0 * ld, ld);
        SLQ_LAUNCH_CHECK(ctx);
        SLQ_CUDA_CHECK(cudaEventRecord(done[s], ctx->stream));
        if (on_rows) on_rows(r0, rows);
    }
    SLQ_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    SLQ_CUDA_CHECK(cudaStreamSynchronize(cs));
    for (int s = 0; s < 2; ++s) {
        cudaEventDestroy(copied[s]);
        cudaEventDestroy(done[s]);
    }
    cudaStreamDestroy(cs);
}

struct Timer {
    cudaEvent_t e;
    explicit Timer(cudaStream_t s) {
        SLQ_CUDA_CHECK(cudaEventCreate(&e));
        SLQ_CUDA_CHECK(cudaEventRecord(e, s));
    }
    ~Timer() { cudaEventDestroy(e); }
    void record(cudaStream_t s) { SLQ_CUDA_CHECK(cudaEventRecord(e, s)); }
    double since(const Timer& o) const {
        float ms = 0.f;
        SLQ_CUDA_CHECK(cudaEventSynchronize(e));
        SLQ_CUDA_CHECK(cudaEventElapsedTime(&ms, o.e, e));
        return ms * 1e-3;
    }
};

// Device buffers of the preconditioner: [M | Mt | R | x0 | qtb | status]
struct PrecondBufs {
    double *M, *Mt, *R, *x0, *qtb, *status;
};

PrecondBufs precond_bufs(slq_ctx* ctx, int64_t n) {
    double* base = static_cast<double*>(ctx->ws.mats.ensure(sizeof(double) * (3 * n * n + 2 * n + 8)));
    return {base, base + n * n, base + 2 * n * n, base + 3 * n * n, base + 3 * n * n + n, base + 3 * n * n + 2 * n};
}

// QR of Yaug (d x (n+1) incl. Sb) -> M, Mt, x0 on the device; times in t[3].
// marks (may be null): four timers re-recorded before QR, before R^-1, before
// x0 and at the end -- read by the caller after its final sync (no host wait here)
void build_precond_dev(slq_ctx* ctx, double* Yaug, int64_t d, int64_t n, bool with_sb, double* Q,
                       const PrecondBufs& P, Timer* const* marks) {
    if (marks) marks[0]->record(ctx->stream);
    slq::qr_factor_dev(ctx, Yaug, d, n, with_sb ? n + 1 : n, d, P.R, with_sb ? P.qtb : nullptr, Q, nullptr);
    if (marks) marks[1]->record(ctx->stream);
    slq::tri_inverse_dev(ctx, P.R, n, P.M, P.Mt);
    if (marks) marks[2]->record(ctx->stream);
    if (with_sb) slq::trmv_upper_dev(ctx, P.Mt, n, P.qtb, P.x0);
    if (marks) marks[3]->record(ctx->stream);
}

void fill_report(slq_report* r, const slq::LsqrOut& o) {
    if (!r) return;
    std::memset(r, 0, sizeof(*r));
    r->iterations = o.iterations;
    r->termination = o.termination;
    r->sync_count = o.allreduces;
    r->broadcasts = 0;
    r->init_reductions = o.init_allreduces;
    r->init_broadcasts = 0;
    r->wall_time = o.seconds;
    r->n_estimate = o.n_estimate;
    r->n_err = o.n_err;
    r->n_true = o.n_true;
    r->backward_error = o.backward_error;
}

// The dense or sparse operand of one rank: how to sketch it and how to make its LSQR pass.
struct Operand {
    int64_t m = 0, n = 0;
    // writes Y_aug (d x (n+1), column-major) = S [A b]; returns seconds spent generating S (0 if fused)
    std::function<void(double* Yaug, int64_t d, int64_t zeta, uint64_t seed, Timer* t_gen)> sketch;
    std::function<std::unique_ptr<slq::PassOp>()> make_op;
};

Operand dense_operand(slq_ctx* ctx, const slq_dense* A) {
    Operand o;
    o.m = A->m;
    o.n = A->n;
    o.sketch = [ctx, A](double* Yaug, int64_t d, int64_t zeta, uint64_t seed, Timer* t_gen) {
        slq::Workspace& ws = ctx->ws;
        const int64_t m = A->m;
        uint32_t* compact = static_cast<uint32_t*>(ws.compact.ensure(sizeof(uint32_t) * std::max<int64_t>(1, m * zeta)));
        int64_t* work = zeta > 32 ? static_cast<int64_t*>(ws.tmp.ensure(sizeof(int64_t) * m * zeta)) : nullptr;
        slq::generate_sparse_sign_dev(ctx, d, zeta, seed, A->row_begin, m, compact, work, nullptr, nullptr, nullptr);
        if (t_gen) SLQ_CUDA_CHECK(cudaEventRecord(t_gen->e, ctx->stream));
        slq::sketch_apply_compact_dev(ctx, A, d, compact, nullptr, zeta, 1.0 / std::sqrt(static_cast<double>(zeta)),
                                      false, Yaug);
    };
    o.make_op = [ctx, A] { return slq::make_dense_op(ctx, A); };
    return o;
}

Operand sparse_operand(slq_ctx* ctx, const slq_sparse* A) {
    Operand o;
    o.m = A->m;
    o.n = A->n;
    o.sketch = [ctx, A](double* Yaug, int64_t d, int64_t zeta, uint64_t seed, Timer* t_gen) {
        if (t_gen) SLQ_CUDA_CHECK(cudaEventRecord(t_gen->e, ctx->stream));
        slq::sketch_apply_sparse_dev(ctx, A, d, zeta, seed, Yaug);
    };
    o.make_op = [ctx, A] { return slq::make_sparse_op(ctx, A, true); };
    return o;
}

// A still on the host (column-major, lda): the sketch uploads it block by block
// into Ad's device storage and applies S to each block as it lands, so the
// HBM-side work of the sketch hides behind the PCIe copy of the next block.
Operand host_dense_operand(slq_ctx* ctx, slq_dense* Ad, const double* Ah, int64_t lda, const double* bh) {
    Operand o;
    o.m = Ad->m;
    o.n = Ad->n;
    o.sketch = [ctx, Ad, Ah, lda, bh](double* Yaug, int64_t d, int64_t zeta, uint64_t seed, Timer* t_gen) {
        slq::Workspace& ws = ctx->ws;
        const int64_t m = Ad->m;
        uint32_t* compact = static_cast<uint32_t*>(ws.compact.ensure(sizeof(uint32_t) * std::max<int64_t>(1, m * zeta)));
        int64_t* work = zeta > 32 ? static_cast<int64_t*>(ws.tmp.ensure(sizeof(int64_t) * m * zeta)) : nullptr;
        slq::generate_sparse_sign_dev(ctx, d, zeta, seed, Ad->row_begin, m, compact, work, nullptr, nullptr, nullptr);
        if (t_gen) SLQ_CUDA_CHECK(cudaEventRecord(t_gen->e, ctx->stream));
        if (m == 0) {
            SLQ_CUDA_CHECK(cudaMemsetAsync(Yaug, 0, sizeof(double) * d * (Ad->n + 1), ctx->stream));
            return;
        }
        slq::DenseGather G = slq::dense_gather_plan(ctx, m, Ad->n, Ad->ld, d, compact, nullptr, zeta,
                                                    1.0 / std::sqrt(static_cast<double>(zeta)), false, Yaug, true);
        upload_dense(ctx, Ah, m, Ad->n, lda, bh, Ad->A, Ad->ld,
                     [&](int64_t r0, int64_t rows) { slq::dense_gather_rows(ctx, G, Ad->A, r0, r0 + rows); },
                     G.chunk_rows());
        slq::dense_gather_finish(ctx, G);
    };
    o.make_op = [ctx, Ad] { return slq::make_dense_op(ctx, Ad); };
    return o;
}

// RAII: inside a solve, device-detected errors go to P.status (no mid-solve
// host reads); restored on every exit path
struct DeferGuard {
    slq_ctx* ctx;
    DeferGuard(slq_ctx* c, double* status) : ctx(c) { ctx->defer_status = status; }
    ~DeferGuard() { ctx->defer_status = nullptr; }
};

int run_solve(slq_ctx* ctx, const Operand& A, int64_t d, int64_t zeta, uint64_t seed, const slq_solve_opts* opts_in,
              double* x_out, slq_report* report, slq_phase_times* times, double* est) {
    const int rc = guarded([&] {
        need(ctx != nullptr, SLQ_INVALID_ARG, "solve: null handle");
        slq_solve_opts opts;
        if (opts_in) opts = *opts_in;
        else slq_solve_opts_default(&opts);
        const int64_t n = A.n;
        need(n >= 1, SLQ_INVALID_DIMS, "solve: n < 1");
        need(d > n, SLQ_INVALID_DIMS, "SketchParams: need n < d <= m");
        need(zeta >= 1 && zeta <= d, SLQ_INVALID_SPARSITY, "SketchParams: need 1 <= zeta <= d");
        const int64_t launches0 = ctx->launches, nccl0 = ctx->nccl_calls;
        slq::Workspace& ws = ctx->ws;
        double* Yaug = static_cast<double*>(ws.yaug.ensure(sizeof(double) * d * (n + 1)));
        PrecondBufs P = precond_bufs(ctx, n);
        // The whole solve is enqueued without a host round trip: device-side
        // error conditions land in P.status (broadcast with M on multiple
        // GPUs; LSQR turns into no-ops when it is set) and are read once at
        // the end together with x.
        SLQ_CUDA_CHECK(cudaMemsetAsync(P.status, 0, sizeof(double), ctx->stream));
        DeferGuard defer(ctx, P.status);

        // SLQ_TRACE=1: host timestamps per phase on stderr (diagnostics)
        static const bool trace = std::getenv("SLQ_TRACE") != nullptr;
        const auto h0 = std::chrono::steady_clock::now();
        auto mark = [&](const char* what) {
            if (trace)
                std::fprintf(stderr, "[slq] %-10s host %.3f ms\n", what,
                             std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count());
        };
        Timer t0(ctx->stream);
        // the operator first: a sparse A's transposed copy (if not built yet)
        // is then built on the side stream while the sketch and QR run
        auto op = A.make_op();
        Timer t1(ctx->stream);
        A.sketch(Yaug, d, zeta, seed, &t1);
        mark("apply");
        Timer t2(ctx->stream);
        slq::reduce_sum_root(ctx, Yaug, d * (n + 1));
        Timer t3(ctx->stream);
        Timer q0(ctx->stream), q1(ctx->stream), q2(ctx->stream), q3(ctx->stream);
        Timer* const qm[4] = {&q0, &q1, &q2, &q3};
        std::string root_error;
        if (ctx->rank == 0) {
            int code = SLQ_OK;
            try {
                build_precond_dev(ctx, Yaug, d, n, true, nullptr, P, qm);
            } catch (const slq::Error& e) {
                code = e.code;
                root_error = e.what();
            } catch (const std::bad_alloc&) {
                // any failure on rank 0 must still reach the status broadcast,
                // or ranks 1..N-1 would block in ncclBroadcast forever
                code = SLQ_OOM;
                root_error = "preconditioner build: host allocation failed";
            } catch (const std::exception& e) {
                code = SLQ_CUDA;
                root_error = e.what();
            }
            if (code != SLQ_OK) {
                if (!slq::has_comm(ctx)) slq::fail(code, root_error);
                const double st = code;
                SLQ_CUDA_CHECK(cudaMemcpyAsync(P.status, &st, sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
            }
        }
        Timer t4(ctx->stream);
        if (slq::has_comm(ctx)) {
            // status travels with M, M^T, x0: every rank learns of a rank-0
            // failure from the same broadcasts, without a host round trip
            slq::broadcast_root(ctx, P.status, 1);
            slq::broadcast_root(ctx, P.M, n * n);
            slq::broadcast_root(ctx, P.Mt, n * n);
            slq::broadcast_root(ctx, P.x0, n);
        }
        mark("precond");
        Timer t5(ctx->stream);
        double* x = static_cast<double*>(ws.xbuf.ensure(sizeof(double) * (n + 8)));
        slq::LsqrOut lo;
        slq::lsqr_dev(ctx, *op, nullptr, P.M, P.Mt, P.x0, x, opts, est, nullptr, nullptr, lo, P.status);
        mark("lsqr");
        Timer t6(ctx->stream);
        double st = 0.0;
        SLQ_CUDA_CHECK(cudaMemcpyAsync(&st, P.status, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        SLQ_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        if (st != 0.0) {
            const int code = static_cast<int>(st);
            if (code == slq::kStatusSketchOverflow) slq::fail(code, "sketch bucket overflow");
            if (!root_error.empty()) slq::fail(code, root_error);
            slq::fail(code, code == SLQ_RANK_DEFICIENT     ? "householder_qr: the sketch is numerically rank deficient"
                            : code == SLQ_SINGULAR_TRIANGULAR ? "tri_inverse: zero diagonal"
                            : ctx->rank == 0                  ? "solve failed on the device"
                                                              : "preconditioner build failed on rank 0");
        }
        if ((opts.backward_tol > 0.0 || opts.a_norm_est > 0.0) && lo.backward_error < 0.0)
            lo.backward_error = slq::backward_error_dev(ctx, *op, nullptr, x, opts.a_norm_est > 0.0 ? opts.a_norm_est : 1.0);
        if (x_out) SLQ_CUDA_CHECK(cudaMemcpy(x_out, x, sizeof(double) * n, cudaMemcpyDeviceToHost));
        fill_report(report, lo);
        mark("finish");
        if (times) {
            // QR / R^-1 / x0 split from the events build_precond_dev recorded
            const double tq[3] = {q1.since(q0), q2.since(q1), q3.since(q2)};
            times->generate = t1.since(t0);
            times->apply = t2.since(t1);
            times->reduce = t3.since(t2);
            times->qr = ctx->rank == 0 ? tq[0] : 0.0;
            times->inverse = ctx->rank == 0 ? tq[1] : 0.0;
            times->x0 = (ctx->rank == 0 ? tq[2] : 0.0) + t5.since(t4);
            times->lsqr = t6.since(t5);
            times->total = t6.since(t0);
            times->lsqr_per_iteration = lo.iterations > 0 ? lo.seconds / static_cast<double>(lo.iterations) : 0.0;
            times->nccl_calls = ctx->nccl_calls - nccl0;
            times->kernel_launches = ctx->launches - launches0;
        }
    });
    if (rc == slq::kStatusSketchOverflow && ctx && !ctx->force_row_gather) {
        // a K2d bucket overflowed (recorded on the device): redo with the register gather
        ctx->force_row_gather = true;
        const int rc2 = run_solve(ctx, A, d, zeta, seed, opts_in, x_out, report, times, est);
        ctx->force_row_gather = false;
        return rc2;
    }
    return rc;
}

}  // namespace

namespace {

// shared body of the dense / sparse gradient_descent_hbm entry points
template <class MakeOp>
void gd_common(slq_ctx* ctx, int64_t m, int64_t n, const double* M, const double* b, const double* x0,
               const slq_gradient_params* params, const slq_solve_opts* opts_in, double* x_out, slq_report* report,
               double* residual_estimate, double* iterates_error, double* residual_true, int64_t b_pad,
               MakeOp make_op) {
    slq_solve_opts opts;
    if (opts_in) opts = *opts_in;
    else slq_solve_opts_default(&opts);
    PrecondBufs P = precond_bufs(ctx, n);
    SLQ_CUDA_CHECK(cudaMemcpyAsync(P.M, M, sizeof(double) * n * n, cudaMemcpyHostToDevice, ctx->stream));
    transpose_square(ctx, P.M, n, P.Mt);
    SLQ_CUDA_CHECK(cudaMemcpyAsync(P.x0, x0, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
    slq::DevBuf db, dx;
    double* bd = nullptr;
    if (b) {
        bd = static_cast<double*>(db.ensure(sizeof(double) * (m + b_pad)));
        if (b_pad) SLQ_CUDA_CHECK(cudaMemsetAsync(bd, 0, sizeof(double) * (m + b_pad), ctx->stream));
        SLQ_CUDA_CHECK(cudaMemcpyAsync(bd, b, sizeof(double) * m, cudaMemcpyHostToDevice, ctx->stream));
    }
    double* x = static_cast<double*>(dx.ensure(sizeof(double) * (n + 8)));
    slq::LsqrOut lo;
    const auto h0 = std::chrono::steady_clock::now();
    slq::gd_dev(ctx, *make_op(), bd, P.M, P.Mt, P.x0, params->alpha, params->beta, x, opts, residual_estimate,
                iterates_error, residual_true, lo);
    SLQ_CUDA_CHECK(cudaMemcpy(x_out, x, sizeof(double) * n, cudaMemcpyDeviceToHost));
    lo.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - h0).count();
    fill_report(report, lo);
}

}  // namespace

extern "C" {

const char* slq_last_error(void) { return g_last_error.c_str(); }
const char* slq_version(void) { return "slq_b200 0.1 (sm_100a)"; }

void slq_solve_opts_default(slq_solve_opts* o) {
    std::memset(o, 0, sizeof(*o));
    o->eps = 1e-10;  // lsqr.hpp:15
    o->maxit = 100;  // lsqr.hpp:16
}

int slq_ctx_create(int device, slq_ctx** out) {
    return guarded([&] {
        need(out != nullptr, SLQ_INVALID_ARG, "ctx_create: null out");
        int ndev = 0;
        SLQ_CUDA_CHECK(cudaGetDeviceCount(&ndev));
        need(device >= 0 && device < ndev, SLQ_INVALID_ARG, "ctx_create: bad device");
        SLQ_CUDA_CHECK(cudaSetDevice(device));
        cudaDeviceProp prop;
        SLQ_CUDA_CHECK(cudaGetDeviceProperties(&prop, device));
        need(prop.major >= 10, SLQ_UNSUPPORTED, "ctx_create: needs an sm_100 (Blackwell) GPU");
        auto* c = new slq_ctx();
        c->device = device;
        c->num_sms = prop.multiProcessorCount;
        SLQ_CUDA_CHECK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        c->own_stream = true;
        *out = c;
    });
}

int slq_ctx_destroy(slq_ctx* ctx) {
    return guarded([&] {
        if (!ctx) return;
        cudaSetDevice(ctx->device);
        cudaStreamSynchronize(ctx->stream);
        slq::comm_destroy(ctx);
        if (ctx->lsqr_exec) cudaGraphExecDestroy(ctx->lsqr_exec);
        for (auto& g : ctx->qr_graphs)
            if (g.exec) cudaGraphExecDestroy(g.exec);
        if (ctx->lsqr_hdone) cudaFreeHost(ctx->lsqr_hdone);
        if (ctx->aux) cudaStreamDestroy(ctx->aux);
        for (cudaEvent_t e : ctx->aux_ev)
            if (e) cudaEventDestroy(e);
        if (ctx->qr_hi) cudaStreamDestroy(ctx->qr_hi);
        if (ctx->qr_lo) cudaStreamDestroy(ctx->qr_lo);
        for (cudaEvent_t e : ctx->qr_ev)
            if (e) cudaEventDestroy(e);
        for (cudaEvent_t e : ctx->lsqr_ev)
            if (e) cudaEventDestroy(e);
        if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
        delete ctx;
    });
}

int slq_ctx_set_stream(slq_ctx* ctx, void* s) {
    return guarded([&] {
        need(ctx != nullptr, SLQ_INVALID_ARG, "null ctx");
        if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
        if (ctx->lsqr_exec) cudaGraphExecDestroy(ctx->lsqr_exec);
        ctx->lsqr_exec = nullptr;
        ctx->lsqr_key.clear();
        for (auto& g : ctx->qr_graphs)
            if (g.exec) cudaGraphExecDestroy(g.exec);
        ctx->qr_graphs.clear();
        ctx->stream = static_cast<cudaStream_t>(s);
        ctx->own_stream = false;
    });
}

int slq_ctx_synchronize(slq_ctx* ctx) {
    return guarded([&] { SLQ_CUDA_CHECK(cudaStreamSynchronize(ctx->stream)); });
}

int64_t slq_ctx_kernel_launches(const slq_ctx* ctx) { return ctx ? ctx->launches : 0; }

int slq_ctx_set_host_comm(slq_ctx* ctx, const slq_host_comm* comm, int rank, int nranks) {
    return guarded([&] {
        need(ctx && comm, SLQ_INVALID_ARG, "set_host_comm: null argument");
        slq::comm_set_host(ctx, *comm, rank, nranks);
    });
}

int slq_comm_unique_id(unsigned char id_out[128]) {
    return guarded([&] { slq::comm_unique_id(id_out); });
}

int slq_ctx_init_comm(slq_ctx* ctx, const unsigned char id[128], int rank, int nranks) {
    return guarded([&] { slq::comm_init(ctx, id, rank, nranks); });
}

int slq_partition_rows(int64_t m, int p, int64_t* boundaries) {
    return guarded([&] {
        // distsim.hpp:31-42
        need(p >= 1 && static_cast<int64_t>(p) <= m, SLQ_INVALID_DIMS, "partition_rows: need 1 <= p <= m");
        const int64_t stride = m / p;
        for (int k = 0; k < p; ++k) boundaries[k] = stride * k;
        boundaries[p] = m;
    });
}

int slq_generate_sparse_sign(slq_ctx* ctx, int64_t d, int64_t col_begin, int64_t ncols, int64_t zeta, uint64_t seed,
                             int64_t* row_indices, double* values, int64_t* col_pointers,
                             slq_rejection_stats* stats) {
    return guarded([&] {
        need(ctx != nullptr, SLQ_INVALID_ARG, "null ctx");
        if (zeta > d || zeta < 1) slq::fail(SLQ_INVALID_SPARSITY, "generate_sparse_sign: need 1 <= zeta <= d");
        need(ncols >= 0 && col_begin >= 0, SLQ_INVALID_DIMS, "generate_sparse_sign: bad column window");
        SLQ_CUDA_CHECK(cudaSetDevice(ctx->device));
        const int64_t nnz = ncols * zeta;
        slq::DevBuf rows, vals, cp, st;
        int64_t* drows = static_cast<int64_t*>(rows.ensure(sizeof(int64_t) * std::max<int64_t>(nnz, 1)));
        double* dvals = static_cast<double*>(vals.ensure(sizeof(double) * std::max<int64_t>(nnz, 1)));
        int64_t* dcp = static_cast<int64_t*>(cp.ensure(sizeof(int64_t) * (ncols + 1)));
        unsigned long long* dst = static_cast<unsigned long long*>(st.ensure(2 * sizeof(unsigned long long)));
        SLQ_CUDA_CHECK(cudaMemsetAsync(dst, 0, 2 * sizeof(unsigned long long), ctx->stream));
        slq::generate_sparse_sign_dev(ctx, d, zeta, seed, col_begin, ncols, nullptr, drows, dvals, dcp, dst);
        if (row_indices) SLQ_CUDA_CHECK(cudaMemcpyAsync(row_indices, drows, sizeof(int64_t) * nnz, cudaMemcpyDeviceToHost, ctx->stream));
        if (values) SLQ_CUDA_CHECK(cudaMemcpyAsync(values, dvals, sizeof(double) * nnz, cudaMemcpyDeviceToHost, ctx->stream));
        if (col_pointers) SLQ_CUDA_CHECK(cudaMemcpyAsync(col_pointers, dcp, sizeof(int64_t) * (ncols + 1), cudaMemcpyDeviceToHost, ctx->stream));
        unsigned long long hs[2] = {0, 0};
        SLQ_CUDA_CHECK(cudaMemcpyAsync(hs, dst, sizeof(hs), cudaMemcpyDeviceToHost, ctx->stream));
        SLQ_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        if (stats) {
            stats->columns_resampled += static_cast<int64_t>(hs[0]);
            stats->resample_rounds += static_cast<int64_t>(hs[1]);
        }
    });
}

int slq_rejection_sample_columns(slq_ctx* ctx, int64_t d, int64_t m, int64_t zeta, uint64_t seed, int64_t* out,
                                 slq_rejection_stats* stats) {
    return guarded([&] {
        need(ctx != nullptr, SLQ_INVALID_ARG, "null ctx");
        if (zeta > d || zeta < 1) slq::fail(SLQ_INVALID_SPARSITY, "rejection_sample_columns: need 1 <= zeta <= d");
        SLQ_CUDA_CHECK(cudaSetDevice(ctx->device));
        const int64_t nnz = m * zeta;
        slq::DevBuf rows, st;
        int64_t* drows = static_cast<int64_t*>(rows.ensure(sizeof(int64_t) * std::max<int64_t>(nnz, 1)));
        unsigned long long* dst = static_cast<unsigned long long*>(st.ensure(2 * sizeof(unsigned long long)));
        SLQ_CUDA_CHECK(cudaMemsetAsync(dst, 0, 2 * sizeof(unsigned long long), ctx->stream));
        // sketch.hpp:105-124 draws column j from substream 2j: identical to the
        // index part of sparse_sign_block with col_begin = 0.
        slq::generate_sparse_sign_dev(ctx, d, zeta, seed, 0, m, nullptr, drows, nullptr, nullptr, dst);
        SLQ_CUDA_CHECK(cudaMemcpyAsync(out, drows, sizeof(int64_t) * nnz, cudaMemcpyDeviceToHost, ctx->stream));
        unsigned long long hs[2] = {0, 0};
        SLQ_CUDA_CHECK(cudaMemcpyAsync(hs, dst, sizeof(hs), cudaMemcpyDeviceToHost, ctx->stream));
        SLQ_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        if (stats) {
            stats->columns_resampled += static_cast<int64_t>(hs[0]);
            stats->resample_rounds += static_cast<int64_t>(hs[1]);
        }
    });
}

int slq_dense_upload(slq_ctx* ctx, const double* A, int64_t m, int64_t n, int64_t lda, const double* b,
                     int64_t row_begin, slq_dense** out) {
    return guarded([&] {
        need(ctx && out, SLQ_INVALID_ARG, "dense_upload: null argument");
        need(m >= 0 && n >= 0 && lda >= m && row_begin >= 0, SLQ_INVALID_DIMS, "dense_upload: bad shape");
        need(A != nullptr || m * n == 0, SLQ_INVALID_ARG, "dense_upload: null A");
        SLQ_CUDA_CHECK(cudaSetDevice(ctx->device));
        auto* h = new slq_dense();
        h->ctx = ctx;
        h->m = m;
        h->n = n;
        h->ld = slq::dense_ld(n);
        h->row_begin = row_begin;
        h->owned = true;
        h->has_b = b != nullptr;
        cudaError_t e = cudaMalloc(&h->A, sizeof(double) * std::max<int64_t>(1, m * h->ld));
        if (e != cudaSuccess) {
            delete h;
            SLQ_CUDA_CHECK(e);
        }
        if (m > 0) upload_dense(ctx, A, m, n, lda, b, h->A, h->ld);
        *out = h;
    });
}

int slq_dense_create(slq_ctx* ctx, int64_t m, int64_t n, int64_t row_begin, slq_dense** out, double** dev_ptr,
                     int64_t* ld) {
    return guarded([&] {
        need(ctx && out, SLQ_INVALID_ARG, "dense_create: null argument");
        need(m >= 0 && n >= 0 && row_begin >= 0, SLQ_INVALID_DIMS, "dense_create: bad shape");
        SLQ_CUDA_CHECK(cudaSetDevice(ctx->device));
        auto* h = new slq_dense();
        h->ctx = ctx;
        h->m = m;
        h->n = n;
        h->ld = slq::dense_ld(n);
        h->row_begin = row_begin;
        h->owned = true;
        h->has_b = true;  // the caller fills column n (zero until then)
        cudaError_t e = cudaMalloc(&h->A, sizeof(double) * std::max<int64_t>(1, m * h->ld));
        if (e != cudaSuccess) {
            delete h;
            SLQ_CUDA_CHECK(e);
        }
        SLQ_CUDA_CHECK(cudaMemsetAsync(h->A, 0, sizeof(double) * m * h->ld, ctx->stream));
        SLQ_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        *out = h;
        if (dev_ptr) *dev_ptr = h->A;
        if (ld) *ld = h->ld;
    });
}

int slq_dense_wrap(slq_ctx* ctx, double* dev_ptr, int64_t m, int64_t n, int64_t ld, int64_t row_begin,
                   slq_dense** out) {
    return guarded([&] {
        need(ctx && out && (dev_ptr || m == 0), SLQ_INVALID_ARG, "dense_wrap: null argument");
        need(ld >= n + 1 && ld % 4 == 0, SLQ_INVALID_DIMS, "dense_wrap: ld must be >= n+1 and a multiple of 4");
        need((reinterpret_cast<uintptr_t>(dev_ptr) & 31) == 0, SLQ_INVALID_ARG, "dense_wrap: pointer not 32-byte aligned");
        auto* h = new slq_dense();
        h->ctx = ctx;
        h->A = dev_ptr;
        h->m = m;
        h->n = n;
        h->ld = ld;
        h->row_begin = row_begin;
        h->owned = false;
        h->has_b = true;
        // The passes multiply the padding columns (n, ld) by p = 0: zero them so
        // that non-finite garbage in caller storage cannot poison u_hat (0 * NaN).
        if (m > 0 && ld > n + 1) {
            SLQ_CUDA_CHECK(cudaMemset2DAsync(dev_ptr + n + 1, sizeof(double) * ld, 0, sizeof(double) * (ld - n - 1), m,
                                             ctx->stream));
            SLQ_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        }
        *out = h;
    });
}

int slq_dense_set_rhs(slq_dense* A, const double* b) {
    return guarded([&] {
        need(A != nullptr, SLQ_INVALID_ARG, "null matrix");
        slq_ctx* ctx = A->ctx;
        slq::DevBuf tmp;
        double* db = nullptr;
        if (b) {
            db = static_cast<double*>(tmp.ensure(sizeof(double) * std::max<int64_t>(1, A->m)));
            SLQ_CUDA_CHECK(cudaMemcpyAsync(db, b, sizeof(double) * A->m, cudaMemcpyHostToDevice, ctx->stream));
        }
        if (A->m > 0) {
            set_column_kernel<<<static_cast<unsigned>(slq::ceil_div(A->m, 256)), 256, 0, ctx->stream>>>(A->A, A->m, A->ld,
                                                                                                    A->n, db);
            SLQ_LAUNCH_CHECK(ctx);
        }
        SLQ_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        A->has_b = b != nullptr;
    });
}

int slq_dense_free(slq_dense* A) {
    return guarded([&] {
        if (!A) return;
        // no access to A->ctx: the matrix may outlive its context (e.g. a
        // garbage collector finalizing both in any order); cudaFree itself
        // waits for the device work that still reads the buffer
        if (A->owned && A->A) cudaFree(A->A);
        delete A;
    });
}

int64_t slq_dense_ld(const slq_dense* A) { return A ? A->ld : 0; }

int slq_sketch_apply(slq_ctx* ctx, const slq_dense* A, int64_t d, int64_t zeta, uint64_t seed, int exact, double* Y,
                     double* Sb) {
    return guarded([&] {
        need(ctx && A, SLQ_INVALID_ARG, "sketch_apply: null handle");
        if (zeta > d || zeta < 1) slq::fail(SLQ_INVALID_SPARSITY, "apply: need 1 <= zeta <= d");
        const int64_t n = A->n;
        double* Yaug = static_cast<double*>(ctx->ws.yaug.ensure(sizeof(double) * d * (n + 1)));
        slq::sketch_apply_dev(ctx, A, d, zeta, seed, exact != 0, Yaug);
        slq::allreduce_sum(ctx, Yaug, d * (n + 1));  // distsim.hpp:383-396: every caller gets the total
        if (Y) SLQ_CUDA_CHECK(cudaMemcpyAsync(Y, Yaug, sizeof(double) * d * n, cudaMemcpyDeviceToHost, ctx->stream));
        if (Sb) SLQ_CUDA_CHECK(cudaMemcpyAsync(Sb, Yaug + d * n, sizeof(double) * d, cudaMemcpyDeviceToHost, ctx->stream));
        SLQ_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    });
}

int slq_spmm_csc_dense(slq_ctx* ctx, int64_t d, int64_t m, const int64_t* row_indices, const double* values,
                       const int64_t* col_pointers, const double* A, int64_t n, int64_t lda, double* Y) {
    return guarded([&] {
        need(ctx && col_pointers && Y, SLQ_INVALID_ARG, "spmm: null argument");
        need(lda >= m, SLQ_INVALID_DIMS, "spmm: lda < m");
        const int64_t nnz = col_pointers[m];
        need(col_pointers[0] == 0 && nnz >= 0, SLQ_INVALID_ARG, "spmm: bad col_pointers");
        slq_dense* Ad = nullptr;
        int st = slq_dense_upload(ctx, A, m, n, lda, nullptr, 0, &Ad);
        if (st != SLQ_OK) slq::fail(st, g_last_error);
        struct Free {
            slq_dense* p;
            ~Free() { slq_dense_free(p); }
        } fr{Ad};
        slq::DevBuf drows, dvals, dcp, dcomp, dY;
        int64_t* r = static_cast<int64_t*>(drows.ensure(sizeof(int64_t) * std::max<int64_t>(1, nnz)));
        double* v = static_cast<double*>(dvals.ensure(sizeof(double) * std::max<int64_t>(1, nnz)));
        int64_t* cp = static_cast<int64_t*>(dcp.ensure(sizeof(int64_t) * (m + 1)));
        double* Yd = static_cast<double*>(dY.ensure(sizeof(double) * std::max<int64_t>(1, d * (n + 1))));
        if (nnz > 0) {
            SLQ_CUDA_CHECK(cudaMemcpyAsync(r, row_indices, sizeof(int64_t) * nnz, cudaMemcpyHostToDevice, ctx->stream));
            SLQ_CUDA_CHECK(cudaMemcpyAsync(v, values, sizeof(double) * nnz, cudaMemcpyHostToDevice, ctx->stream));
        }
        SLQ_CUDA_CHECK(cudaMemcpyAsync(cp, col_pointers, sizeof(int64_t) * (m + 1), cudaMemcpyHostToDevice, ctx->stream));
        const slq::SpmmCheck chk = slq::csc_check_dev(ctx, r, v, nnz, d);
        need(!chk.row_out_of_range, SLQ_INVALID_ARG, "spmm: row index out of range");
        if (chk.mixed_magnitudes) {
            // arbitrary values: the general kernel (reference order, bit-identical)
            slq::spmm_general_dev(ctx, d, m, nnz, r, v, cp, n, Ad->A, Ad->ld, nullptr, nullptr, nullptr, Yd);
        } else {
            // a sparse-sign matrix (one magnitude): the sketch gather in exact mode
            const double val = nnz > 0 ? std::fabs(values[0]) : 0.0;
            uint32_t* comp = static_cast<uint32_t*>(dcomp.ensure(sizeof(uint32_t) * std::max<int64_t>(1, nnz)));
            if (nnz > 0) {
                csc_to_compact_kernel<<<static_cast<unsigned>(slq::ceil_div(nnz, 256)), 256, 0, ctx->stream>>>(r, v, nnz,
                                                                                                            comp);
                SLQ_LAUNCH_CHECK(ctx);
            }
            int64_t zmax = 1;
            for (int64_t j = 0; j < m; ++j) zmax = std::max(zmax, col_pointers[j + 1] - col_pointers[j]);
            slq::sketch_apply_compact_dev(ctx, Ad, d, comp, cp, zmax, val, true, Yd);
        }
        if (d * n > 0)
            SLQ_CUDA_CHECK(cudaMemcpyAsync(Y, Yd, sizeof(double) * d * n, cudaMemcpyDeviceToHost, ctx->stream));
        SLQ_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    });
}

int slq_householder_qr(slq_ctx* ctx, const double* Y, int64_t d, int64_t n, int64_t ldy, double* Q, double* R) {
    return guarded([&] {
        need(ctx && Y && R, SLQ_INVALID_ARG, "householder_qr: null argument");
        if (d < n) slq::fail(SLQ_DIMENSION_MISMATCH, "householder_qr: need rows >= cols");
        need(ldy >= d, SLQ_INVALID_DIMS, "householder_qr: ldy < d");
        slq::DevBuf dY, dQ, dR;
        double* y = static_cast<double*>(dY.ensure(sizeof(double) * std::max<int64_t>(1, d * n)));
        SLQ_CUDA_CHECK(cudaMemcpy2DAsync(y, sizeof(double) * d, Y, sizeof(double) * ldy, sizeof(double) * d, n,
                                         cudaMemcpyHostToDevice, ctx->stream));
        double* r = static_cast<double*>(dR.ensure(sizeof(double) * std::max<int64_t>(1, n * n)));
        double* q = Q ? static_cast<double*>(dQ.ensure(sizeof(double) * std::max<int64_t>(1, d * n))) : nullptr;
        slq::qr_factor_dev(ctx, y, d, n, n, d, r, nullptr, q, nullptr);
        SLQ_CUDA_CHECK(cudaMemcpyAsync(R, r, sizeof(double) * n * n, cudaMemcpyDeviceToHost, ctx->stream));
        if (Q) SLQ_CUDA_CHECK(cudaMemcpyAsync(Q, q, sizeof(double) * d * n, cudaMemcpyDeviceToHost, ctx->stream));
        SLQ_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    });
}

int slq_tri_inverse(slq_ctx* ctx, const double* R, int64_t n, double* M) {
    return guarded([&] {
        need(ctx && R && M, SLQ_INVALID_ARG, "tri_inverse: null argument");
        slq::DevBuf dR, dM;
        double* r = static_cast<double*>(dR.ensure(sizeof(double) * std::max<int64_t>(1, n * n)));
        double* mm = static_cast<double*>(dM.ensure(sizeof(double) * std::max<int64_t>(1, n * n)));
        SLQ_CUDA_CHECK(cudaMemcpyAsync(r, R, sizeof(double) * n * n, cudaMemcpyHostToDevice, ctx->stream));
        slq::tri_inverse_dev(ctx, r, n, mm, nullptr);
        SLQ_CUDA_CHECK(cudaMemcpyAsync(M, mm, sizeof(double) * n * n, cudaMemcpyDeviceToHost, ctx->stream));
        SLQ_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    });
}

int slq_build_preconditioner(slq_ctx* ctx, const double* Y, int64_t d, int64_t n, int64_t ldy, const double* Sb,
                             double* M, double* Q, double* x0, double* build_time) {
    return guarded([&] {
        need(ctx && Y && M, SLQ_INVALID_ARG, "build_preconditioner: null argument");
        if (d < n) slq::fail(SLQ_DIMENSION_MISMATCH, "householder_qr: need rows >= cols");
        need(ldy >= d, SLQ_INVALID_DIMS, "build_preconditioner: ldy < d");
        const bool with_sb = Sb != nullptr;
        double* Yaug = static_cast<double*>(ctx->ws.yaug.ensure(sizeof(double) * d * (n + 1)));
        SLQ_CUDA_CHECK(cudaMemcpy2DAsync(Yaug, sizeof(double) * d, Y, sizeof(double) * ldy, sizeof(double) * d, n,
                                         cudaMemcpyHostToDevice, ctx->stream));
        if (with_sb)
            SLQ_CUDA_CHECK(cudaMemcpyAsync(Yaug + d * n, Sb, sizeof(double) * d, cudaMemcpyHostToDevice, ctx->stream));
        slq::DevBuf dQ;
        double* q = Q ? static_cast<double*>(dQ.ensure(sizeof(double) * std::max<int64_t>(1, d * n))) : nullptr;
        PrecondBufs P = precond_bufs(ctx, n);
        Timer q0(ctx->stream), q1(ctx->stream), q2(ctx->stream), q3(ctx->stream);
        Timer* const qm[4] = {&q0, &q1, &q2, &q3};
        build_precond_dev(ctx, Yaug, d, n, with_sb, q, P, qm);
        SLQ_CUDA_CHECK(cudaMemcpyAsync(M, P.M, sizeof(double) * n * n, cudaMemcpyDeviceToHost, ctx->stream));
        if (Q) SLQ_CUDA_CHECK(cudaMemcpyAsync(Q, q, sizeof(double) * d * n, cudaMemcpyDeviceToHost, ctx->stream));
        if (x0 && with_sb) SLQ_CUDA_CHECK(cudaMemcpyAsync(x0, P.x0, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
        SLQ_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        if (build_time) *build_time = q2.since(q0);  // QR + inversion
    });
}

int slq_initial_guess(slq_ctx* ctx, const double* M, const double* Q, int64_t d, int64_t n, const double* Sb,
                      double* x0) {
    return guarded([&] {
        need(ctx && M && Q && Sb && x0, SLQ_INVALID_ARG, "initial_guess: null argument");
        slq::DevBuf dM, dQ, dv, dt;
        double* mm = static_cast<double*>(dM.ensure(sizeof(double) * std::max<int64_t>(1, 2 * n * n)));
        double* q = static_cast<double*>(dQ.ensure(sizeof(double) * std::max<int64_t>(1, d * n)));
        double* v = static_cast<double*>(dv.ensure(sizeof(double) * std::max<int64_t>(1, d)));
        double* t = static_cast<double*>(dt.ensure(sizeof(double) * std::max<int64_t>(1, 2 * n)));
        SLQ_CUDA_CHECK(cudaMemcpyAsync(mm, M, sizeof(double) * n * n, cudaMemcpyHostToDevice, ctx->stream));
        SLQ_CUDA_CHECK(cudaMemcpyAsync(q, Q, sizeof(double) * d * n, cudaMemcpyHostToDevice, ctx->stream));
        SLQ_CUDA_CHECK(cudaMemcpyAsync(v, Sb, sizeof(double) * d, cudaMemcpyHostToDevice, ctx->stream));
        if (n > 0) {
            gemv_t_kernel<<<static_cast<unsigned>(slq::ceil_div(n * 32, 256)), 256, 0, ctx->stream>>>(q, d, n, v, t);
            SLQ_LAUNCH_CHECK(ctx);
            transpose_square(ctx, mm, n, mm + n * n);
            slq::trmv_upper_dev(ctx, mm + n * n, n, t, t + n);
        }
        SLQ_CUDA_CHECK(cudaMemcpyAsync(x0, t + n, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
        SLQ_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    });
}

int slq_tri_upper_matvec(slq_ctx* ctx, const double* R, int64_t n, const double* x, double* y, int trans) {
    return guarded([&] {
        need(ctx && R && x && y, SLQ_INVALID_ARG, "tri_upper_matvec: null argument");
        slq::DevBuf dR, dv;
        double* r = static_cast<double*>(dR.ensure(sizeof(double) * std::max<int64_t>(1, 2 * n * n)));
        double* v = static_cast<double*>(dv.ensure(sizeof(double) * std::max<int64_t>(1, 2 * n)));
        SLQ_CUDA_CHECK(cudaMemcpyAsync(r, R, sizeof(double) * n * n, cudaMemcpyHostToDevice, ctx->stream));
        SLQ_CUDA_CHECK(cudaMemcpyAsync(v, x, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
        if (n > 0) {
            if (trans) {
                slq::trmv_upper_trans_dev(ctx, r, n, v, v + n);
            } else {
                transpose_square(ctx, r, n, r + n * n);
                slq::trmv_upper_dev(ctx, r + n * n, n, v, v + n);
            }
        }
        SLQ_CUDA_CHECK(cudaMemcpyAsync(y, v + n, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
        SLQ_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    });
}

namespace {
// y = A x / z = A^T y (+ ||y||^2) for the Op surface, host vectors in and out
void op_products(slq_ctx* ctx, const slq::PassOp& op, const double* x, double* y, const double* yin, double* z,
                 double* ynorm2) {
    const int64_t m = op.m, n = op.n;
    slq::DevBuf du, dn, dz;
    double* u = static_cast<double*>(du.ensure(sizeof(double) * (m + slq::kSparseRowPad)));
    double* v = static_cast<double*>(dn.ensure(sizeof(double) * (n + 8)));
    if (x) {
        SLQ_CUDA_CHECK(cudaMemcpyAsync(v, x, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
        slq::op_matvec_dev(ctx, op, v, u);
        SLQ_CUDA_CHECK(cudaMemcpyAsync(y, u, sizeof(double) * m, cudaMemcpyDeviceToHost, ctx->stream));
    } else {
        double* zz = static_cast<double*>(dz.ensure(sizeof(double) * (n + 1)));
        SLQ_CUDA_CHECK(cudaMemsetAsync(u, 0, sizeof(double) * (m + slq::kSparseRowPad), ctx->stream));
        SLQ_CUDA_CHECK(cudaMemcpyAsync(u, yin, sizeof(double) * m, cudaMemcpyHostToDevice, ctx->stream));
        slq::op_rmatvec_dev(ctx, op, u, zz, v);
        SLQ_CUDA_CHECK(cudaMemcpyAsync(z, zz, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
        if (ynorm2) SLQ_CUDA_CHECK(cudaMemcpyAsync(ynorm2, zz + n, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    }
    SLQ_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
}
}  // namespace

int slq_dense_matvec(slq_ctx* ctx, const slq_dense* A, const double* x, double* y) {
    return guarded([&] {
        need(ctx && A && (x || A->n == 0) && (y || A->m == 0), SLQ_INVALID_ARG, "dense_matvec: null argument");
        op_products(ctx, *slq::make_dense_op(ctx, A), x ? x : &kZero, y, nullptr, nullptr, nullptr);
    });
}

int slq_dense_rmatvec(slq_ctx* ctx, const slq_dense* A, const double* y, double* z, double* ynorm2) {
    return guarded([&] {
        need(ctx && A && (y || A->m == 0) && (z || A->n == 0), SLQ_INVALID_ARG, "dense_rmatvec: null argument");
        op_products(ctx, *slq::make_dense_op(ctx, A), nullptr, nullptr, y ? y : &kZero, z, ynorm2);
    });
}

int slq_sparse_matvec(slq_ctx* ctx, const slq_sparse* A, const double* x, double* y) {
    return guarded([&] {
        need(ctx && A && (x || A->n == 0) && (y || A->m == 0), SLQ_INVALID_ARG, "sparse_matvec: null argument");
        op_products(ctx, *slq::make_sparse_op(ctx, A), x ? x : &kZero, y, nullptr, nullptr, nullptr);
    });
}

int slq_sparse_rmatvec(slq_ctx* ctx, const slq_sparse* A, const double* y, double* z, double* ynorm2) {
    return guarded([&] {
        need(ctx && A && (y || A->m == 0) && (z || A->n == 0), SLQ_INVALID_ARG, "sparse_rmatvec: null argument");
        op_products(ctx, *slq::make_sparse_op(ctx, A), nullptr, nullptr, y ? y : &kZero, z, ynorm2);
    });
}

int slq_lsqr(slq_ctx* ctx, const slq_dense* A, const double* M, const double* b, const double* x0,
             const slq_solve_opts* opts_in, double* x_out, slq_report* report, double* residual_estimate,
             double* iterates_error, double* residual_true) {
    return guarded([&] {
        need(ctx && A && M && x0 && x_out, SLQ_INVALID_ARG, "lsqr: null argument");
        need(b != nullptr || A->has_b, SLQ_INVALID_ARG, "lsqr: no right-hand side");
        slq_solve_opts opts;
        if (opts_in) opts = *opts_in;
        else slq_solve_opts_default(&opts);
        const int64_t n = A->n, m = A->m;
        PrecondBufs P = precond_bufs(ctx, n);
        SLQ_CUDA_CHECK(cudaMemcpyAsync(P.M, M, sizeof(double) * n * n, cudaMemcpyHostToDevice, ctx->stream));
        transpose_square(ctx, P.M, n, P.Mt);
        SLQ_CUDA_CHECK(cudaMemcpyAsync(P.x0, x0, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
        slq::DevBuf db, dx;
        double* bd = nullptr;
        if (b) {
            bd = static_cast<double*>(db.ensure(sizeof(double) * std::max<int64_t>(1, m)));
            SLQ_CUDA_CHECK(cudaMemcpyAsync(bd, b, sizeof(double) * m, cudaMemcpyHostToDevice, ctx->stream));
        }
        double* x = static_cast<double*>(dx.ensure(sizeof(double) * (n + 8)));
        slq::LsqrOut lo;
        const auto h0 = std::chrono::steady_clock::now();
        slq::lsqr_dev(ctx, *slq::make_dense_op(ctx, A), bd, P.M, P.Mt, P.x0, x, opts, residual_estimate, iterates_error,
                      residual_true, lo);
        SLQ_CUDA_CHECK(cudaMemcpy(x_out, x, sizeof(double) * n, cudaMemcpyDeviceToHost));
        lo.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - h0).count();
        fill_report(report, lo);
    });
}

int slq_solve(slq_ctx* ctx, const slq_dense* A, int64_t d, int64_t zeta, uint64_t seed, const slq_solve_opts* opts,
              double* x_out, slq_report* report, slq_phase_times* times, double* residual_estimate) {
    if (!ctx || !A) {
        g_last_error = "solve: null handle";
        return SLQ_INVALID_ARG;
    }
    if (!A->has_b) {
        g_last_error = "solve: the matrix has no right-hand side (slq_dense_set_rhs)";
        return SLQ_INVALID_ARG;
    }
    return run_solve(ctx, dense_operand(ctx, A), d, zeta, seed, opts, x_out, report, times, residual_estimate);
}

int slq_solve_sparse(slq_ctx* ctx, const slq_sparse* A, int64_t d, int64_t zeta, uint64_t seed,
                     const slq_solve_opts* opts, double* x_out, slq_report* report, slq_phase_times* times,
                     double* residual_estimate) {
    if (!ctx || !A) {
        g_last_error = "solve_sparse: null handle";
        return SLQ_INVALID_ARG;
    }
    if (!A->b) {
        g_last_error = "solve_sparse: the matrix has no right-hand side (slq_sparse_set_rhs)";
        return SLQ_INVALID_ARG;
    }
    return run_solve(ctx, sparse_operand(ctx, A), d, zeta, seed, opts, x_out, report, times, residual_estimate);
}

int slq_sparse_upload_csc(slq_ctx* ctx, int64_t m, int64_t n, const int64_t* col_pointers, const int64_t* row_indices,
                          const double* values, const double* b, int64_t row_begin, slq_sparse** out) {
    return guarded([&] {
        need(ctx && out && col_pointers, SLQ_INVALID_ARG, "sparse_upload_csc: null argument");
        need(m >= 0 && n >= 0 && row_begin >= 0, SLQ_INVALID_DIMS, "sparse_upload_csc: bad shape");
        need(n < (int64_t(1) << 31), SLQ_UNSUPPORTED, "sparse_upload_csc: n >= 2^31");
        const int64_t nnz = col_pointers[n];
        for (int64_t e = 0; e < nnz; ++e)
            if (row_indices[e] < 0 || row_indices[e] >= m) slq::fail(SLQ_INVALID_ARG, "sparse_upload_csc: row index out of range");
        SLQ_CUDA_CHECK(cudaSetDevice(ctx->device));
        auto* A = new slq_sparse();
        A->ctx = ctx;
        A->m = m;
        A->n = n;
        A->nnz = nnz;
        A->row_begin = row_begin;
        try {
            slq::sparse_alloc(ctx, A, true);
            slq::sparse_from_csc(ctx, A, col_pointers, row_indices, values);
            if (b) SLQ_CUDA_CHECK(cudaMemcpy(A->b, b, sizeof(double) * m, cudaMemcpyHostToDevice));
            else {
                cudaFree(A->b);
                A->b = nullptr;
            }
        } catch (...) {
            slq::sparse_free(A);
            delete A;
            throw;
        }
        *out = A;
    });
}

int slq_sparse_create_csr(slq_ctx* ctx, int64_t m, int64_t n, int64_t nnz, int64_t row_begin, int with_b,
                          slq_sparse** out, int64_t** row_ptr, int32_t** col_idx, double** values, double** b) {
    return guarded([&] {
        need(ctx && out, SLQ_INVALID_ARG, "sparse_create_csr: null argument");
        need(m >= 0 && n >= 0 && nnz >= 0 && row_begin >= 0, SLQ_INVALID_DIMS, "sparse_create_csr: bad shape");
        SLQ_CUDA_CHECK(cudaSetDevice(ctx->device));
        auto* A = new slq_sparse();
        A->ctx = ctx;
        A->m = m;
        A->n = n;
        A->nnz = nnz;
        A->row_begin = row_begin;
        try {
            slq::sparse_alloc(ctx, A, with_b != 0);
            SLQ_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        } catch (...) {
            slq::sparse_free(A);
            delete A;
            throw;
        }
        *out = A;
        if (row_ptr) *row_ptr = A->rowptr;
        if (col_idx) *col_idx = A->colidx;
        if (values) *values = A->vals;
        if (b) *b = A->b;
    });
}

int slq_sparse_fill_random(slq_sparse* A, int64_t nnz_per_row, uint64_t seed, const double* col_scale) {
    return guarded([&] {
        need(A != nullptr, SLQ_INVALID_ARG, "null matrix");
        need(A->nnz == A->m * nnz_per_row, SLQ_DIMENSION_MISMATCH, "sparse_fill_random: nnz != m * nnz_per_row");
        slq_ctx* ctx = A->ctx;
        if (A->t_pending) {  // a transposed-copy build may still be reading the CSR
            SLQ_CUDA_CHECK(cudaStreamWaitEvent(ctx->stream, A->t_ready, 0));
            A->t_pending = false;
        }
        slq::DevBuf sc;
        double* dsc = nullptr;
        if (col_scale) {
            dsc = static_cast<double*>(sc.ensure(sizeof(double) * std::max<int64_t>(1, A->n)));
            SLQ_CUDA_CHECK(cudaMemcpyAsync(dsc, col_scale, sizeof(double) * A->n, cudaMemcpyHostToDevice, ctx->stream));
        }
        slq::generate_sparse_rows_dev(ctx, A->n, nnz_per_row, seed, A->row_begin, A->m, dsc, A->rowptr, A->colidx,
                                      A->vals);
        A->t_valid = false;
        A->s_valid = false;
    });
}

int slq_sparse_prepare(slq_ctx* ctx, slq_sparse* A) {
    return guarded([&] {
        need(ctx && A, SLQ_INVALID_ARG, "sparse_prepare: null argument");
        SLQ_CUDA_CHECK(cudaSetDevice(ctx->device));
        if (A->t_pending) SLQ_CUDA_CHECK(cudaStreamWaitEvent(ctx->stream, A->t_ready, 0));
        A->t_pending = false;
        A->t_valid = false;
        A->s_valid = false;  // slab tables of the sketch gather: rebuilt on next use
        slq::prepare_two_pass(ctx, A);
        SLQ_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    });
}

int slq_sparse_set_rhs(slq_sparse* A, const double* b) {
    return guarded([&] {
        need(A != nullptr, SLQ_INVALID_ARG, "null matrix");
        if (!A->b) {
            SLQ_CUDA_CHECK(cudaMalloc(&A->b, sizeof(double) * (A->m + slq::kSparseRowPad)));
            SLQ_CUDA_CHECK(cudaMemset(A->b, 0, sizeof(double) * (A->m + slq::kSparseRowPad)));
        }
        if (b) SLQ_CUDA_CHECK(cudaMemcpy(A->b, b, sizeof(double) * A->m, cudaMemcpyHostToDevice));
    });
}

int slq_sparse_free(slq_sparse* A) {
    return guarded([&] {
        if (!A) return;
        slq::sparse_free(A);  // cudaFree waits for pending device work; A->ctx may be gone
        delete A;
    });
}

int slq_sketch_apply_sparse(slq_ctx* ctx, const slq_sparse* A, int64_t d, int64_t zeta, uint64_t seed, double* Y,
                            double* Sb) {
    return guarded([&] {
        need(ctx && A, SLQ_INVALID_ARG, "sketch_apply_sparse: null handle");
        const int64_t n = A->n;
        double* Yaug = static_cast<double*>(ctx->ws.yaug.ensure(sizeof(double) * d * (n + 1)));
        slq::sketch_apply_sparse_dev(ctx, A, d, zeta, seed, Yaug);
        slq::allreduce_sum(ctx, Yaug, d * (n + 1));
        if (Y) SLQ_CUDA_CHECK(cudaMemcpyAsync(Y, Yaug, sizeof(double) * d * n, cudaMemcpyDeviceToHost, ctx->stream));
        if (Sb) SLQ_CUDA_CHECK(cudaMemcpyAsync(Sb, Yaug + d * n, sizeof(double) * d, cudaMemcpyDeviceToHost, ctx->stream));
        SLQ_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    });
}

int slq_spmm_csc_csc(slq_ctx* ctx, int64_t d, int64_t m, const int64_t* s_rows, const double* s_vals,
                     const int64_t* s_colptr, int64_t n, const int64_t* a_colptr, const int64_t* a_rows,
                     const double* a_vals, double* Y) {
    return guarded([&] {
        need(ctx && s_colptr && a_colptr && Y, SLQ_INVALID_ARG, "spmm_csc_csc: null argument");
        const int64_t snnz = s_colptr[m];
        const int64_t annz = a_colptr[n];
        need(s_colptr[0] == 0 && snnz >= 0 && a_colptr[0] == 0 && annz >= 0, SLQ_INVALID_ARG,
             "spmm_csc_csc: bad col_pointers");
        slq::DevBuf drows, dvals, dcp, dcomp, dY;
        int64_t* r = static_cast<int64_t*>(drows.ensure(sizeof(int64_t) * std::max<int64_t>(1, snnz)));
        double* v = static_cast<double*>(dvals.ensure(sizeof(double) * std::max<int64_t>(1, snnz)));
        int64_t* cp = static_cast<int64_t*>(dcp.ensure(sizeof(int64_t) * (m + 1)));
        double* Yd = static_cast<double*>(dY.ensure(sizeof(double) * std::max<int64_t>(1, d * (n + 1))));
        if (snnz > 0) {
            SLQ_CUDA_CHECK(cudaMemcpyAsync(r, s_rows, sizeof(int64_t) * snnz, cudaMemcpyHostToDevice, ctx->stream));
            SLQ_CUDA_CHECK(cudaMemcpyAsync(v, s_vals, sizeof(double) * snnz, cudaMemcpyHostToDevice, ctx->stream));
        }
        SLQ_CUDA_CHECK(cudaMemcpyAsync(cp, s_colptr, sizeof(int64_t) * (m + 1), cudaMemcpyHostToDevice, ctx->stream));
        const slq::SpmmCheck chk = slq::csc_check_dev(ctx, r, v, snnz, d);
        need(!chk.row_out_of_range, SLQ_INVALID_ARG, "spmm: row index out of range");
        if (chk.mixed_magnitudes) {
            slq::DevBuf dacp, dar, dav;
            int64_t* acp = static_cast<int64_t*>(dacp.ensure(sizeof(int64_t) * (n + 1)));
            int64_t* ar = static_cast<int64_t*>(dar.ensure(sizeof(int64_t) * std::max<int64_t>(1, annz)));
            double* av = static_cast<double*>(dav.ensure(sizeof(double) * std::max<int64_t>(1, annz)));
            SLQ_CUDA_CHECK(cudaMemcpyAsync(acp, a_colptr, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, ctx->stream));
            if (annz > 0) {
                SLQ_CUDA_CHECK(cudaMemcpyAsync(ar, a_rows, sizeof(int64_t) * annz, cudaMemcpyHostToDevice, ctx->stream));
                SLQ_CUDA_CHECK(cudaMemcpyAsync(av, a_vals, sizeof(double) * annz, cudaMemcpyHostToDevice, ctx->stream));
            }
            slq::spmm_general_dev(ctx, d, m, snnz, r, v, cp, n, nullptr, 0, acp, ar, av, Yd);
        } else {
            slq_sparse* As = nullptr;
            int st = slq_sparse_upload_csc(ctx, m, n, a_colptr, a_rows, a_vals, nullptr, 0, &As);
            if (st != SLQ_OK) slq::fail(st, g_last_error);
            struct Free {
                slq_sparse* p;
                ~Free() { slq_sparse_free(p); }
            } fr{As};
            const double val = snnz > 0 ? std::fabs(s_vals[0]) : 0.0;
            int64_t zmax = 1;
            for (int64_t j = 0; j < m; ++j) zmax = std::max(zmax, s_colptr[j + 1] - s_colptr[j]);
            uint32_t* comp = static_cast<uint32_t*>(dcomp.ensure(sizeof(uint32_t) * std::max<int64_t>(1, snnz)));
            if (snnz > 0) {
                csc_to_compact_kernel<<<static_cast<unsigned>(slq::ceil_div(snnz, 256)), 256, 0, ctx->stream>>>(r, v, snnz,
                                                                                                             comp);
                SLQ_LAUNCH_CHECK(ctx);
            }
            slq::sketch_apply_sparse_compact_dev(ctx, As, d, comp, cp, zmax, val, Yd);
        }
        if (d * n > 0)
            SLQ_CUDA_CHECK(cudaMemcpyAsync(Y, Yd, sizeof(double) * d * n, cudaMemcpyDeviceToHost, ctx->stream));
        SLQ_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    });
}

int slq_lsqr_sparse(slq_ctx* ctx, const slq_sparse* A, const double* M, const double* b, const double* x0,
                    const slq_solve_opts* opts_in, double* x_out, slq_report* report, double* residual_estimate,
                    double* iterates_error, double* residual_true) {
    return guarded([&] {
        need(ctx && A && M && x0 && x_out, SLQ_INVALID_ARG, "lsqr_sparse: null argument");
        need(b != nullptr || A->b != nullptr, SLQ_INVALID_ARG, "lsqr_sparse: no right-hand side");
        slq_solve_opts opts;
        if (opts_in) opts = *opts_in;
        else slq_solve_opts_default(&opts);
        const int64_t n = A->n, m = A->m;
        PrecondBufs P = precond_bufs(ctx, n);
        SLQ_CUDA_CHECK(cudaMemcpyAsync(P.M, M, sizeof(double) * n * n, cudaMemcpyHostToDevice, ctx->stream));
        transpose_square(ctx, P.M, n, P.Mt);
        SLQ_CUDA_CHECK(cudaMemcpyAsync(P.x0, x0, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
        slq::DevBuf db, dx;
        double* bd = nullptr;
        if (b) {
            bd = static_cast<double*>(db.ensure(sizeof(double) * (m + slq::kSparseRowPad)));
            SLQ_CUDA_CHECK(cudaMemsetAsync(bd, 0, sizeof(double) * (m + slq::kSparseRowPad), ctx->stream));
            SLQ_CUDA_CHECK(cudaMemcpyAsync(bd, b, sizeof(double) * m, cudaMemcpyHostToDevice, ctx->stream));
        }
        double* x = static_cast<double*>(dx.ensure(sizeof(double) * (n + 8)));
        slq::LsqrOut lo;
        const auto h0 = std::chrono::steady_clock::now();
        slq::lsqr_dev(ctx, *slq::make_sparse_op(ctx, A, true), bd, P.M, P.Mt, P.x0, x, opts, residual_estimate,
                      iterates_error, residual_true, lo);
        SLQ_CUDA_CHECK(cudaMemcpy(x_out, x, sizeof(double) * n, cudaMemcpyDeviceToHost));
        lo.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - h0).count();
        fill_report(report, lo);
    });
}

int slq_hbm_params(double eta, slq_gradient_params* out) {
    return guarded([&] {
        need(out != nullptr, SLQ_INVALID_ARG, "hbm_params: null output");
        need(eta >= 0.0 && eta < 1.0, SLQ_INVALID_DISTORTION, "hbm_params: need 0 <= eta_hat < 1");
        const double e2 = eta * eta;
        *out = slq_gradient_params{(1.0 - e2) * (1.0 - e2), e2, eta};
    });
}

int slq_gd_params(double eta, slq_gradient_params* out) {
    return guarded([&] {
        need(out != nullptr, SLQ_INVALID_ARG, "gd_params: null output");
        need(eta >= 0.0 && eta < 1.0, SLQ_INVALID_DISTORTION, "gd_step_size: need 0 <= eta_hat < 1");
        const double e2 = eta * eta;
        *out = slq_gradient_params{(1.0 - e2) * (1.0 - e2) / (1.0 + e2), 0.0, eta};
    });
}

int slq_gradient_descent_hbm(slq_ctx* ctx, const slq_dense* A, const double* M, const double* b, const double* x0,
                             const slq_gradient_params* params, const slq_solve_opts* opts, double* x_out,
                             slq_report* report, double* residual_estimate, double* iterates_error,
                             double* residual_true) {
    return guarded([&] {
        need(ctx && A && M && x0 && x_out && params, SLQ_INVALID_ARG, "gradient_descent_hbm: null argument");
        need(b != nullptr || A->has_b, SLQ_INVALID_ARG, "gradient_descent_hbm: no right-hand side");
        gd_common(ctx, A->m, A->n, M, b, x0, params, opts, x_out, report, residual_estimate, iterates_error,
                  residual_true, 0, [&] { return slq::make_dense_op(ctx, A); });
    });
}

int slq_gradient_descent_hbm_sparse(slq_ctx* ctx, const slq_sparse* A, const double* M, const double* b,
                                    const double* x0, const slq_gradient_params* params, const slq_solve_opts* opts,
                                    double* x_out, slq_report* report, double* residual_estimate,
                                    double* iterates_error, double* residual_true) {
    return guarded([&] {
        need(ctx && A && M && x0 && x_out && params, SLQ_INVALID_ARG, "gradient_descent_hbm_sparse: null argument");
        need(b != nullptr || A->b != nullptr, SLQ_INVALID_ARG, "gradient_descent_hbm_sparse: no right-hand side");
        gd_common(ctx, A->m, A->n, M, b, x0, params, opts, x_out, report, residual_estimate, iterates_error,
                  residual_true, slq::kSparseRowPad, [&] { return slq::make_sparse_op(ctx, A, true); });
    });
}

int slq_time_kernels(slq_ctx* ctx, const slq_dense* A, int64_t d, int64_t zeta, uint64_t seed, int reps,
                     double* out) {
    return guarded([&] {
        need(ctx && A && out, SLQ_INVALID_ARG, "time_kernels: null argument");
        const int64_t n = A->n, m = A->m;
        out[0] = slq::time_fused_pass(ctx, *slq::make_dense_op(ctx, A), reps);
        slq::Workspace& ws = ctx->ws;
        double* Yaug = static_cast<double*>(ws.yaug.ensure(sizeof(double) * d * (n + 1)));
        uint32_t* compact = static_cast<uint32_t*>(ws.compact.ensure(sizeof(uint32_t) * std::max<int64_t>(1, m * zeta)));
        Timer a0(ctx->stream);
        slq::generate_sparse_sign_dev(ctx, d, zeta, seed, A->row_begin, m, compact, nullptr, nullptr, nullptr, nullptr);
        Timer a1(ctx->stream);
        slq::sketch_apply_compact_dev(ctx, A, d, compact, nullptr, zeta, 1.0 / std::sqrt(static_cast<double>(zeta)),
                                      false, Yaug);
        Timer a2(ctx->stream);
        PrecondBufs P = precond_bufs(ctx, n);
        build_precond_dev(ctx, Yaug, d, n, true, nullptr, P, nullptr);
        Timer a3(ctx->stream);
        out[1] = a2.since(a0);
        out[2] = a1.since(a0);
        out[3] = a3.since(a2);
    });
}

int slq_time_sparse_pass(slq_ctx* ctx, const slq_sparse* A, int reps, double* seconds) {
    return guarded([&] {
        need(ctx && A && seconds, SLQ_INVALID_ARG, "time_sparse_pass: null argument");
        SLQ_CUDA_CHECK(cudaSetDevice(ctx->device));
        *seconds = slq::time_fused_pass(ctx, *slq::make_sparse_op(ctx, A, true), reps);
    });
}

int slq_solve_host(slq_ctx* ctx, const double* A, int64_t m, int64_t n, int64_t lda, const double* b,
                   int64_t row_begin, int64_t d, int64_t zeta, uint64_t seed, const slq_solve_opts* opts,
                   double* x_out, slq_report* report, slq_phase_times* times, double* residual_estimate) {
    // The device copy of A lives in a context-owned, grow-only buffer, so
    // repeated host solves neither cudaMalloc nor cudaFree 8*m*ld bytes (a
    // 32 GB free/alloc pair costs tens to hundreds of milliseconds).
    slq_dense Ad;
    const int st0 = guarded([&] {
        need(ctx != nullptr, SLQ_INVALID_ARG, "solve_host: null ctx");
        need(m >= 0 && n >= 0 && lda >= m && row_begin >= 0, SLQ_INVALID_DIMS, "solve_host: bad shape");
        need(A != nullptr || m * n == 0, SLQ_INVALID_ARG, "solve_host: null A");
        need(b != nullptr, SLQ_INVALID_ARG, "solve_host: null b");
        SLQ_CUDA_CHECK(cudaSetDevice(ctx->device));
        Ad.ctx = ctx;
        Ad.m = m;
        Ad.n = n;
        Ad.ld = slq::dense_ld(n);
        Ad.row_begin = row_begin;
        Ad.owned = false;
        Ad.has_b = true;
        Ad.A = static_cast<double*>(ctx->ws.host_A.ensure(sizeof(double) * std::max<int64_t>(1, m * Ad.ld)));
    });
    if (st0 != SLQ_OK) return st0;
    // the upload happens inside the sketch phase, overlapped with it
    return run_solve(ctx, host_dense_operand(ctx, &Ad, A, lda, b), d, zeta, seed, opts, x_out, report, times,
                     residual_estimate);
}

}  // extern "C"

// ---------------------------------------------------------- guard bands

namespace slq {
namespace guard {
namespace {
struct Rec {
    void* base;
    size_t ub;
};
std::mutex g_mu;
std::unordered_map<const void*, Rec>& live() {
    static auto* m = new std::unordered_map<const void*, Rec>();  // never destroyed: DevBufs may outlive statics
    return *m;
}
int64_t g_bad = 0;

bool band_intact(const void* dev) {
    std::vector<unsigned char> h(kBand);
    if (cudaMemcpy(h.data(), dev, kBand, cudaMemcpyDeviceToHost) != cudaSuccess) return true;  // context gone
    for (unsigned char c : h)
        if (c != 0xA5) return false;
    return true;
}
bool intact(const Rec& r) {
    return band_intact(r.base) && band_intact(static_cast<const char*>(r.base) + kBand + r.ub);
}
}  // namespace

bool enabled() {
    static const bool on = slq_env_flag("SLQ_GUARD");
    return on;
}

void on_alloc(void* base, size_t ub, const void* owner) {
    SLQ_CUDA_CHECK(cudaMemset(base, 0xA5, kBand));
    SLQ_CUDA_CHECK(cudaMemset(static_cast<char*>(base) + kBand + ub, 0xA5, kBand));
    SLQ_CUDA_CHECK(cudaDeviceSynchronize());
    std::lock_guard<std::mutex> lk(g_mu);
    live()[owner] = Rec{base, ub};
}

void on_release(void* base, const void* owner) {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = live().find(owner);
    if (it == live().end() || it->second.base != base) return;
    if (cudaDeviceSynchronize() == cudaSuccess && !intact(it->second)) {
        ++g_bad;
        std::fprintf(stderr, "[slq] guard band overwritten around a %zu-byte device buffer\n", it->second.ub);
    }
    live().erase(it);
}
}  // namespace guard
}  // namespace slq

int slq_debug_check_guards(int64_t* corrupted) {
    return guarded([&] {
        need(corrupted != nullptr, SLQ_INVALID_ARG, "debug_check_guards: null argument");
        SLQ_CUDA_CHECK(cudaDeviceSynchronize());
        std::lock_guard<std::mutex> lk(slq::guard::g_mu);
        int64_t bad = 0;
        for (auto& kv : slq::guard::live())
            if (!slq::guard::intact(kv.second)) ++bad;
        *corrupted = bad + slq::guard::g_bad;
    });
}

namespace {
__global__ void guard_selftest_kernel(double* p, int64_t i) { p[i] = 1.0; }
}  // namespace

int slq_debug_guard_selftest(int* detected) {
    return guarded([&] {
        need(detected != nullptr, SLQ_INVALID_ARG, "debug_guard_selftest: null argument");
        need(slq::guard::enabled(), SLQ_INVALID_ARG, "debug_guard_selftest: needs SLQ_GUARD=1");
        int64_t before = 0, after = 0;
        SLQ_CUDA_CHECK(cudaDeviceSynchronize());
        {
            std::lock_guard<std::mutex> lk(slq::guard::g_mu);
            before = slq::guard::g_bad;
        }
        {
            slq::DevBuf b;
            double* p = static_cast<double*>(b.ensure(1000 * sizeof(double)));
            guard_selftest_kernel<<<1, 1>>>(p, 1024 + 3);  // one element past the 8 KB rounding: in the band
            SLQ_CUDA_CHECK(cudaGetLastError());
        }  // release checks the bands
        {
            std::lock_guard<std::mutex> lk(slq::guard::g_mu);
            after = slq::guard::g_bad;
            slq::guard::g_bad = before;  // the planted corruption does not count against the process
        }
        *detected = after > before ? 1 : 0;
    });
}
