// common.cuh -- shared host/device plumbing for the sm_100a solver library.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "slq_b200.h"

namespace slq {

// Exception carrying an slq_status; converted to a return code at the C-ABI.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& what) : std::runtime_error(what), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& what) { throw Error(code, what); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess) {
        std::string msg = std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" +
                          std::to_string(line) + ")";
        fail(e == cudaErrorMemoryAllocation ? SLQ_OOM : SLQ_CUDA, msg);
    }
}
#define SLQ_CUDA_CHECK(x) ::slq::cuda_check((x), #x, __FILE__, __LINE__)
#define SLQ_LAUNCH_CHECK(ctx)                                        \
    do {                                                             \
        ::slq::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__); \
        (ctx)->launches++;                                           \
    } while (0)

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// Diagnostic switches (environment variables set to a non-empty value other than "0").
inline bool slq_env_flag(const char* name) {
    const char* v = std::getenv(name);
    return v && v[0] && !(v[0] == '0' && v[1] == 0);
}

// Guard-band mode (SLQ_GUARD=1, diagnostics): every DevBuf allocation gets
// 64 KB bands before and after it filled with 0xA5; the bands are verified
// when the buffer is released and on slq_debug_check_guards().  Catches
// out-of-bounds device writes into the library's scratch (compute-sanitizer
// is not available on every GPU pool).
namespace guard {
constexpr size_t kBand = 64 * 1024;
bool enabled();
void on_alloc(void* base, size_t user_bytes, const void* owner);
void on_release(void* base, const void* owner);  // checks, then forgets
}  // namespace guard

// Device buffer with RAII; grow-only reuse via ensure().
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) {
            if (base_ != p) {  // guarded allocation
                guard::on_release(base_, this);
                cudaFree(base_);
            } else {
                cudaFree(p);
            }
        }
        p = base_ = nullptr;
        bytes = 0;
    }
    void* ensure(size_t b) {
        if (b <= bytes && p) return p;
        release();
        if (b == 0) b = 16;
        if (guard::enabled()) {
            const size_t ub = (b + 255) & ~size_t(255);
            SLQ_CUDA_CHECK(cudaMalloc(&base_, ub + 2 * guard::kBand));
            p = static_cast<char*>(base_) + guard::kBand;
            guard::on_alloc(base_, ub, this);
        } else {
            SLQ_CUDA_CHECK(cudaMalloc(&p, b));
            base_ = p;
        }
        bytes = b;
        return p;
    }
    template <class T>
    T* as() const { return static_cast<T*>(p); }

private:
    void* base_ = nullptr;
};

// Per-context scratch, grow-only (sizes at C3 in DESIGN.md).
struct Workspace {
    DevBuf compact;      // sketch entries, u32 (row | neg << 31), column order
    DevBuf chunk_ptr;    // per-chunk row pointers (u16)
    DevBuf chunk_ent;    // per-chunk sorted entries (u16: k_local << 1 | neg)
    DevBuf tile_ent;     // per-(chunk, row block) tile-grouped entries of the DMMA gather
    DevBuf ypart;        // sketch partials [nsplit][ld][d]
    DevBuf yaug;         // Y_aug = [S A | S b], d x (n+1) column-major
    DevBuf flags;        // small device counters / error flags
    DevBuf staging[2];   // upload staging
    DevBuf qr_t, qr_w, qr_w2, qr_cnt, qr_cnt2, qr_q, qr_misc;
    DevBuf lsqr_vec, lsqr_part, lsqr_state, lsqr_u;
    DevBuf mats;         // M, Mt
    DevBuf xbuf;         // solution vector
    DevBuf tmp;
    DevBuf host_A;       // device copy of A for slq_solve_host (kept across calls)
    DevBuf st_ptr, st_cnt, st_scan;  // sparse sketch: S^T row pointers, counts, scan scratch
};

}  // namespace slq

// Opaque handles of the C-ABI (defined here so every translation unit agrees).
struct slq_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int num_sms = 148;
    int64_t launches = 0;
    slq::Workspace ws;
    // multi-GPU (NCCL communicator stored as void* to keep nccl.h local to comm.cu)
    void* comm = nullptr;
    slq_host_comm host_comm{};     // caller-provided host collectives (instead of NCCL)
    double* host_stage = nullptr;  // pinned staging for host collectives
    int64_t host_stage_n = 0;
    int rank = 0;
    int nranks = 1;
    int64_t nccl_calls = 0;
    // cached LSQR iteration graph (rebuilt when any captured pointer / size changes)
    cudaGraphExec_t lsqr_exec = nullptr;
    std::vector<uint64_t> lsqr_key;
    // QR look-ahead streams (panel + narrow update / wide update) and events
    cudaStream_t qr_hi = nullptr, qr_lo = nullptr;
    cudaEvent_t qr_ev[3] = {nullptr, nullptr, nullptr};
    // cached QR panel schedules (one CUDA graph per shape / buffer set, captured
    // on the second solve that uses it: the first sizes the workspace)
    struct QrGraph {
        std::vector<uint64_t> key;
        cudaGraphExec_t exec = nullptr;
        int64_t launches = 0;
    };
    std::vector<QrGraph> qr_graphs;
    int* lsqr_hdone = nullptr;            // pinned done-flag mirror (2 ints)
    int64_t lsqr_live_m = -1, lsqr_live_n = -1;  // shape whose LSQR vectors the workspace holds
    // Inside slq_solve: error conditions found on the device (rank-deficient
    // sketch, zero diagonal of R, a sketch bucket overflow) are recorded in
    // this device word instead of being read back mid-solve; the solve checks
    // it once at the end (and broadcasts it with M on multiple GPUs).
    double* defer_status = nullptr;
    bool force_row_gather = false;  // rerun after a K2d bucket overflow
    cudaEvent_t lsqr_ev[2] = {nullptr, nullptr};
    // side stream for work that overlaps the sketch (the sparse operator's
    // transposed-copy build); aux_ev[0]: main -> aux (the join back is the
    // matrix's own event, slq_sparse::t_ready)
    cudaStream_t aux = nullptr;
    cudaEvent_t aux_ev[2] = {nullptr, nullptr};
};

struct slq_dense {
    slq_ctx* ctx = nullptr;
    double* A = nullptr;  // row-major, element (i, j) at A[i*ld + j]; column n holds b
    int64_t m = 0;        // rows of this block
    int64_t n = 0;
    int64_t ld = 0;
    int64_t row_begin = 0;  // global id of row 0 (sketch column key)
    bool owned = false;
    bool has_b = false;
};

// Sparse row block in CSR (device).  Arrays carry slack past their logical
// end (colidx / vals: +4 entries, rowptr: +2, b: +kSparseRowPad) so bulk
// copies can round their ranges to 16-byte boundaries.
struct slq_sparse {
    slq_ctx* ctx = nullptr;
    int64_t m = 0, n = 0, nnz = 0;
    int64_t row_begin = 0;
    int64_t* rowptr = nullptr;  // m + 1 (+2 slack)
    int32_t* colidx = nullptr;  // nnz (+4 slack)
    double* vals = nullptr;     // nnz (+4 slack)
    double* b = nullptr;        // m (+ slack) right-hand side rows, may be null
    bool owned = true;
    // row-blocked CSC copy for the two-pass LSQR operator (sparse.cu), built
    // on the first solve and kept with the matrix; invalidated by the entry
    // points that rewrite the CSR (slq_sparse_prepare rebuilds it)
    uint32_t* t_blkcol = nullptr;  // [nblk][n + 1] column starts per row block
    uint16_t* t_crow = nullptr;    // [nnz] row offset within the block
    double* t_cval = nullptr;      // [nnz]
    double* t_uscr = nullptr;      // [m + pad] u_hat scratch for passes that do not keep it
    uint16_t* t_col16 = nullptr;   // [nnz + pad] the CSR's column indices as u16 (n < 65536)
    int64_t t_nblk = 0;
    bool t_valid = false;
    bool t_pending = false;        // built on a side stream; nobody has waited for it yet
    cudaEvent_t t_ready = nullptr; // recorded after the side-stream build
    // per-row column-slab segments for the sparse sketch gather ([m][S] per
    // slab geometry (S slabs of w columns), sparse.cu slab_ptr_kernel): built on
    // first use of a geometry and then immutable (a sketch of another d on
    // another stream gets its own table; `ready` orders the build before every
    // use); dropped when the CSR is rewritten (s_valid = false)
    struct SlabTable {
        uint64_t* p = nullptr;
        int S = 0, w = 0;
        cudaEvent_t ready = nullptr;
    };
    static constexpr int kSlabTables = 4;
    SlabTable s_tab[kSlabTables];
    int s_ntab = 0;
    bool s_valid = false;
};

namespace slq {

constexpr int64_t kSparseRowPad = 256;

// a communicator of either kind is attached (collectives are issued)
inline bool has_comm(const slq_ctx* c) { return c->comm != nullptr || c->host_comm.allreduce_sum != nullptr; }

// Internal (non-C-ABI) device status: a K2d bucket overflowed; the solve is
// redone with the register gather.
constexpr int kStatusSketchOverflow = 1000;

// Record `code` in ctx->defer_status (first error wins) when the device int
// `flag` meets the condition: kCondNonzero (flag[0] != 0), kCondNotBig
// (flag[0] != INT_MAX), kCondAny2 (flag[0] | flag[1]).  Stream-ordered, no sync.
enum DeferCond : int { kCondNonzero = 0, kCondNotBig = 1, kCondAny2 = 2 };
void defer_status_dev(slq_ctx* ctx, const int* flag, int cond, int code);

// Row stride of the device layout: [A | b | zero pad], 32-byte aligned rows.
inline int64_t dense_ld(int64_t n) { return round_up(n + 1, 4); }

}  // namespace slq
