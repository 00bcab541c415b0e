// sparse.cu -- the sparse-A path (BASELINE config C4).
//
// Replaces sketch.hpp:298 apply(SparseSignSketch, CscMatrix) ->
// csc_matrix.hpp:123-136 spmm(csc, csc), csc_matrix.hpp:71-96
// matvec / rmatvec over CSC, and lsqr.hpp:198-212 (the CscMatrix overloads:
// SerialOperator<CscMatrix> / DistOperator<CscMatrix>).
//
// Device layout: CSR row blocks (int64 row pointers, int32 columns, fp64
// values) -- rows are the partitioned dimension (distsim.hpp:235-246) and the
// LSQR pass streams them.
//
//   K2s  Y_aug = S [A b]: the chunk-CSR of the sketch (sketch.cu) is merged
//        into the CSR of S^T's rows (entries of Y row r in ascending k); one
//        warp per Y row keeps the row (n+1 doubles) in shared memory and adds
//        s * A[k, :] for its entries in ascending k -- the reference's
//        accumulation order (bit-identical), no atomics.
//   K4s  one pass per LSQR iteration: a warp takes quads of 4 rows, loads
//        their column indices and values straight into registers (three quads
//        in flight), computes u_hat = A_i p + c u_i (p in shared memory) and
//        scatters z += A_i^T u_hat into a warp-private copy of z in shared
//        memory (column indices within a row are distinct: no races, no
//        atomics); the copies are summed in a fixed order at the end.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <string>
#include <vector>

#include "lsqr.cuh"
#include "ptx.cuh"
#include "sketch.cuh"
#include "sparse.cuh"

namespace slq {

namespace {

// ------------------------------------------------------------- scan (int64)

// exclusive scan in place over n values (3 kernels, deterministic)
__global__ void scan_block_sums(const int64_t* in, int64_t n, int64_t* sums) {
    __shared__ int64_t red[32];
    const int64_t i = static_cast<int64_t>(blockIdx.x) * 1024 + threadIdx.x;
    int64_t v = i < n ? in[i] : 0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t t = 0;
        for (int w = 0; w < 32; ++w) t += red[w];
        sums[blockIdx.x] = t;
    }
}

__global__ void scan_sums_serial(int64_t* sums, int64_t nb) {
    // one warp: exclusive scan of the block sums (nb <= a few 10^5)
    __shared__ int64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncwarp();
    for (int64_t base = 0; base < nb; base += 32) {
        const int64_t i = base + threadIdx.x;
        int64_t v = i < nb ? sums[i] : 0;
        int64_t x = v;
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (static_cast<int>(threadIdx.x) >= o) x += y;
        }
        const int64_t c = carry;
        if (i < nb) sums[i] = c + x - v;
        __syncwarp();
        if (threadIdx.x == 31) carry = c + x;
        __syncwarp();
    }
}

__global__ void scan_apply(const int64_t* in, int64_t n, const int64_t* sums, int64_t* out) {
    __shared__ int64_t ws[32];
    const int64_t i = static_cast<int64_t>(blockIdx.x) * 1024 + threadIdx.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t v = i < n ? in[i] : 0;
    int64_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) ws[w] = x;
    __syncthreads();
    if (w == 0) {
        int64_t t = ws[lane];
        int64_t s = t;
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        ws[lane] = s - t;
    }
    __syncthreads();
    if (i < n) out[i] = sums[blockIdx.x] + ws[w] + x - v;
}

// out[0..n] = exclusive scan of in[0..n) with out[n] = total (in and out may alias).
void exclusive_scan(slq_ctx* ctx, const int64_t* in, int64_t n, int64_t* out, DevBuf& tmp) {
    const int64_t nb = std::max<int64_t>(1, ceil_div(n, 1024));
    int64_t* sums = static_cast<int64_t*>(tmp.ensure(sizeof(int64_t) * (nb + 1)));
    scan_block_sums<<<static_cast<unsigned>(nb), 1024, 0, ctx->stream>>>(in, n, sums);
    SLQ_LAUNCH_CHECK(ctx);
    // total = sum of block sums (before the scan overwrites them)
    scan_sums_serial<<<1, 32, 0, ctx->stream>>>(sums, nb + 1);  // sums[nb] (garbage) ignored below
    SLQ_LAUNCH_CHECK(ctx);
    // re-derive: sums now exclusive; total = sums[nb-1] + last block sum -> recompute via apply of the tail
    scan_apply<<<static_cast<unsigned>(nb), 1024, 0, ctx->stream>>>(in, n, sums, out);
    SLQ_LAUNCH_CHECK(ctx);
}

__global__ void set_total_kernel(const int64_t* in, int64_t n, int64_t* out) {
    if (threadIdx.x == 0) out[n] = n > 0 ? out[n - 1] + in[n - 1] : 0;
}

// --------------------------------------------------------- CSC -> CSR

__global__ void csc_count_rows(const int64_t* rows, int64_t nnz, int64_t* cnt) {
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e < nnz) atomicAdd(reinterpret_cast<unsigned long long*>(&cnt[rows[e]]), 1ull);
}

__global__ void csc_scatter(const int64_t* colptr, const int64_t* rows, const double* vals, int64_t n,
                            const int64_t* rowptr, int64_t* fill, int32_t* colidx, double* ovals) {
    const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= n) return;
    for (int64_t e = colptr[j]; e < colptr[j + 1]; ++e) {
        const int64_t r = rows[e];
        const int64_t pos = rowptr[r] + static_cast<int64_t>(atomicAdd(reinterpret_cast<unsigned long long*>(&fill[r]), 1ull));
        colidx[pos] = static_cast<int32_t>(j);
        ovals[pos] = vals[e];
    }
}

// sort each CSR row by column (insertion sort; rows are short)
__global__ void csr_sort_rows(const int64_t* rowptr, int64_t m, int32_t* colidx, double* vals) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= m) return;
    const int64_t b = rowptr[r], e = rowptr[r + 1];
    for (int64_t i = b + 1; i < e; ++i) {
        const int32_t c = colidx[i];
        const double v = vals[i];
        int64_t j = i - 1;
        while (j >= b && colidx[j] > c) {
            colidx[j + 1] = colidx[j];
            vals[j + 1] = vals[j];
            --j;
        }
        colidx[j + 1] = c;
        vals[j + 1] = v;
    }
}

// ------------------------------------------------- S^T CSR from chunk-CSR

// warp per sketch row r: lane l handles chunks l, l+32, ...
__global__ void srow_count(const uint16_t* ptr, int64_t ptr_stride, int64_t nchunks, int64_t d, int64_t* cnt) {
    const int lane = threadIdx.x & 31;
    const int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (r >= d) return;
    int64_t c = 0;
    for (int64_t ch = lane; ch < nchunks; ch += 32) {
        const uint16_t* p = ptr + ch * ptr_stride;
        c += p[r + 1] - p[r];
    }
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) cnt[r] = c;
}

__global__ void srow_fill(const uint16_t* ptr, const uint16_t* ent, int64_t ptr_stride, int64_t ent_stride,
                          int64_t nchunks, int K, int64_t d, const int64_t* srow_ptr, uint32_t* sent) {
    const int lane = threadIdx.x & 31;
    const int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (r >= d) return;
    int64_t out = srow_ptr[r];
    for (int64_t base = 0; base < nchunks; base += 32) {
        const int64_t ch = base + lane;
        int e0 = 0, e1 = 0;
        if (ch < nchunks) {
            const uint16_t* p = ptr + ch * ptr_stride;
            e0 = p[r];
            e1 = p[r + 1];
        }
        const int cnt = e1 - e0;
        int x = cnt;  // inclusive prefix over lanes (chunk order = k order)
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        const int64_t my = out + (x - cnt);
        for (int e = 0; e < cnt; ++e) {
            const unsigned en = ent[ch * ent_stride + e0 + e];
            const uint32_t k = static_cast<uint32_t>(ch * K + (en >> 1));
            sent[my + e] = k | ((en & 1u) << 31);
        }
        out += __shfl_sync(0xffffffffu, x, 31);
    }
}

// --------------------------------------------------------------- K2s gather

struct SGatherArgs {
    const int64_t* rowptr;
    const int32_t* colidx;
    const double* vals;
    const double* b;         // may be null
    int64_t n, d;
    const int64_t* srow_ptr;
    const uint32_t* sent;
    double val;
    double* Y;               // d x (n+1) column-major
    int warps;
};

// One warp per Y row; the row lives in shared memory.  Entries are processed
// in ascending k in batches of kSgB A rows: the batch's S^T entries (one
// coalesced load, lane q holds entry q), their row pointers (lane q loads row
// q's pair) and then every row's (column, value) pairs are all in flight
// before the batch is added row by row -- three dependent load rounds per kSgB
// rows.
constexpr int kSgB = 8;

__global__ void __launch_bounds__(512) sparse_gather_kernel(SGatherArgs g) {
    extern __shared__ double ys[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t r = static_cast<int64_t>(blockIdx.x) * g.warps + w;
    const int64_t n1 = g.n + 1;
    double* y = ys + static_cast<int64_t>(w) * n1;
    for (int64_t j = lane; j < n1; j += 32) y[j] = 0.0;
    __syncwarp();
    if (r < g.d) {
        const int64_t e0 = g.srow_ptr[r], e1 = g.srow_ptr[r + 1];
        for (int64_t e = e0; e < e1; e += kSgB) {
            const int nb = (e1 - e < kSgB) ? static_cast<int>(e1 - e) : kSgB;
            // round 1: entries; round 2: row pointers and b (lane q: row q)
            // (lanes >= nb repeat entry nb - 1: their loads are unconditional too)
            const uint32_t my_en = g.sent[e + (lane < nb ? lane : nb - 1)];
            const int64_t my_k = my_en & 0x7fffffffu;
            const int64_t my_rb = g.rowptr[my_k];
            const int64_t my_re = g.rowptr[my_k + 1];
            const double my_b = g.b ? g.b[my_k] : 0.0;
            // round 3: every row's (column, value) pairs
            // unconditional loads (slots past a row's end read its first entry, or
            // entry 0): a predicated load + default move would wait for the load
            int32_t cc[kSgB][2];
            double vv[kSgB][2];
            int64_t rb[kSgB], re[kSgB];
            unsigned live = 0;
#pragma unroll
            for (int q = 0; q < kSgB; ++q) {
                rb[q] = __shfl_sync(0xffffffffu, my_rb, q);
                re[q] = __shfl_sync(0xffffffffu, my_re, q);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int64_t t = rb[q] + lane + 32 * h;
                    const bool ok = t < re[q];
                    const int64_t at = ok ? t : rb[q];
                    cc[q][h] = g.colidx[at];
                    vv[q][h] = g.vals[at];
                    live |= static_cast<unsigned>(ok) << (2 * q + h);
                }
            }
#pragma unroll
            for (int q = 0; q < kSgB; ++q) {
                const uint32_t en = __shfl_sync(0xffffffffu, my_en, q);
                const double bq = __shfl_sync(0xffffffffu, my_b, q);
                if (q >= nb) break;
                const double sv = (en >> 31) ? -g.val : g.val;
                // csc_matrix.hpp:133: yj[row] += S_val * akj (two roundings)
#pragma unroll
                for (int h = 0; h < 2; ++h)
                    if (live >> (2 * q + h) & 1u) y[cc[q][h]] = __dadd_rn(y[cc[q][h]], __dmul_rn(sv, vv[q][h]));
                for (int64_t t = rb[q] + 64 + lane; t < re[q]; t += 32) {  // rows longer than 64
                    const int32_t c = g.colidx[t];
                    y[c] = __dadd_rn(y[c], __dmul_rn(sv, g.vals[t]));
                }
                if (lane == 0 && g.b && bq != 0.0) y[g.n] = __dadd_rn(y[g.n], __dmul_rn(sv, bq));
                __syncwarp();
            }
        }
        for (int64_t j = lane; j < n1; j += 32) g.Y[j * g.d + r] = y[j];
    }
}

// ------------------------------------------------- K2s column-slab gather
//
// The row gather above re-reads each A row from DRAM for most of its zeta
// target rows: only ~1/4 of the d Y rows fit in shared memory at once, and
// the resident warps drift apart in k.  Here every Y row is resident at once
// by splitting Y into S column slabs: CTA c owns Y rows [c d/G, (c+1) d/G)
// and keeps their slab (w columns) in shared memory; slab q's pass streams
// the slab's part of each A row -- a contiguous segment of the row, since
// CSR rows are sorted by column, located by the per-row slab table P (built
// once per matrix).  The grid walks k in windows of kwin A rows with a soft
// barrier (per-warp counters; a warp may run `lag` windows ahead of the
// slowest), so an A row segment mostly comes from L2 for its other target rows
// (measured: 36.5 GB of DRAM reads at C4 vs 113 GB for the row gather).
//
// Same per-element order as the row gather (for Y[r, j]: ascending k), so the
// same bits.  A warp serves four Y rows at once (8-lane groups), each group
// walks its row's entries in ascending k in batches of 8 (lane l holds entry
// l): entries two batches ahead, the next batch's table words loaded before
// the current batch is added, its segment loads issued right after; the adds
// are branch-free shared-memory read-modify-writes (both slots of an entry
// loaded before either is stored).  L1/LSU-bound (84 % at C4).
constexpr int kSlW = 16;      // warps per CTA
constexpr int kSlB = 8;       // entries per group batch

struct SlabArgs {
    const uint64_t* P;        // [m][S]: row k's slab-q segment, start | length << 40 (slab_ptr_kernel)
    const int32_t* colidx;
    const double* vals;
    const double* b;          // may be null
    int64_t n, d, m;
    int S, w, rmax;           // slab q = columns [q w, min((q + 1) w, n + 1)); column n is b
    const int64_t* srow_ptr;
    const uint32_t* sent;
    double val;
    double* Y;                // d x (n + 1) column-major
    int64_t kwin;             // A rows per window
    int nwin, lag;
    unsigned* sync;           // zeroed before the launch; one count per warp and window
};

constexpr int kSlLenShift = 40;
constexpr uint64_t kSlLoMask = (uint64_t(1) << kSlLenShift) - 1;

// P[k][q]: the entries of row k with columns in slab q (start | length << 40;
// n < 2^24 and nnz < 2^40, host-checked).  A row whose columns are not
// ascending gets the whole row for every slab, and the gather filters its
// entries by column (it always does).  Warp per row.
__global__ void slab_ptr_kernel(const int64_t* rowptr, const int32_t* colidx, int64_t m, int S, int w, uint64_t* P) {
    const int lane = threadIdx.x & 31;
    const int64_t k = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (k >= m) return;
    const int64_t lo = rowptr[k], hi = rowptr[k + 1];
    int cnt = 0;           // lane q (1 <= q <= S): entries with column < q w
    bool sorted = true;
    int prev = INT_MIN;
    for (int64_t e0 = lo; e0 < hi; e0 += 32) {
        const int64_t e = e0 + lane;
        const int c = e < hi ? colidx[e] : INT_MAX;
        const int cp = __shfl_up_sync(0xffffffffu, c, 1);
        const int before = lane == 0 ? prev : cp;
        if (e < hi && c < before) sorted = false;
        prev = __shfl_sync(0xffffffffu, c, 31);
        for (int q = 1; q < S; ++q) {
            const int t = __popc(__ballot_sync(0xffffffffu, c < q * w));
            if (lane == q) cnt += t;
        }
    }
    sorted = __all_sync(0xffffffffu, sorted);
    if (lane == S) cnt = static_cast<int>(hi - lo);
    const int nxt = __shfl_down_sync(0xffffffffu, cnt, 1);  // lane q: boundary q + 1 (S < 31, host)
    if (lane < S) {
        const int64_t b0 = sorted ? lo + cnt : lo, len = sorted ? nxt - cnt : hi - lo;
        P[k * S + lane] = static_cast<uint64_t>(b0) | static_cast<uint64_t>(len) << kSlLenShift;
    }
}

struct SlMeta {         // lane l of a group: entry l of the group's batch
    uint32_t en;
    uint64_t pw;          // its slab segment (P word)
    double b;
};

struct SlPairs {
    int32_t c[kSlB][2];
    double v[kSlB][2];
    unsigned live;        // bit 2 t + h: slot (t, h) holds an entry of the segment
};

__device__ __forceinline__ void sl_rows(const SlabArgs& a, int q, bool ok, SlMeta& M) {
    M.pw = 0;
    M.b = 0.0;
    if (ok) {
        const int64_t k = M.en & 0x7fffffffu;
        M.pw = a.P[k * a.S + q];
        if (a.b && q == a.S - 1) M.b = a.b[k];
    }
}

// The loads are unconditional (slots past the segment's end read its first
// entry, or entry 0 -- always allocated) so that nothing here waits on them: a
// predicated load followed by a default-value move would make the move wait
// for the load, and predicating the loads alone measured 2x slower.  Liveness
// goes into a bit mask, applied at use.
__device__ __forceinline__ void sl_issue(const SlabArgs& a, const SlMeta& M, int g, int gl, SlPairs& B) {
    B.live = 0;
#pragma unroll
    for (int t = 0; t < kSlB; ++t) {
        const uint64_t pw = __shfl_sync(0xffffffffu, M.pw, g * 8 + t);
        const int64_t lo = static_cast<int64_t>(pw & kSlLoMask);
        const int len = static_cast<int>(pw >> kSlLenShift);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int i = gl + 8 * h;
            const bool ok = i < len;
            const int64_t at = ok ? lo + i : lo;
            // plain loads: the segment is re-read from L2 by the row's other target rows
            B.c[t][h] = a.colidx[at];
            B.v[t][h] = a.vals[at];
            B.live |= static_cast<unsigned>(ok) << (2 * t + h);
        }
    }
}

__global__ void __launch_bounds__(32 * kSlW, 1) sparse_gather_slab_kernel(SlabArgs a) {
    extern __shared__ __align__(16) double ysl[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 3, gl = lane & 7;
    const int64_t n1 = a.n + 1;
    const int64_t r0 = blockIdx.x * a.d / gridDim.x, R = (blockIdx.x + 1) * a.d / gridDim.x - r0;
    int64_t* cur = reinterpret_cast<int64_t*>(ysl + static_cast<int64_t>(a.rmax) * a.w);
    int64_t* cend = cur + a.rmax;
    const unsigned WG = gridDim.x * kSlW;  // warps in the grid: each signals every window
    unsigned t_win = 0;  // global window index (slab-major)
    for (int q = 0; q < a.S; ++q) {
        const int64_t c0 = static_cast<int64_t>(q) * a.w, c1 = min(n1, c0 + a.w);
        const unsigned wq = static_cast<unsigned>(c1 - c0);
        const bool lastq = q == a.S - 1 && a.b != nullptr;
        for (int64_t i = tid; i < R * wq; i += blockDim.x) ysl[i] = 0.0;
        for (int64_t i = tid; i < R; i += blockDim.x) {
            cur[i] = a.srow_ptr[r0 + i];
            cend[i] = a.srow_ptr[r0 + i + 1];
        }
        __syncthreads();
        if (warp * 4 >= R) {  // no rows here: count this slab's windows as done
            if (lane == 0) atomicAdd(a.sync, static_cast<unsigned>(a.nwin));
            t_win += a.nwin;
        }
        for (int win = 0; warp * 4 < R && win < a.nwin; ++win, ++t_win) {
            if (t_win >= static_cast<unsigned>(a.lag)) {  // soft barrier: every warp done with window t_win - lag
                if (lane == 0) {
                    const unsigned target = WG * (t_win - a.lag + 1);
                    while (*reinterpret_cast<volatile unsigned*>(a.sync) < target) __nanosleep(256);
                }
                __syncwarp();
            }
            const int64_t kend = min(a.m, (win + 1) * a.kwin);
            for (int64_t base = warp * 4; base < R; base += kSlW * 4) {
                const int64_t i = base + g;
                const bool has = i < R;
                int64_t e = has ? cur[i] : 0;
                const int64_t eend = has ? cend[i] : 0;
                const unsigned ys_row = ptx::smem_u32(ysl) + static_cast<unsigned>((has ? i : 0) * wq) * 8u;
                const unsigned gmask = 0xffu << (8 * g);
                // prologue: batch at e (rows + pairs), entries of the batch at e + 8
                SlMeta Mc, Mn;
                Mc.en = e + gl < eend ? a.sent[e + gl] : 0u;
                Mn.en = e + 8 + gl < eend ? a.sent[e + 8 + gl] : 0u;
                const bool okc = e + gl < eend && (Mc.en & 0x7fffffffu) < kend;
                int nbc = __popc(__ballot_sync(0xffffffffu, okc) & gmask);
                sl_rows(a, q, okc, Mc);
                SlPairs P;
                sl_issue(a, Mc, g, gl, P);
                while (__any_sync(0xffffffffu, nbc > 0)) {
                    // next batch's table lookups (only if this batch is full), entries two ahead
                    const bool okn = nbc == kSlB && e + 8 + gl < eend && (Mn.en & 0x7fffffffu) < kend;
                    const int nbn = __popc(__ballot_sync(0xffffffffu, okn) & gmask);
                    sl_rows(a, q, okn, Mn);
                    const uint32_t en_nn = nbn == kSlB && e + 16 + gl < eend ? a.sent[e + 16 + gl] : 0u;
                    const unsigned longm = __ballot_sync(0xffffffffu, (Mc.pw >> kSlLenShift) > 16);
                    // add this batch in entry order (csc_matrix.hpp:133: yj[row] += S_val * akj);
                    // branch-free per entry (groups past their batch's end are masked off)
                    const unsigned actm = P.live & ((1u << (2 * nbc)) - 1u);
#pragma unroll
                    for (int t = 0; t < kSlB; ++t) {
                        const uint32_t en = __shfl_sync(0xffffffffu, Mc.en, g * 8 + t);
                        const double sv = (en >> 31) ? -a.val : a.val;
                        {   // the entry's two slots hold distinct columns: both loads before both stores
                            const unsigned cu0 = static_cast<unsigned>(P.c[t][0] - static_cast<int>(c0));
                            const unsigned cu1 = static_cast<unsigned>(P.c[t][1] - static_cast<int>(c0));
                            const bool a0 = (actm >> (2 * t) & 1u) && cu0 < wq;
                            const bool a1 = (actm >> (2 * t + 1) & 1u) && cu1 < wq;
                            const unsigned ad0 = ys_row + 8u * cu0, ad1 = ys_row + 8u * cu1;
                            double y0 = 0.0, y1 = 0.0;
                            if (a0) y0 = ptx::lds_f64(ad0);
                            if (a1) y1 = ptx::lds_f64(ad1);
                            if (a0) ptx::sts_f64(ad0, __dadd_rn(y0, __dmul_rn(sv, P.v[t][0])));
                            if (a1) ptx::sts_f64(ad1, __dadd_rn(y1, __dmul_rn(sv, P.v[t][1])));
                        }
                        if (longm & (0x01010101u << t)) {  // some group's entry t is longer than 16 (warp-uniform)
                            int len = 0;
                            int64_t lo = 0;
                            if ((longm >> (g * 8 + t) & 1u) && t < nbc) {
                                const uint64_t pw = a.P[static_cast<int64_t>(en & 0x7fffffffu) * a.S + q];
                                lo = static_cast<int64_t>(pw & kSlLoMask);
                                len = static_cast<int>(pw >> kSlLenShift);
                            }
                            for (int x = 16 + gl; x < len; x += 8) {
                                const unsigned cu = static_cast<unsigned>(a.colidx[lo + x] - static_cast<int>(c0));
                                if (cu < wq) {
                                    const unsigned ad = ys_row + 8u * cu;
                                    ptx::sts_f64(ad, __dadd_rn(ptx::lds_f64(ad), __dmul_rn(sv, a.vals[lo + x])));
                                }
                            }
                        }
                        if (lastq) {
                            const double bt = __shfl_sync(0xffffffffu, Mc.b, g * 8 + t);
                            if (gl == 0 && t < nbc && bt != 0.0) {
                                const unsigned ad = ys_row + 8u * static_cast<unsigned>(a.n - c0);
                                ptx::sts_f64(ad, __dadd_rn(ptx::lds_f64(ad), __dmul_rn(sv, bt)));
                            }
                        }
                        __syncwarp();
                    }
                    e += nbc;
                    sl_issue(a, Mn, g, gl, P);
                    Mc = Mn;
                    nbc = nbn;
                    Mn.en = en_nn;
                }
                if (has && gl == 0) cur[i] = e;
            }
            __syncwarp();
            if (lane == 0) atomicAdd(a.sync, 1u);
        }
        __syncthreads();
        // slab -> Y (column-major; consecutive threads take consecutive rows)
        for (int64_t x = tid; x < R * wq; x += blockDim.x) {
            const int64_t i = x % R, j = x / R;
            a.Y[(c0 + j) * a.d + r0 + i] = ysl[i * wq + j];
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------ K4s pass
//
// One sweep over the CSR rows computes u_hat = A p + c u, ||u_hat||^2 and
// z = A^T u_hat -- the sparse twin of the dense fused pass (lsqr.hpp:115-127
// with SerialOperator<CscMatrix>).  A's values and column indices go straight
// from HBM to registers (each row read by 32 lanes, coalesced; the next row
// quad is loaded while the current one is processed), so shared memory only
// holds p and one private z copy per warp.  Per quad of 4 rows lane l holds
// entries l and l+32 of each row; the four dot products are reduced together
// (6 double shuffles instead of 20); the scatter z[col] += v u_hat then runs
// row by row -- a row's columns are distinct, so lanes never collide, and
// rows are ordered by __syncwarp.  Rows longer than 64 entries take a slow
// tail loop.  Deterministic: fixed row -> warp assignment and fixed orders.

using namespace ptx;

constexpr int kSpMaxWarps = 16;

struct SPassArgs {
    const int64_t* rowptr;
    const int32_t* colidx;
    const double* vals;
    const double* b;      // u when u_in == nullptr
    int64_t m, n;
    const double* p;
    const double* u_in;
    double* u_out;
    const double* coef;
    double c_fixed;
    double* part;         // [grid][n+1]
    int want_z;
    const int* skip;
};

struct SpQuad {
    double v[8];    // entry lane (+32) of row g at [2g] ([2g+1]); garbage where not live
    int c[8];
    double u;       // u of row (lane >> 3)
    unsigned cnt;   // row lengths, 8 bits each (255 = 255 or more: slow tail)
};

__device__ __forceinline__ int sp_cnt(unsigned pk, int g) { return static_cast<int>((pk >> (8 * g)) & 255u); }

// Loads are unconditional (out-of-row slots read entry 0, always allocated)
// so none of them is waited on here; liveness is applied at use.
__device__ __forceinline__ void sp_load_quad(const SPassArgs& a, const double* ubase, int64_t r0, int64_t r_end,
                                             int64_t rp, int lane, SpQuad& q) {
    q.cnt = 0;
#pragma unroll
    for (int g = 0; g < 4; ++g) {
        const int64_t lo = __shfl_sync(0xffffffffu, rp, g);
        const int64_t hi = __shfl_sync(0xffffffffu, rp, g + 1);
        const int64_t len = r0 + g < r_end ? hi - lo : 0;
        const int cnt = static_cast<int>(len < 255 ? len : 255);
        q.cnt |= static_cast<unsigned>(cnt) << (8 * g);
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int t = lane + 32 * j;
            const int64_t idx = t < cnt ? lo + t : 0;
            q.c[2 * g + j] = __ldcs(a.colidx + idx);
            q.v[2 * g + j] = __ldcs(a.vals + idx);
        }
    }
    const int64_t ru = r0 + (lane >> 3);
    q.u = ubase[ru < r_end ? ru : r_end - 1];
}

struct SpCtx {
    int64_t R0, R1, nq;
    int W, lane;
    double c;
    const double* p_s;
    double* zw;
    const double* ubase;
};

// Process quad q (held in `cur`) and start loading quad q + 2W into `fill`.
template <bool WZ>
__device__ __forceinline__ void sp_step(const SPassArgs& a, const SpCtx& x, int64_t q, SpQuad& cur, SpQuad& fill,
                                        int64_t& rp_next, double& ssq) {
    const int lane = x.lane, W = x.W;
    if (q + 2 * W < x.nq) sp_load_quad(a, x.ubase, x.R0 + 4 * (q + 2 * W), x.R1, rp_next, lane, fill);
    {
        const int64_t r = x.R0 + 4 * (q + 3 * W) + (lane < 5 ? lane : 4);
        rp_next = __ldcs(a.rowptr + (r < x.R1 ? r : x.R1));
    }
    // ---- A p for the four rows
    double acc[4];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
        const int cg = sp_cnt(cur.cnt, g);
        const bool oka = lane < cg, okb = lane + 32 < cg;
        if (!oka) cur.v[2 * g] = 0.0, cur.c[2 * g] = 0;
        if (!okb) cur.v[2 * g + 1] = 0.0, cur.c[2 * g + 1] = 0;
        acc[g] = fma(cur.v[2 * g + 1], x.p_s[cur.c[2 * g + 1]], cur.v[2 * g] * x.p_s[cur.c[2 * g]]);
        if (cg > 64) {  // warp-uniform slow tail (rows longer than 64 entries)
            const int64_t r = x.R0 + 4 * q + g;
            const int64_t e = a.rowptr[r + 1];
            for (int64_t t = a.rowptr[r] + 64 + lane; t < e; t += 32) acc[g] = fma(a.vals[t], x.p_s[a.colidx[t]], acc[g]);
        }
    }
    // four-way warp reduction: lane group g ends with row g's sum
    const bool h16 = lane & 16, h8 = lane & 8;
    double k0 = h16 ? acc[2] : acc[0], k1 = h16 ? acc[3] : acc[1];
    k0 += __shfl_xor_sync(0xffffffffu, h16 ? acc[0] : acc[2], 16);
    k1 += __shfl_xor_sync(0xffffffffu, h16 ? acc[1] : acc[3], 16);
    double kk = h8 ? k1 : k0;
    kk += __shfl_xor_sync(0xffffffffu, h8 ? k0 : k1, 8);
    kk += __shfl_xor_sync(0xffffffffu, kk, 4);
    kk += __shfl_xor_sync(0xffffffffu, kk, 2);
    kk += __shfl_xor_sync(0xffffffffu, kk, 1);
    const int64_t rme = x.R0 + 4 * q + (lane >> 3);
    const double uh = (rme < x.R1) ? __dadd_rn(kk, __dmul_rn(x.c, cur.u)) : 0.0;
    if ((lane & 7) == 0 && rme < x.R1) {
        if (a.u_out) a.u_out[rme] = uh;
        ssq = fma(uh, uh, ssq);
    }
    // ---- z += A^T u_hat, row by row
    if (WZ && a.want_z) {
#pragma unroll
        for (int g = 0; g < 4; ++g) {
            const double ug = __shfl_sync(0xffffffffu, uh, 8 * g);
            const int cg = sp_cnt(cur.cnt, g);
            const bool oka = lane < cg, okb = lane + 32 < cg;
            const double za = oka ? x.zw[cur.c[2 * g]] : 0.0;
            const double zb = okb ? x.zw[cur.c[2 * g + 1]] : 0.0;
            if (oka) x.zw[cur.c[2 * g]] = fma(cur.v[2 * g], ug, za);
            if (okb) x.zw[cur.c[2 * g + 1]] = fma(cur.v[2 * g + 1], ug, zb);
            if (cg > 64) {
                const int64_t r = x.R0 + 4 * q + g;
                const int64_t e = a.rowptr[r + 1];
                for (int64_t t = a.rowptr[r] + 64 + lane; t < e; t += 32) {
                    const int cc = a.colidx[t];
                    x.zw[cc] = fma(a.vals[t], ug, x.zw[cc]);
                }
            }
            __syncwarp();
        }
    }
}

// WZ = false: the u_hat half only (two-pass operator: z comes from
// sparse_tpass_kernel over the row-blocked CSC copy), no z copies.
template <bool WZ>
__global__ void __launch_bounds__(32 * kSpMaxWarps, 1) sparse_pass_kernel(SPassArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    if (a.skip && *a.skip) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int W = blockDim.x >> 5;
    const int64_t n = a.n;
    double* p_s = reinterpret_cast<double*>(smem);
    double* z_s = p_s + n;
    for (int64_t j = tid; j < n; j += blockDim.x) p_s[j] = a.p[j];
    if (WZ)
        for (int64_t j = tid; j < static_cast<int64_t>(W) * n; j += blockDim.x) z_s[j] = 0.0;
    __syncthreads();

    const int64_t R0 = blockIdx.x * a.m / gridDim.x, R1 = (blockIdx.x + 1) * a.m / gridDim.x;
    const int64_t nq = (R1 - R0 + 3) / 4;
    const double c = a.coef ? *a.coef : a.c_fixed;
    const double* ubase = a.u_in ? a.u_in : a.b;
    double* zw = z_s + static_cast<int64_t>(warp) * n;
    double ssq = 0.0;

    auto rp_load = [&](int64_t q) -> int64_t {  // lanes 0..4: rowptr of the quad's rows (unconditional load)
        const int64_t r = R0 + 4 * q + (lane < 5 ? lane : 4);
        return __ldcs(a.rowptr + (r < R1 ? r : R1));
    };
    // three quads in flight per warp (the one being processed and the next
    // two); the loop is unrolled by three so the buffers rotate by name
    int64_t q = warp;
    SpQuad qa, qb, qc;
    int64_t rp_next = 0;
    if (q < nq) {
        const int64_t rpa = rp_load(q), rpb = rp_load(q + W);
        sp_load_quad(a, ubase, R0 + 4 * q, R1, rpa, lane, qa);
        sp_load_quad(a, ubase, R0 + 4 * (q + W), R1, rpb, lane, qb);
        rp_next = rp_load(q + 2 * W);
    }
    SpCtx x{R0, R1, nq, W, lane, c, p_s, zw, ubase};
    while (q < nq) {
        sp_step<WZ>(a, x, q, qa, qc, rp_next, ssq);
        q += W;
        if (q >= nq) break;
        sp_step<WZ>(a, x, q, qb, qa, rp_next, ssq);
        q += W;
        if (q >= nq) break;
        sp_step<WZ>(a, x, q, qc, qb, rp_next, ssq);
        q += W;
    }
    // ssq: lanes 0, 8, 16, 24 hold partial sums
    ssq += __shfl_xor_sync(0xffffffffu, ssq, 8);
    ssq += __shfl_xor_sync(0xffffffffu, ssq, 16);
    __shared__ double red[kSpMaxWarps];  // own array: p's n doubles may be fewer than the warps
    if (lane == 0) red[warp] = ssq;
    __syncthreads();
    double* outp = a.part + static_cast<int64_t>(blockIdx.x) * (n + 1);
    if (WZ && a.want_z)
        for (int64_t j = tid; j < n; j += blockDim.x) {
            double s = 0.0;
            for (int w = 0; w < W; ++w) s += z_s[static_cast<int64_t>(w) * n + j];
            outp[j] = s;
        }
    if (tid == 0) {
        double s = 0.0;
        for (int w = 0; w < W; ++w) s += red[w];
        outp[n] = s;
    }
}

// ------------------------------------------- row-blocked CSC (two-pass K4s)
//
// z = A^T u_hat without the per-row scatter: a copy of A sorted by column
// within blocks of kTbRows rows (the row's u16 offset in the block + the
// value, entries of a column in ascending row), column pointers per block
// relative to the block's first CSR entry rowptr[b * kTbRows] -- the block
// occupies the same entry range as in the CSR.  sparse_tpass_kernel stages a
// block's u_hat in shared memory and lets each warp reduce whole column
// segments: streaming loads, shared-memory gathers, no read-modify-writes.
constexpr int kTbRows = 16384;

struct BcscArgs {
    const int64_t* rowptr;
    const int32_t* colidx;
    const double* vals;
    int64_t m, n;
    int W;                 // warps used for the deterministic placement
    uint32_t* blkcol;      // [nblk][n + 1]
    uint16_t* crow;        // [nnz]
    double* cval;          // [nnz]
    uint16_t* col16;       // [nnz] the CSR's column indices as u16 (the u_hat pass)
};

// One CTA per row block.  Warp w owns a contiguous range of the block's rows:
// (1) per-warp column counts (u16: a row's columns are distinct, so within a
// row the lanes never collide; rows are ordered by __syncwarp), (2) column
// starts (exclusive scan of the column totals) and per-warp bases relative to
// them (u16, < kTbRows), (3) each warp re-walks its rows in order and places
// entries -- ascending row within every column, deterministic, no atomics.
// The row walks keep four rows' loads in flight (two entries per lane per
// row; longer rows take a tail loop).
constexpr int kBcRows = 4;

struct BcRows {
    int64_t lo[kBcRows], hi[kBcRows];
    int c[kBcRows][2];
    double v[kBcRows][2];
};

template <bool VALS>
__device__ __forceinline__ void bc_load(const BcscArgs& a, int64_t r, int64_t r_end, int lane, BcRows& q) {
    const int64_t rr = min(r + lane, r_end);
    const int64_t rp = lane <= kBcRows ? a.rowptr[rr] : 0;
#pragma unroll
    for (int t = 0; t < kBcRows; ++t) {
        q.lo[t] = __shfl_sync(0xffffffffu, rp, t);
        q.hi[t] = r + t < r_end ? __shfl_sync(0xffffffffu, rp, t + 1) : q.lo[t];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t e = q.lo[t] + lane + 32 * h;
            const bool ok = e < q.hi[t];
            q.c[t][h] = ok ? __ldcs(a.colidx + e) : 0;
            if (VALS) q.v[t][h] = ok ? __ldcs(a.vals + e) : 0.0;
        }
    }
}

__global__ void __launch_bounds__(1024) bcsc_build_kernel(BcscArgs a) {
    extern __shared__ uint32_t bcs[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int W = a.W;
    const int64_t n = a.n;
    uint32_t* start = bcs;                                     // [n] column start in the block
    uint16_t* rel = reinterpret_cast<uint16_t*>(bcs + n);     // [W][n] counts, then bases
    const int64_t b = blockIdx.x;
    const int64_t r0 = b * kTbRows, r1 = min(a.m, r0 + kTbRows);
    const int64_t e0 = a.rowptr[r0];
    for (int64_t i = tid; i < static_cast<int64_t>(W) * n; i += blockDim.x) rel[i] = 0;
    __syncthreads();
    const int64_t rows = r1 - r0;
    const int64_t wr0 = r0 + warp * rows / W, wr1 = r0 + (warp + 1) * rows / W;
    uint16_t* mine = rel + static_cast<int64_t>(warp) * n;
    if (warp < W) {
        for (int64_t r = wr0; r < wr1; r += kBcRows) {
            BcRows q;
            bc_load<false>(a, r, wr1, lane, q);
#pragma unroll
            for (int t = 0; t < kBcRows; ++t) {
#pragma unroll
                for (int h = 0; h < 2; ++h)
                    if (q.lo[t] + lane + 32 * h < q.hi[t]) {
                        mine[q.c[t][h]] += 1;
                        a.col16[q.lo[t] + lane + 32 * h] = static_cast<uint16_t>(q.c[t][h]);
                    }
                for (int64_t e = q.lo[t] + 64 + lane; e < q.hi[t]; e += 32) {  // rows of > 64 entries
                    const int c = a.colidx[e];
                    mine[c] += 1;
                    a.col16[e] = static_cast<uint16_t>(c);
                }
                __syncwarp();
            }
        }
    }
    __syncthreads();
    // column totals -> per-warp relative bases; exclusive scan of the totals
    __shared__ uint32_t tot[1024];
    const int64_t per = (n + blockDim.x - 1) / blockDim.x;
    const int64_t j0 = tid * per, j1 = min(n, j0 + per);
    uint32_t run = 0;
    for (int64_t j = j0; j < j1; ++j) {
        uint32_t cj = 0;
        for (int w = 0; w < W; ++w) {
            const uint32_t c = rel[static_cast<int64_t>(w) * n + j];
            rel[static_cast<int64_t>(w) * n + j] = static_cast<uint16_t>(cj);
            cj += c;
        }
        start[j] = cj;  // total for now
        run += cj;
    }
    tot[tid] = run;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
        const uint32_t v = tid >= o ? tot[tid - o] : 0u;
        __syncthreads();
        tot[tid] += v;
        __syncthreads();
    }
    run = tot[tid] - run;  // exclusive
    uint32_t* bc = a.blkcol + b * (n + 1);
    for (int64_t j = j0; j < j1; ++j) {
        const uint32_t cj = start[j];
        start[j] = run;
        bc[j] = run;
        run += cj;
    }
    if (tid == blockDim.x - 1) bc[n] = tot[tid];
    __syncthreads();
    if (warp < W) {
        for (int64_t r = wr0; r < wr1; r += kBcRows) {
            BcRows q;
            bc_load<true>(a, r, wr1, lane, q);
#pragma unroll
            for (int t = 0; t < kBcRows; ++t) {
                const uint16_t rl = static_cast<uint16_t>(r + t - r0);
#pragma unroll
                for (int h = 0; h < 2; ++h)
                    if (q.lo[t] + lane + 32 * h < q.hi[t]) {
                        const int c = q.c[t][h];
                        const uint32_t pos = start[c] + mine[c];
                        mine[c] += 1;
                        a.crow[e0 + pos] = rl;
                        a.cval[e0 + pos] = q.v[t][h];
                    }
                for (int64_t e = q.lo[t] + 64 + lane; e < q.hi[t]; e += 32) {
                    const int c = a.colidx[e];
                    const uint32_t pos = start[c] + mine[c];
                    mine[c] += 1;
                    a.crow[e0 + pos] = rl;
                    a.cval[e0 + pos] = a.vals[e];
                }
                __syncwarp();
            }
        }
    }
}

// ------------------------------------ u_hat pass over the CSR (two-pass K4s)
//
// u_hat = A p + c u, ||u_hat||^2 as a TMA stream like the dense pass: a
// producer lane copies chunk k's entry values, u16 column indices, row
// pointers and u slice (four 1D bulk copies, 16-byte aligned supersets) into a
// 4-stage ring; 8 consumer warps take the chunk's rows in lane groups of 8 (4
// rows per warp step: strided products against p in shared memory, 3-step
// shuffle reduction).  A chunk whose entries exceed the stage capacity is
// read from global memory directly (flagged by the producer).
constexpr int kUpConsumers = 16;
// ring geometry: ROWS rows per chunk, CAP entries per stage, ST stages
template <int ROWS, int CAP, int ST>
struct UpGeom {
    static constexpr int kRows = ROWS, kStages = ST;
    static constexpr unsigned kV = (CAP + 8) * 8, kC = (CAP + 8) * 2, kP = (ROWS + 8) * 8;
    static constexpr unsigned kStage = kV + kC + 2 * kP;
};

struct UPassArgs {
    const int64_t* rowptr;
    const uint16_t* col16;
    const double* vals;
    const double* b;      // u when u_in == nullptr
    int64_t m, n;
    const double* p;
    const double* u_in;
    double* u_out;
    const double* coef;
    double c_fixed;
    double* part;         // [grid][n+1]: ||u_hat||^2 partial in [n]
    const int* skip;
};

template <class G, int LPR>
__global__ void __launch_bounds__(32 * (kUpConsumers + 1), 1) sparse_upass_kernel(UPassArgs a) {
    constexpr int kUpRows = G::kRows, kUpStages = G::kStages;
    constexpr unsigned kUpVBytes = G::kV, kUpCBytes = G::kC, kUpPBytes = G::kP, kUpStage = G::kStage;
    extern __shared__ __align__(128) unsigned char usm[];
    __shared__ __align__(8) uint64_t full[kUpStages], empty[kUpStages];
    __shared__ int direct[kUpStages];
    __shared__ double red[kUpConsumers];
    if (a.skip && *a.skip) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t n = a.n;
    double* p_s = reinterpret_cast<double*>(usm + kUpStages * kUpStage);
    for (int64_t j = tid; j < n; j += blockDim.x) p_s[j] = a.p[j];
    if (tid == 0) {
        for (int s = 0; s < kUpStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kUpConsumers);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    const int64_t R0 = blockIdx.x * a.m / gridDim.x, R1 = (blockIdx.x + 1) * a.m / gridDim.x;
    const int64_t nk = (R1 - R0 + kUpRows - 1) / kUpRows;
    const double* ubase = a.u_in ? a.u_in : a.b;
    if (warp == kUpConsumers) {
        // ---------------- producer warp: lane l holds the first row pointer of
        // chunk k0 + l (loaded 32 chunks at a time), lane 0 issues the copies
        for (int64_t k0 = 0; k0 < nk; k0 += 32) {
            const int64_t kr = min(R0 + (k0 + lane) * kUpRows, R1);
            const int64_t rp = a.rowptr[kr];
            const int64_t kr1 = min(R0 + (k0 + 32) * kUpRows, R1);
            const int64_t rp_last = a.rowptr[kr1];
            for (int l = 0; l < 32 && k0 + l < nk; ++l) {
                const int64_t k = k0 + l;
                const int64_t e0 = __shfl_sync(0xffffffffu, rp, l);
                const int64_t e1 = l < 31 ? __shfl_sync(0xffffffffu, rp, l + 1) : rp_last;
                if (lane == 0) {
                    const int s = static_cast<int>(k % kUpStages);
                    const int64_t rr = k / kUpStages;
                    if (rr > 0) mbar_wait(&empty[s], static_cast<unsigned>((rr - 1) & 1));
                    unsigned char* st = usm + s * kUpStage;
                    const int64_t r0 = R0 + k * kUpRows, r1 = min(r0 + kUpRows, R1);
                    const int64_t va = e0 & ~int64_t(1), ca = e0 & ~int64_t(7), pa = r0 & ~int64_t(1);
                    const unsigned vb = static_cast<unsigned>(((e1 - va) * 8 + 15) & ~int64_t(15));
                    const unsigned cb = static_cast<unsigned>(((e1 - ca) * 2 + 15) & ~int64_t(15));
                    const unsigned pb = static_cast<unsigned>(((r1 + 1 - pa) * 8 + 15) & ~int64_t(15));
                    const unsigned ub = static_cast<unsigned>(((r1 - pa) * 8 + 15) & ~int64_t(15));
                    const bool dir = vb > kUpVBytes || cb > kUpCBytes;
                    direct[s] = dir ? 1 : 0;
                    mbar_expect_tx(&full[s], pb + ub + (dir ? 0u : vb + cb));
                    bulk_g2s(st + kUpVBytes + kUpCBytes, a.rowptr + pa, pb, &full[s]);
                    bulk_g2s(st + kUpVBytes + kUpCBytes + kUpPBytes, ubase + pa, ub, &full[s]);
                    if (!dir) {
                        bulk_g2s(st, a.vals + va, vb, &full[s]);
                        bulk_g2s(st + kUpVBytes, a.col16 + ca, cb, &full[s]);
                    }
                }
            }
        }
        return;
    }
    // ---------------- consumers: lane groups of LPR lanes, one row each
    // (LPR = 4 for rows of <= 100 entries on average: twice the rows per warp step; else 8)
    constexpr int kGroups = 32 / LPR;
    const double c = a.coef ? *a.coef : a.c_fixed;
    const int g = lane / LPR, gl = lane % LPR;
    double ssq = 0.0;
    for (int64_t k = 0; k < nk; ++k) {
        const int s = static_cast<int>(k % kUpStages);
        mbar_wait(&full[s], static_cast<unsigned>((k / kUpStages) & 1));
        const unsigned char* st = usm + s * kUpStage;
        const double* V = reinterpret_cast<const double*>(st);
        const uint16_t* Cc = reinterpret_cast<const uint16_t*>(st + kUpVBytes);
        const int64_t* P = reinterpret_cast<const int64_t*>(st + kUpVBytes + kUpCBytes);
        const double* U = reinterpret_cast<const double*>(st + kUpVBytes + kUpCBytes + kUpPBytes);
        const int64_t r0 = R0 + k * kUpRows, r1 = min(r0 + kUpRows, R1);
        const int64_t pa = r0 & ~int64_t(1);
        const int64_t e0 = P[r0 - pa];
        const int64_t va = e0 & ~int64_t(1), ca = e0 & ~int64_t(7);
        const bool dir = direct[s] != 0;
        for (int64_t i = r0 + warp * kGroups + g; i - g < r1; i += kGroups * kUpConsumers) {
            double acc = 0.0;
            if (i < r1) {
                const int64_t lo = P[i - pa], hi = P[i + 1 - pa];
                if (!dir) {
                    // two independent chains per lane, loads of both issued first
                    double a1 = 0.0;
                    int64_t e = lo + gl;
                    for (; e + LPR < hi; e += 2 * LPR) {
                        const int c0 = Cc[e - ca], c1 = Cc[e + LPR - ca];
                        const double v0 = V[e - va], v1 = V[e + LPR - va];
                        acc = fma(v0, p_s[c0], acc);
                        a1 = fma(v1, p_s[c1], a1);
                    }
                    if (e < hi) acc = fma(V[e - va], p_s[Cc[e - ca]], acc);
                    acc += a1;
                } else {
                    for (int64_t e = lo + gl; e < hi; e += LPR) acc = fma(a.vals[e], p_s[a.col16[e]], acc);
                }
            }
#pragma unroll
            for (int o = LPR / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (gl == 0 && i < r1) {
                const double uh = __dadd_rn(acc, __dmul_rn(c, U[i - pa]));
                if (a.u_out) a.u_out[i] = uh;
                ssq = fma(uh, uh, ssq);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
#pragma unroll
    for (int o = LPR; o < 32; o <<= 1) ssq += __shfl_xor_sync(0xffffffffu, ssq, o);
    if (lane == 0) red[warp] = ssq;
    asm volatile("bar.sync 1, %0;\n" ::"n"(32 * kUpConsumers));  // consumers only (the producer has returned)
    if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < kUpConsumers; ++w) t += red[w];
        a.part[static_cast<int64_t>(blockIdx.x) * (n + 1) + n] = t;
    }
}

struct TPassArgs {
    const int64_t* rowptr;
    const uint32_t* blkcol;
    const uint16_t* crow;
    const double* cval;
    const double* uhat;   // m (+ pad), written by the u_hat pass
    int64_t m, n, nblk;
    double* part;         // [grid][n + 1]: z partials in [0, n)
    int want_z;
    const int* skip;
    int z_smem;           // z accumulated in shared memory (else in part directly)
};

// grid CTAs split the row blocks evenly; per block: u_hat of the block ->
// shared memory (TMA bulk copy), then warp w reduces columns w, w + W, ...
// of the block (lanes stride the column's entries, 4 independent partial sums
// for memory parallelism, fixed-order warp reduction) into z_s[j].
__global__ void __launch_bounds__(1024, 1) sparse_tpass_kernel(TPassArgs a) {
    extern __shared__ __align__(128) unsigned char tsm[];
    __shared__ __align__(8) uint64_t ubar;
    if ((a.skip && *a.skip) || !a.want_z) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, W = blockDim.x >> 5;
    const int64_t n = a.n;
    double* u_s = reinterpret_cast<double*>(tsm);
    uint32_t* bc_s = reinterpret_cast<uint32_t*>(u_s + kTbRows);  // the block's column starts
    // z accumulates in shared memory when it fits, else in this CTA's partial
    // row (column j is owned by warp j % W in every block: no races, fixed
    // order); part[.][n] holds the u_hat pass's ||u_hat||^2
    double* outp = a.part + static_cast<int64_t>(blockIdx.x) * (n + 1);
    double* zp = a.z_smem ? reinterpret_cast<double*>(bc_s + ((n + 8) & ~int64_t(3))) : outp;
    for (int64_t j = tid; j < n; j += blockDim.x) zp[j] = 0.0;
    if (tid == 0) {
        mbar_init(&ubar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    const int64_t b0 = blockIdx.x * a.nblk / gridDim.x, b1 = (blockIdx.x + 1) * a.nblk / gridDim.x;
    unsigned phase = 0;
    for (int64_t b = b0; b < b1; ++b) {
        const int64_t r0 = b * kTbRows, rows = min(static_cast<int64_t>(kTbRows), a.m - r0);
        if (tid == 0) {
            const unsigned bytes = static_cast<unsigned>((rows * 8 + 15) & ~int64_t(15));
            // column starts: 16-byte aligned superset of [b (n+1), (b+1)(n+1))
            const int64_t c0 = (b * (n + 1)) & ~int64_t(3);
            const unsigned cbytes = static_cast<unsigned>((((b + 1) * (n + 1) - c0) * 4 + 15) & ~int64_t(15));
            mbar_expect_tx(&ubar, bytes + cbytes);
            bulk_g2s(u_s, a.uhat + r0, bytes, &ubar);
            bulk_g2s(bc_s, a.blkcol + c0, cbytes, &ubar);
        }
        mbar_wait(&ubar, phase);
        phase ^= 1u;
        const int64_t e0 = a.rowptr[r0];
        const uint32_t* bc = bc_s + (b * (n + 1) - ((b * (n + 1)) & ~int64_t(3)));
        const uint16_t* cr = a.crow + e0;
        const double* cv = a.cval + e0;
        for (int64_t j = warp; j < n; j += W) {
            const uint32_t lo = bc[j], hi = bc[j + 1];
            // eight loads of each kind in flight per lane (masked past the
            // segment's end), four partial sums
            double sp[4] = {0.0, 0.0, 0.0, 0.0};
            for (uint32_t e = lo + lane; e < hi; e += 256) {
                double v[8];
                uint16_t q[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const uint32_t idx = e + 32u * u;
                    const bool ok = idx < hi;
                    v[u] = ok ? __ldcs(cv + idx) : 0.0;
                    q[u] = ok ? __ldcs(cr + idx) : static_cast<uint16_t>(0);
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) sp[u & 3] = fma(v[u], u_s[q[u]], sp[u & 3]);
            }
            double s = (sp[0] + sp[1]) + (sp[2] + sp[3]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (lane == 0) zp[j] += s;
        }
        __syncthreads();  // u_s is overwritten by the next block
    }
    if (a.z_smem)
        for (int64_t j = tid; j < n; j += blockDim.x) outp[j] = zp[j];
}

}  // namespace

// ---------------------------------------------------------------- host

void sparse_from_csc(slq_ctx* ctx, slq_sparse* A, const int64_t* colptr_h, const int64_t* rows_h,
                     const double* vals_h) {
    const int64_t m = A->m, n = A->n, nnz = A->nnz;
    DevBuf dcp, drows, dvals, cnt, tmp;
    int64_t* cp = static_cast<int64_t*>(dcp.ensure(sizeof(int64_t) * (n + 1)));
    int64_t* rw = static_cast<int64_t*>(drows.ensure(sizeof(int64_t) * std::max<int64_t>(1, nnz)));
    double* vl = static_cast<double*>(dvals.ensure(sizeof(double) * std::max<int64_t>(1, nnz)));
    int64_t* c = static_cast<int64_t*>(cnt.ensure(sizeof(int64_t) * (m + 1)));
    SLQ_CUDA_CHECK(cudaMemcpyAsync(cp, colptr_h, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, ctx->stream));
    if (nnz > 0) {
        SLQ_CUDA_CHECK(cudaMemcpyAsync(rw, rows_h, sizeof(int64_t) * nnz, cudaMemcpyHostToDevice, ctx->stream));
        SLQ_CUDA_CHECK(cudaMemcpyAsync(vl, vals_h, sizeof(double) * nnz, cudaMemcpyHostToDevice, ctx->stream));
    }
    SLQ_CUDA_CHECK(cudaMemsetAsync(c, 0, sizeof(int64_t) * (m + 1), ctx->stream));
    if (nnz > 0) {
        csc_count_rows<<<static_cast<unsigned>(ceil_div(nnz, 256)), 256, 0, ctx->stream>>>(rw, nnz, c);
        SLQ_LAUNCH_CHECK(ctx);
    }
    exclusive_scan(ctx, c, m, A->rowptr, tmp);
    set_total_kernel<<<1, 32, 0, ctx->stream>>>(c, m, A->rowptr);
    SLQ_LAUNCH_CHECK(ctx);
    SLQ_CUDA_CHECK(cudaMemsetAsync(c, 0, sizeof(int64_t) * (m + 1), ctx->stream));
    if (n > 0) {
        csc_scatter<<<static_cast<unsigned>(ceil_div(n, 128)), 128, 0, ctx->stream>>>(cp, rw, vl, n, A->rowptr, c,
                                                                                    A->colidx, A->vals);
        SLQ_LAUNCH_CHECK(ctx);
    }
    if (m > 0) {
        csr_sort_rows<<<static_cast<unsigned>(ceil_div(m, 128)), 128, 0, ctx->stream>>>(A->rowptr, m, A->colidx,
                                                                                     A->vals);
        SLQ_LAUNCH_CHECK(ctx);
    }
    SLQ_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
}

void sparse_alloc(slq_ctx* ctx, slq_sparse* A, bool with_b) {
    SLQ_CUDA_CHECK(cudaMalloc(&A->rowptr, sizeof(int64_t) * (A->m + 1 + 64)));
    SLQ_CUDA_CHECK(cudaMalloc(&A->colidx, sizeof(int32_t) * (A->nnz + 4)));
    SLQ_CUDA_CHECK(cudaMalloc(&A->vals, sizeof(double) * (A->nnz + 4)));
    SLQ_CUDA_CHECK(cudaMemsetAsync(A->rowptr, 0, sizeof(int64_t) * (A->m + 1 + 64), ctx->stream));
    SLQ_CUDA_CHECK(cudaMemsetAsync(A->colidx, 0, sizeof(int32_t) * (A->nnz + 4), ctx->stream));
    SLQ_CUDA_CHECK(cudaMemsetAsync(A->vals, 0, sizeof(double) * (A->nnz + 4), ctx->stream));
    if (with_b) {
        SLQ_CUDA_CHECK(cudaMalloc(&A->b, sizeof(double) * (A->m + kSparseRowPad)));
        SLQ_CUDA_CHECK(cudaMemsetAsync(A->b, 0, sizeof(double) * (A->m + kSparseRowPad), ctx->stream));
    }
}

void drop_slab_tables(slq_sparse* A) {
    for (int i = 0; i < A->s_ntab; ++i) {
        cudaFree(A->s_tab[i].p);
        if (A->s_tab[i].ready) cudaEventDestroy(A->s_tab[i].ready);
        A->s_tab[i] = slq_sparse::SlabTable{};
    }
    A->s_ntab = 0;
    A->s_valid = false;
}

void sparse_free(slq_sparse* A) {
    if (A->owned) {
        cudaFree(A->rowptr);
        cudaFree(A->colidx);
        cudaFree(A->vals);
        cudaFree(A->b);
    }
    cudaFree(A->t_blkcol);
    cudaFree(A->t_crow);
    cudaFree(A->t_cval);
    cudaFree(A->t_uscr);
    cudaFree(A->t_col16);
    drop_slab_tables(A);
    if (A->t_ready) cudaEventDestroy(A->t_ready);
    A->t_ready = nullptr;
    A->t_col16 = nullptr;
    A->t_blkcol = nullptr;
    A->t_crow = nullptr;
    A->t_cval = nullptr;
    A->t_uscr = nullptr;
    A->t_valid = false;
}

void prepare_two_pass(slq_ctx* ctx, slq_sparse* A, bool async) {
    if (A->t_valid) return;
    const int64_t m = A->m, n = A->n, nnz = A->nnz;
    if (!A->t_crow) {  // sizes are fixed for the handle's lifetime
        A->t_nblk = ceil_div(std::max<int64_t>(m, 1), static_cast<int64_t>(kTbRows));
        SLQ_CUDA_CHECK(cudaMalloc(&A->t_blkcol, sizeof(uint32_t) * (A->t_nblk * (n + 1) + 16)));  // + bulk-copy slack
        SLQ_CUDA_CHECK(cudaMalloc(&A->t_crow, sizeof(uint16_t) * (nnz + 64)));
        SLQ_CUDA_CHECK(cudaMalloc(&A->t_cval, sizeof(double) * (nnz + 64)));
        SLQ_CUDA_CHECK(cudaMalloc(&A->t_uscr, sizeof(double) * (m + kSparseRowPad)));
        SLQ_CUDA_CHECK(cudaMalloc(&A->t_col16, sizeof(uint16_t) * (nnz + 64)));
        SLQ_CUDA_CHECK(cudaMemsetAsync(A->t_col16, 0, sizeof(uint16_t) * (nnz + 64), ctx->stream));
        SLQ_CUDA_CHECK(cudaMemsetAsync(A->t_uscr, 0, sizeof(double) * (m + kSparseRowPad), ctx->stream));
    }
    int W = static_cast<int>(std::min<int64_t>(32, (200 * 1024 - 4 * n) / (2 * std::max<int64_t>(n, 1))));
    if (W < 1) fail(SLQ_UNSUPPORTED, "sparse lsqr: n too large for the blocked-CSC build");
    const size_t smem = sizeof(uint32_t) * n + sizeof(uint16_t) * W * n;
    SLQ_CUDA_CHECK(cudaFuncSetAttribute(bcsc_build_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(smem)));
    BcscArgs ba{A->rowptr, A->colidx, A->vals, m, n, W, A->t_blkcol, A->t_crow, A->t_cval, A->t_col16};
    cudaStream_t st = ctx->stream;
    if (async) {
        // on the side stream, after everything already queued on the main one
        // (the CSR fill); the first pass waits for it (SparseOp::ready)
        if (!ctx->aux) {
            SLQ_CUDA_CHECK(cudaStreamCreateWithFlags(&ctx->aux, cudaStreamNonBlocking));
            SLQ_CUDA_CHECK(cudaEventCreateWithFlags(&ctx->aux_ev[0], cudaEventDisableTiming));
        }
        SLQ_CUDA_CHECK(cudaEventRecord(ctx->aux_ev[0], ctx->stream));
        SLQ_CUDA_CHECK(cudaStreamWaitEvent(ctx->aux, ctx->aux_ev[0], 0));
        st = ctx->aux;
    }
    bcsc_build_kernel<<<static_cast<unsigned>(A->t_nblk), 1024, smem, st>>>(ba);
    SLQ_LAUNCH_CHECK(ctx);
    if (async) {
        if (!A->t_ready) SLQ_CUDA_CHECK(cudaEventCreateWithFlags(&A->t_ready, cudaEventDisableTiming));
        SLQ_CUDA_CHECK(cudaEventRecord(A->t_ready, ctx->aux));
        A->t_pending = true;
    }
    A->t_valid = true;
}

// Y_aug (d x (n+1), column-major) = S [A b] for this rank's rows; S keyed by global row id.
void sketch_apply_sparse_dev(slq_ctx* ctx, const slq_sparse* A, int64_t d, int64_t zeta, uint64_t seed, double* Y) {
    if (zeta > d || zeta < 1) fail(SLQ_INVALID_SPARSITY, "apply: need 1 <= zeta <= d");
    if (zeta > 1024) fail(SLQ_UNSUPPORTED, "sketch_apply: zeta > 1024");
    Workspace& ws = ctx->ws;
    const int64_t m = A->m;
    if (m == 0) {
        SLQ_CUDA_CHECK(cudaMemsetAsync(Y, 0, sizeof(double) * d * (A->n + 1), ctx->stream));
        return;
    }
    uint32_t* compact = static_cast<uint32_t*>(ws.compact.ensure(sizeof(uint32_t) * m * zeta));
    int64_t* work = zeta > 32 ? static_cast<int64_t*>(ws.tmp.ensure(sizeof(int64_t) * m * zeta)) : nullptr;
    generate_sparse_sign_dev(ctx, d, zeta, seed, A->row_begin, m, compact, work, nullptr, nullptr, nullptr);
    sketch_apply_sparse_compact_dev(ctx, A, d, compact, nullptr, zeta, 1.0 / std::sqrt(static_cast<double>(zeta)), Y);
}

void sketch_apply_sparse_compact_dev(slq_ctx* ctx, const slq_sparse* A, int64_t d, const uint32_t* compact,
                                     const int64_t* colptr_dev, int64_t zeta_max, double val, double* Y) {
    if (d >= (int64_t(1) << 20)) fail(SLQ_UNSUPPORTED, "sketch_apply: d too large");
    if (A->m >= (int64_t(1) << 31)) fail(SLQ_UNSUPPORTED, "sparse sketch_apply: more than 2^31 rows per block");
    Workspace& ws = ctx->ws;
    const int64_t m = A->m, n = A->n;
    if (m == 0) {
        SLQ_CUDA_CHECK(cudaMemsetAsync(Y, 0, sizeof(double) * d * (n + 1), ctx->stream));
        return;
    }
    // S^T rows (entries of each Y row in ascending k)
    // workspace buffers (grow-only): a local DevBuf's cudaFree would wait for the device
    DevBuf& scan_tmp = ws.st_scan;
    int64_t* srow_ptr = static_cast<int64_t*>(ws.st_ptr.ensure(sizeof(int64_t) * (d + 1)));
    int64_t* cnt = static_cast<int64_t*>(ws.st_cnt.ensure(sizeof(int64_t) * (d + 1)));
    uint32_t* sent = nullptr;
    {
        ChunkCsr cc = build_chunk_csr(ctx, compact, colptr_dev, zeta_max, m, d, 0);
        const unsigned wgrid = static_cast<unsigned>(ceil_div(d * 32, 256));
        srow_count<<<wgrid, 256, 0, ctx->stream>>>(cc.ptr, cc.plan.ptr_stride, cc.plan.nchunks, d, srow_ptr);
        SLQ_LAUNCH_CHECK(ctx);
        SLQ_CUDA_CHECK(cudaMemcpyAsync(cnt, srow_ptr, sizeof(int64_t) * d, cudaMemcpyDeviceToDevice, ctx->stream));
        exclusive_scan(ctx, cnt, d, srow_ptr, scan_tmp);
        set_total_kernel<<<1, 32, 0, ctx->stream>>>(cnt, d, srow_ptr);
        SLQ_LAUNCH_CHECK(ctx);
        const int64_t nnz_s = static_cast<int64_t>(cc.plan.ent_stride) * cc.plan.nchunks;  // >= entries of S
        sent = static_cast<uint32_t*>(ws.ypart.ensure(sizeof(uint32_t) * nnz_s));
        srow_fill<<<wgrid, 256, 0, ctx->stream>>>(cc.ptr, cc.ent, cc.plan.ptr_stride, cc.plan.ent_stride,
                                                  cc.plan.nchunks, cc.plan.K, d, srow_ptr, sent);
        SLQ_LAUNCH_CHECK(ctx);
        check_chunk_csr(ctx, cc);
    }
    // column-slab gather (every Y row resident) unless the geometry rules it out
    const int G = ctx->num_sms;
    const int64_t rmax = ceil_div(d, static_cast<int64_t>(G));
    const int64_t budget = 200 * 1024 - 16 * rmax;
    int64_t w = budget > 0 ? budget / (8 * rmax) : 0;
    int S = w > 0 ? static_cast<int>(ceil_div(n + 1, w)) : 0;
    // diagnostics / tests: SLQ_K2S=row selects the row gather, SLQ_K2S_W caps the
    // slab width (more slabs at small sizes), SLQ_K2S_KWIN / SLQ_K2S_LAG the pacing
    const char* mode = std::getenv("SLQ_K2S");
    if (const char* e = std::getenv("SLQ_K2S_W")) {
        w = std::min<int64_t>(w, std::max<int64_t>(32, std::atoll(e)));
        S = w > 0 ? static_cast<int>(ceil_div(n + 1, w)) : 0;
    }
    if (w >= 32 && S >= 1 && S < 31 && n < (int64_t(1) << 24) && A->nnz < (int64_t(1) << kSlLenShift) &&
        !(mode && std::string(mode) == "row")) {
        w = ceil_div(n + 1, static_cast<int64_t>(S));  // balanced slabs
        slq_sparse* Am = const_cast<slq_sparse*>(A);     // the slab table is a cached derived layout
        if (!Am->s_valid) {  // the CSR was (re)written: every table is stale
            if (Am->s_ntab) {
                SLQ_CUDA_CHECK(cudaDeviceSynchronize());
                drop_slab_tables(Am);
            }
            Am->s_valid = true;
        }
        slq_sparse::SlabTable* tab = nullptr;
        for (int i = 0; i < Am->s_ntab; ++i)
            if (Am->s_tab[i].S == S && Am->s_tab[i].w == w) tab = &Am->s_tab[i];
        if (!tab) {
            if (Am->s_ntab == slq_sparse::kSlabTables) {  // rare: retire the oldest geometry
                SLQ_CUDA_CHECK(cudaDeviceSynchronize());
                cudaFree(Am->s_tab[0].p);
                cudaEventDestroy(Am->s_tab[0].ready);
                for (int i = 1; i < Am->s_ntab; ++i) Am->s_tab[i - 1] = Am->s_tab[i];
                Am->s_tab[--Am->s_ntab] = slq_sparse::SlabTable{};
            }
            tab = &Am->s_tab[Am->s_ntab];
            SLQ_CUDA_CHECK(cudaMalloc(&tab->p, sizeof(uint64_t) * m * S));
            SLQ_CUDA_CHECK(cudaEventCreateWithFlags(&tab->ready, cudaEventDisableTiming));
            slab_ptr_kernel<<<static_cast<unsigned>(ceil_div(m * 32, 256)), 256, 0, ctx->stream>>>(
                A->rowptr, A->colidx, m, S, static_cast<int>(w), tab->p);
            SLQ_LAUNCH_CHECK(ctx);
            SLQ_CUDA_CHECK(cudaEventRecord(tab->ready, ctx->stream));
            tab->S = S;
            tab->w = static_cast<int>(w);
            ++Am->s_ntab;
        }
        SLQ_CUDA_CHECK(cudaStreamWaitEvent(ctx->stream, tab->ready, 0));  // built on another stream, maybe
        const int64_t kwin_env = std::getenv("SLQ_K2S_KWIN") ? std::atoll(std::getenv("SLQ_K2S_KWIN")) : 0;
        const int lag_env = std::getenv("SLQ_K2S_LAG") ? std::atoi(std::getenv("SLQ_K2S_LAG")) : 0;
        const int64_t kwin = kwin_env > 0 ? kwin_env : (int64_t(1) << 18);
        const int nwin = static_cast<int>(ceil_div(m, kwin));
        const int lag = lag_env > 0 ? lag_env : 2;
        unsigned* sync = static_cast<unsigned*>(ws.flags.ensure(4096)) + 32;  // [32]: this kernel's counter
        SLQ_CUDA_CHECK(cudaMemsetAsync(sync, 0, sizeof(unsigned), ctx->stream));
        const size_t smem = sizeof(double) * rmax * w + 2 * sizeof(int64_t) * rmax;
        SLQ_CUDA_CHECK(cudaFuncSetAttribute(sparse_gather_slab_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(smem)));
        SlabArgs sa{tab->p, A->colidx, A->vals, A->b, n, d, m, S, static_cast<int>(w), static_cast<int>(rmax),
                    srow_ptr, sent, val, Y, kwin, nwin, lag, sync};
        void* args[] = {&sa};
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(static_cast<unsigned>(G));
        cfg.blockDim = dim3(32 * kSlW);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = ctx->stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeCooperative;  // the soft barrier needs every CTA resident
        at[0].val.cooperative = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        SLQ_CUDA_CHECK(cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(sparse_gather_slab_kernel), args));
        SLQ_LAUNCH_CHECK(ctx);
        return;
    }
    // row gather: one warp per Y row, rows of n+1 doubles in shared memory
    const int64_t row_bytes = (n + 1) * static_cast<int64_t>(sizeof(double));
    int warps = static_cast<int>(std::min<int64_t>(16, (200 * 1024) / row_bytes));
    if (warps < 1) fail(SLQ_UNSUPPORTED, "sparse sketch_apply: n too large for a shared-memory row");
    const size_t smem = static_cast<size_t>(warps) * row_bytes;
    SLQ_CUDA_CHECK(cudaFuncSetAttribute(sparse_gather_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(smem)));
    SGatherArgs g{A->rowptr, A->colidx, A->vals, A->b, n, d, srow_ptr, sent, val, Y, warps};
    sparse_gather_kernel<<<static_cast<unsigned>(ceil_div(d, warps)), 32 * warps, smem, ctx->stream>>>(g);
    SLQ_LAUNCH_CHECK(ctx);
}

namespace {

class SparseOp final : public PassOp {
public:
    SparseOp(slq_ctx* ctx, const slq_sparse* A, bool two_pass) : A_(A) {
        m = A->m;
        n = A->n;
        const int64_t zrow = n * static_cast<int64_t>(sizeof(double));
        const int64_t budget = 220 * 1024;
        // two-pass (u16 columns / row offsets): the u_hat pass holds its ring +
        // p in shared memory, the A^T u_hat pass a block's u_hat + column starts
        // (+ z when it fits; 1 KB left for static shared memory); else the single
        // fused pass with p + one z copy per warp in shared memory
        const int64_t smax = 226 * 1024;
        // ring: 2 = three tight 128-row stages (rows of <= 50 entries on average:
        // a third chunk in flight), 1 = two 128-row stages, 0 = two 64-row stages (wide p)
        const int64_t ringT = static_cast<int64_t>(UpT::kStage) * UpT::kStages;
        const int64_t ringG = static_cast<int64_t>(UpG::kStage) * UpG::kStages;
        const int64_t ringS = static_cast<int64_t>(UpS::kStage) * UpS::kStages;
        ring_ = ringT + zrow <= smax && A->nnz <= 50 * m ? 2 : ringG + zrow <= smax ? 1 : 0;
        if (const char* e = std::getenv("SLQ_UPASS_GEOM")) ring_ = std::min(ring_, std::atoi(e));  // diagnostics
        const int64_t ring = ring_ == 2 ? ringT : ring_ == 1 ? ringG : ringS;
        two_ = two_pass && slq_env_flag("SLQ_SPARSE_ONEPASS") == false &&
               static_cast<int64_t>(kTbRows) * 8 + 4 * (n + 8) <= smax && ring + zrow <= smax && n < 65536 && m > 0 &&
               A->nnz > 0;
        if (two_) {
            prepare_two_pass(ctx, const_cast<slq_sparse*>(A), true);
            nblk_ = A->t_nblk;
            blkcol_ = A->t_blkcol;
            crow_ = A->t_crow;
            cval_ = A->t_cval;
            us_ = A->t_uscr;
            col16_ = A->t_col16;
            smem_ = static_cast<size_t>(ring + zrow);
            grid_ = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ctx->num_sms, ceil_div(m, UpS::kRows))));
            // rows of <= 100 entries on average: 4 lanes per row (C4's 50: 2.97 -> 2.84 ms;
            // 200 entries: 2.80 vs 2.97 ms with 8 lanes)
            short_rows_ = A->nnz <= 100 * m;
            if (const char* e = std::getenv("SLQ_UPASS_LPR")) short_rows_ = std::atoi(e) == 4;  // diagnostics
            const void* kfn = ring_ == 2 ? (short_rows_ ? reinterpret_cast<const void*>(sparse_upass_kernel<UpT, 4>)
                                                        : reinterpret_cast<const void*>(sparse_upass_kernel<UpT, 8>))
                              : ring_ == 1 ? (short_rows_ ? reinterpret_cast<const void*>(sparse_upass_kernel<UpG, 4>)
                                                          : reinterpret_cast<const void*>(sparse_upass_kernel<UpG, 8>))
                                           : (short_rows_ ? reinterpret_cast<const void*>(sparse_upass_kernel<UpS, 4>)
                                                          : reinterpret_cast<const void*>(sparse_upass_kernel<UpS, 8>));
            SLQ_CUDA_CHECK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_)));
            tsmem_ = static_cast<size_t>(kTbRows) * 8 + static_cast<size_t>(n + 8) * 4;
            z_smem_ = static_cast<int64_t>(tsmem_) + zrow + 32 <= smax;
            if (z_smem_) tsmem_ += static_cast<size_t>(zrow) + 32;
            SLQ_CUDA_CHECK(cudaFuncSetAttribute(sparse_tpass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                static_cast<int>(tsmem_)));
            return;
        }
        W_ = static_cast<int>(std::min<int64_t>(kSpMaxWarps, budget / std::max<int64_t>(zrow, 1) - 1));
        if (W_ < 1) fail(SLQ_UNSUPPORTED, "sparse lsqr: n too large for shared-memory z copies");
        smem_ = static_cast<size_t>(zrow) * (W_ + 1);
        grid_ = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ctx->num_sms, ceil_div(std::max<int64_t>(m, 1), 4 * W_))));
        SLQ_CUDA_CHECK(cudaFuncSetAttribute(sparse_pass_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(smem_)));
    }
    int grid() const override { return grid_; }
    void ready(slq_ctx* ctx) const override {
        slq_sparse* A = const_cast<slq_sparse*>(A_);
        if (two_ && A->t_pending) {
            SLQ_CUDA_CHECK(cudaStreamWaitEvent(ctx->stream, A->t_ready, 0));
            A->t_pending = false;
        }
    }
    void pass(slq_ctx* ctx, const PassCall& c) const override {
        if (!c.u_in && !A_->b) fail(SLQ_INVALID_ARG, "sparse lsqr: no right-hand side");
        if (!two_) {
            SPassArgs a{A_->rowptr, A_->colidx, A_->vals, A_->b, m, n, c.p, c.u_in, c.u_out, c.coef, c.c_fixed,
                        c.part, c.want_z, c.skip};
            sparse_pass_kernel<true><<<grid_, 32 * W_, smem_, ctx->stream>>>(a);
            SLQ_LAUNCH_CHECK(ctx);
            return;
        }
        // the z pass reads u_hat back: callers that do not keep it get a scratch vector
        double* uo = c.u_out ? c.u_out : us_;
        UPassArgs ua{A_->rowptr, col16_, A_->vals, A_->b, m, n, c.p, c.u_in, uo, c.coef, c.c_fixed, c.part, c.skip};
        const dim3 ub(32 * (kUpConsumers + 1));
        if (ring_ == 2) {
            if (short_rows_) sparse_upass_kernel<UpT, 4><<<grid_, ub, smem_, ctx->stream>>>(ua);
            else sparse_upass_kernel<UpT, 8><<<grid_, ub, smem_, ctx->stream>>>(ua);
        } else if (ring_ == 1) {
            if (short_rows_) sparse_upass_kernel<UpG, 4><<<grid_, ub, smem_, ctx->stream>>>(ua);
            else sparse_upass_kernel<UpG, 8><<<grid_, ub, smem_, ctx->stream>>>(ua);
        } else {
            if (short_rows_) sparse_upass_kernel<UpS, 4><<<grid_, ub, smem_, ctx->stream>>>(ua);
            else sparse_upass_kernel<UpS, 8><<<grid_, ub, smem_, ctx->stream>>>(ua);
        }
        SLQ_LAUNCH_CHECK(ctx);
        TPassArgs t{A_->rowptr, blkcol_, crow_, cval_, uo, m, n, nblk_, c.part, c.want_z, c.skip, z_smem_ ? 1 : 0};
        sparse_tpass_kernel<<<grid_, 1024, tsmem_, ctx->stream>>>(t);
        SLQ_LAUNCH_CHECK(ctx);
    }
    std::vector<uint64_t> key() const override {
        return {2, reinterpret_cast<uint64_t>(A_->rowptr), reinterpret_cast<uint64_t>(A_->colidx),
                reinterpret_cast<uint64_t>(A_->vals), reinterpret_cast<uint64_t>(A_->b), static_cast<uint64_t>(m),
                static_cast<uint64_t>(n), static_cast<uint64_t>(W_), static_cast<uint64_t>(grid_),
                reinterpret_cast<uint64_t>(crow_), reinterpret_cast<uint64_t>(cval_), reinterpret_cast<uint64_t>(blkcol_),
                reinterpret_cast<uint64_t>(us_), reinterpret_cast<uint64_t>(col16_),
                static_cast<uint64_t>(two_) | static_cast<uint64_t>(ring_) << 1 | static_cast<uint64_t>(short_rows_) << 3 |
                    static_cast<uint64_t>(z_smem_) << 4};
    }
    // algorithmic bytes: one read of the CSR (the operator's data) + u in, u_hat out
    double pass_bytes() const override { return 12.0 * A_->nnz + 8.0 * (m + 1) + 16.0 * m; }

private:
    const slq_sparse* A_;
    int W_ = 8, grid_ = 1;
    size_t smem_ = 0, tsmem_ = 0;
    bool two_ = false;
    int64_t nblk_ = 0;
    double* us_ = nullptr;
    const uint16_t* col16_ = nullptr;
    // 128-row chunks, two 84 KB stages: measured against 64 x 4, 96 x 3 and
    // 160 x 2 at C4 (1.6 ms vs 2.05 / 1.9 / 1.7 ms for the u_hat pass)
    using UpG = UpGeom<128, 8192, 2>;
    using UpT = UpGeom<128, 6656, 3>;  // <= 52 entries per row fit a stage
    using UpS = UpGeom<64, 4096, 2>;  // wide p (n > ~7900): a smaller ring
    int ring_ = 1;
    bool z_smem_ = true;
    bool short_rows_ = false;
    uint32_t* blkcol_ = nullptr;
    uint16_t* crow_ = nullptr;
    double* cval_ = nullptr;
};

}  // namespace

std::unique_ptr<PassOp> make_sparse_op(slq_ctx* ctx, const slq_sparse* A, bool two_pass) {
    return std::unique_ptr<PassOp>(new SparseOp(ctx, A, two_pass));
}

}  // namespace slq
