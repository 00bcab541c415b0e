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
#include <cmath>
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
            const uint32_t my_en = lane < nb ? g.sent[e + lane] : 0u;
            const int64_t my_k = my_en & 0x7fffffffu;
            const int64_t my_rb = lane < nb ? g.rowptr[my_k] : 0;
            const int64_t my_re = lane < nb ? g.rowptr[my_k + 1] : 0;
            const double my_b = (g.b && lane < nb) ? g.b[my_k] : 0.0;
            // round 3: every row's (column, value) pairs
            int32_t cc[kSgB][2];
            double vv[kSgB][2];
            int64_t rb[kSgB], re[kSgB];
#pragma unroll
            for (int q = 0; q < kSgB; ++q) {
                rb[q] = __shfl_sync(0xffffffffu, my_rb, q);
                re[q] = __shfl_sync(0xffffffffu, my_re, q);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int64_t t = rb[q] + lane + 32 * h;
                    const bool ok = t < re[q];
                    cc[q][h] = ok ? g.colidx[t] : -1;
                    vv[q][h] = ok ? g.vals[t] : 0.0;
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
                    if (cc[q][h] >= 0) y[cc[q][h]] = __dadd_rn(y[cc[q][h]], __dmul_rn(sv, vv[q][h]));
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
    if (a.want_z) {
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

__global__ void __launch_bounds__(32 * kSpMaxWarps, 1) sparse_pass_kernel(SPassArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    if (a.skip && *a.skip) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int W = blockDim.x >> 5;
    const int64_t n = a.n;
    double* p_s = reinterpret_cast<double*>(smem);
    double* z_s = p_s + n;
    for (int64_t j = tid; j < n; j += blockDim.x) p_s[j] = a.p[j];
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
        sp_step(a, x, q, qa, qc, rp_next, ssq);
        q += W;
        if (q >= nq) break;
        sp_step(a, x, q, qb, qa, rp_next, ssq);
        q += W;
        if (q >= nq) break;
        sp_step(a, x, q, qc, qb, rp_next, ssq);
        q += W;
    }
    // ssq: lanes 0, 8, 16, 24 hold partial sums
    ssq += __shfl_xor_sync(0xffffffffu, ssq, 8);
    ssq += __shfl_xor_sync(0xffffffffu, ssq, 16);
    __shared__ double red[kSpMaxWarps];  // own array: p's n doubles may be fewer than the warps
    if (lane == 0) red[warp] = ssq;
    __syncthreads();
    double* outp = a.part + static_cast<int64_t>(blockIdx.x) * (n + 1);
    if (a.want_z)
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

void sparse_free(slq_sparse* A) {
    if (A->owned) {
        cudaFree(A->rowptr);
        cudaFree(A->colidx);
        cudaFree(A->vals);
        cudaFree(A->b);
    }
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
    ChunkCsr cc = build_chunk_csr(ctx, compact, colptr_dev, zeta_max, m, d, 0);
    // S^T rows (entries of each Y row in ascending k)
    DevBuf srp, scan_tmp;
    int64_t* srow_ptr = static_cast<int64_t*>(srp.ensure(sizeof(int64_t) * (d + 1)));
    const unsigned wgrid = static_cast<unsigned>(ceil_div(d * 32, 256));
    srow_count<<<wgrid, 256, 0, ctx->stream>>>(cc.ptr, cc.plan.ptr_stride, cc.plan.nchunks, d, srow_ptr);
    SLQ_LAUNCH_CHECK(ctx);
    DevBuf cnt_copy;
    int64_t* cnt = static_cast<int64_t*>(cnt_copy.ensure(sizeof(int64_t) * (d + 1)));
    SLQ_CUDA_CHECK(cudaMemcpyAsync(cnt, srow_ptr, sizeof(int64_t) * d, cudaMemcpyDeviceToDevice, ctx->stream));
    exclusive_scan(ctx, cnt, d, srow_ptr, scan_tmp);
    set_total_kernel<<<1, 32, 0, ctx->stream>>>(cnt, d, srow_ptr);
    SLQ_LAUNCH_CHECK(ctx);
    const int64_t nnz_s = static_cast<int64_t>(cc.plan.ent_stride) * cc.plan.nchunks;  // >= entries of S
    uint32_t* sent = static_cast<uint32_t*>(ws.ypart.ensure(sizeof(uint32_t) * nnz_s));
    srow_fill<<<wgrid, 256, 0, ctx->stream>>>(cc.ptr, cc.ent, cc.plan.ptr_stride, cc.plan.ent_stride, cc.plan.nchunks,
                                              cc.plan.K, d, srow_ptr, sent);
    SLQ_LAUNCH_CHECK(ctx);
    check_chunk_csr(ctx, cc);
    // gather: one warp per Y row, rows of n+1 doubles in shared memory
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
    SparseOp(slq_ctx* ctx, const slq_sparse* A) : A_(A) {
        m = A->m;
        n = A->n;
        // p + one z copy per warp in shared memory
        const int64_t zrow = n * static_cast<int64_t>(sizeof(double));
        const int64_t budget = 220 * 1024;
        W_ = static_cast<int>(std::min<int64_t>(kSpMaxWarps, budget / std::max<int64_t>(zrow, 1) - 1));
        if (W_ < 1) fail(SLQ_UNSUPPORTED, "sparse lsqr: n too large for shared-memory z copies");
        smem_ = static_cast<size_t>(zrow) * (W_ + 1);
        grid_ = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ctx->num_sms, ceil_div(std::max<int64_t>(m, 1), 4 * W_))));
        SLQ_CUDA_CHECK(cudaFuncSetAttribute(sparse_pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(smem_)));
    }
    int grid() const override { return grid_; }
    void pass(slq_ctx* ctx, const PassCall& c) const override {
        if (!c.u_in && !A_->b) fail(SLQ_INVALID_ARG, "sparse lsqr: no right-hand side");
        SPassArgs a{A_->rowptr, A_->colidx, A_->vals, A_->b, m, n, c.p, c.u_in, c.u_out, c.coef, c.c_fixed,
                    c.part, c.want_z, c.skip};
        sparse_pass_kernel<<<grid_, 32 * W_, smem_, ctx->stream>>>(a);
        SLQ_LAUNCH_CHECK(ctx);
    }
    std::vector<uint64_t> key() const override {
        return {2, reinterpret_cast<uint64_t>(A_->rowptr), reinterpret_cast<uint64_t>(A_->colidx),
                reinterpret_cast<uint64_t>(A_->vals), reinterpret_cast<uint64_t>(A_->b), static_cast<uint64_t>(m),
                static_cast<uint64_t>(n), static_cast<uint64_t>(W_), static_cast<uint64_t>(grid_)};
    }
    double pass_bytes() const override { return 12.0 * A_->nnz + 8.0 * (m + 1) + 16.0 * m; }

private:
    const slq_sparse* A_;
    int W_ = 8, grid_ = 1;
    size_t smem_ = 0;
};

}  // namespace

std::unique_ptr<PassOp> make_sparse_op(slq_ctx* ctx, const slq_sparse* A) {
    return std::unique_ptr<PassOp>(new SparseOp(ctx, A));
}

}  // namespace slq
