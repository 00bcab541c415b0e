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
//   K4s  one pass per LSQR iteration: row tiles (column indices, values, row
//        pointers, u) arrive by TMA bulk copy into a 3-stage mbarrier ring; a
//        warp per row computes u_hat = A_i p + c u_i (p in shared memory) and
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

__global__ void max_tile_nnz_kernel(const int64_t* rowptr, int64_t m, int R, unsigned long long* out) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t r0 = t * R;
    if (r0 >= m) return;
    const int64_t r1 = min(m, r0 + R);
    const int64_t base = rowptr[r0] & ~int64_t(3);
    const int64_t cnt = ((rowptr[r1] - base) + 3) & ~int64_t(3);
    atomicMax(out, static_cast<unsigned long long>(cnt));
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
// in ascending k; the (column, value) pairs of 4 consecutive A rows are
// loaded before they are applied (loads in flight), then added row by row.
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
        for (int64_t e = e0; e < e1; e += 4) {
            const int nb = (e1 - e < 4) ? static_cast<int>(e1 - e) : 4;
            uint32_t en[4];
            int64_t rb[4], re[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                en[q] = q < nb ? g.sent[e + q] : 0u;
                const int64_t k = en[q] & 0x7fffffffu;
                rb[q] = q < nb ? g.rowptr[k] : 0;
                re[q] = q < nb ? g.rowptr[k + 1] : 0;
            }
            int32_t cc[4][2];
            double vv[4][2];
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int64_t t = rb[q] + lane + 32 * h;
                    const bool ok = t < re[q];
                    cc[q][h] = ok ? g.colidx[t] : -1;
                    vv[q][h] = ok ? g.vals[t] : 0.0;
                }
            double bq[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) bq[q] = (g.b && q < nb && lane == 0) ? g.b[en[q] & 0x7fffffffu] : 0.0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (q >= nb) break;
                const double s = (en[q] >> 31) ? -g.val : g.val;
                // csc_matrix.hpp:133: yj[row] += S_val * akj (two roundings)
#pragma unroll
                for (int h = 0; h < 2; ++h)
                    if (cc[q][h] >= 0) y[cc[q][h]] = __dadd_rn(y[cc[q][h]], __dmul_rn(s, vv[q][h]));
                for (int64_t t = rb[q] + 64 + lane; t < re[q]; t += 32) {  // rows longer than 64
                    const int32_t c = g.colidx[t];
                    y[c] = __dadd_rn(y[c], __dmul_rn(s, g.vals[t]));
                }
                if (lane == 0 && g.b && bq[q] != 0.0) y[g.n] = __dadd_rn(y[g.n], __dmul_rn(s, bq[q]));
                __syncwarp();
            }
        }
        for (int64_t j = lane; j < n1; j += 32) g.Y[j * g.d + r] = y[j];
    }
}

// ------------------------------------------------------------ K4s pass

using namespace ptx;

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
    int R, S, W;          // rows per tile, stages, consumer warps (= z copies)
    int64_t cap;          // nnz capacity of a stage (multiple of 4)
};

__global__ void __launch_bounds__(288, 1) sparse_pass_kernel(SPassArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    if (a.skip && *a.skip) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int W = a.W;
    const int64_t n = a.n;
    // layout: stages [S] x {vals cap f64 | cols cap i32 | rowptr R+2 i64 | u R f64}, p[n], z[W][n], bars
    const size_t st_vals = static_cast<size_t>(a.cap) * 8, st_cols = static_cast<size_t>(a.cap) * 4;
    const size_t st_rp = static_cast<size_t>(a.R + 2) * 8, st_u = static_cast<size_t>(a.R) * 8;
    const size_t st_bytes = st_vals + st_cols + st_rp + st_u;
    double* p_s = reinterpret_cast<double*>(smem + a.S * st_bytes);
    double* z_s = p_s + n;
    uint64_t* full = reinterpret_cast<uint64_t*>(z_s + static_cast<int64_t>(W) * n);
    uint64_t* empty = full + a.S;

    const int64_t ntiles = (a.m + a.R - 1) / a.R;
    const int64_t t0 = blockIdx.x * ntiles / gridDim.x;
    const int64_t t1 = (blockIdx.x + 1) * ntiles / gridDim.x;
    const int64_t nt = t1 - t0;

    if (tid == 0) {
        for (int s = 0; s < a.S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], W);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    for (int64_t j = tid; j < n; j += blockDim.x) p_s[j] = a.p[j];
    for (int64_t j = tid; j < static_cast<int64_t>(W) * n; j += blockDim.x) z_s[j] = 0.0;
    __syncthreads();

    double ssq = 0.0;
    const double* ubase = a.u_in ? a.u_in : a.b;
    if (warp == W) {
        // producer: the tile bounds (two row pointers each) are prefetched 32
        // tiles at a time by the warp's lanes, so issuing a tile's copies never
        // waits on a dependent global load
        int s = -1;
        unsigned ph = 1;
        int64_t pre_lo = 0, pre_hi = 0;
        for (int64_t k = 0; k < nt; ++k) {
            if ((k & 31) == 0) {
                const int64_t kk = k + lane;
                if (kk < nt) {
                    const int64_t r0 = (t0 + kk) * a.R;
                    pre_lo = a.rowptr[r0];
                    pre_hi = a.rowptr[min(a.m, r0 + a.R)];
                }
            }
            const int64_t lo = __shfl_sync(0xffffffffu, pre_lo, static_cast<int>(k & 31));
            const int64_t hi = __shfl_sync(0xffffffffu, pre_hi, static_cast<int>(k & 31));
            if (++s == a.S) {
                s = 0;
                ph ^= 1u;
            }
            if (lane == 0) {
                if (k >= a.S) mbar_wait(&empty[s], ph);
                const int64_t row0 = (t0 + k) * a.R;
                const int64_t base = lo & ~int64_t(3);
                const int64_t cnt = ((hi - base) + 3) & ~int64_t(3);
                unsigned char* st = smem + s * st_bytes;
                const unsigned bytes = static_cast<unsigned>(cnt * 8 + cnt * 4 + st_rp + st_u);
                mbar_expect_tx(&full[s], bytes);
                if (cnt > 0) {
                    bulk_g2s(st, a.vals + base, static_cast<unsigned>(cnt * 8), &full[s]);
                    bulk_g2s(st + st_vals, a.colidx + base, static_cast<unsigned>(cnt * 4), &full[s]);
                }
                bulk_g2s(st + st_vals + st_cols, a.rowptr + row0, static_cast<unsigned>(st_rp), &full[s]);
                bulk_g2s(st + st_vals + st_cols + st_rp, ubase + row0, static_cast<unsigned>(st_u), &full[s]);
            }
            __syncwarp();
        }
    } else {
        const double c = a.coef ? *a.coef : a.c_fixed;
        double* zw = z_s + static_cast<int64_t>(warp) * n;
        int s = -1;
        unsigned ph = 1;
        for (int64_t k = 0; k < nt; ++k) {
            if (++s == a.S) {
                s = 0;
                ph ^= 1u;
            }
            mbar_wait(&full[s], ph ^ 1u);
            const unsigned char* st = smem + s * st_bytes;
            const double* sv = reinterpret_cast<const double*>(st);
            const int32_t* sc = reinterpret_cast<const int32_t*>(st + st_vals);
            const int64_t* srp = reinterpret_cast<const int64_t*>(st + st_vals + st_cols);
            const double* su = reinterpret_cast<const double*>(st + st_vals + st_cols + st_rp);
            const int64_t row0 = (t0 + k) * a.R;
            const int rows = static_cast<int>(min(static_cast<int64_t>(a.R), a.m - row0));
            const int64_t base = srp[0] & ~int64_t(3);
            // four rows per warp step, eight lanes per row for A p (three
            // independent reduction trees in flight instead of one), then the
            // rows' A^T u_hat scatter one row at a time with all lanes (rows
            // may share columns; a row's columns are distinct, so lanes never
            // collide inside one scatter)
            const int g = lane >> 3, sub = lane & 7;
            for (int i0 = warp * 4; i0 < rows; i0 += 4 * W) {
                const int i = i0 + g;
                const bool rv = i < rows;
                const int b0 = rv ? static_cast<int>(srp[i] - base) : 0;
                const int b1 = rv ? static_cast<int>(srp[i + 1] - base) : 0;
                double acc = 0.0;
                for (int t = b0 + sub; t < b1; t += 8) acc = fma(sv[t], p_s[sc[t]], acc);
                acc += __shfl_xor_sync(0xffffffffu, acc, 4);
                acc += __shfl_xor_sync(0xffffffffu, acc, 2);
                acc += __shfl_xor_sync(0xffffffffu, acc, 1);
                const double uh = rv ? __dadd_rn(acc, __dmul_rn(c, su[i])) : 0.0;
                if (rv && sub == 0) {
                    if (a.u_out) a.u_out[row0 + i] = uh;
                    ssq = fma(uh, uh, ssq);
                }
                if (a.want_z) {
                    const int ng = rows - i0 < 4 ? rows - i0 : 4;
                    for (int gg = 0; gg < ng; ++gg) {
                        const double ug = __shfl_sync(0xffffffffu, uh, gg * 8);
                        const int c0 = __shfl_sync(0xffffffffu, b0, gg * 8), c1 = __shfl_sync(0xffffffffu, b1, gg * 8);
                        // first 64 entries with both loads issued before the
                        // read-modify-writes (a row's columns are distinct)
                        const int ta = c0 + lane, tb = c0 + 32 + lane;
                        const bool oka = ta < c1, okb = tb < c1;
                        const int ca = oka ? sc[ta] : 0, cb = okb ? sc[tb] : 0;
                        const double va = oka ? sv[ta] : 0.0, vb = okb ? sv[tb] : 0.0;
                        const double za = oka ? zw[ca] : 0.0, zb = okb ? zw[cb] : 0.0;
                        if (oka) zw[ca] = fma(va, ug, za);
                        if (okb) zw[cb] = fma(vb, ug, zb);
                        for (int t = c0 + 64 + lane; t < c1; t += 32) zw[sc[t]] = fma(sv[t], ug, zw[sc[t]]);
                        __syncwarp();
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
    }
    __syncthreads();
    double* red = reinterpret_cast<double*>(smem);  // stage memory is free now
    ssq += __shfl_xor_sync(0xffffffffu, ssq, 8);     // lanes 0, 8, 16, 24 hold the row-group sums
    ssq += __shfl_xor_sync(0xffffffffu, ssq, 16);
    if (warp < W && lane == 0) red[warp] = ssq;
    __syncthreads();
    double* outp = a.part + static_cast<int64_t>(blockIdx.x) * (n + 1);
    if (a.want_z)
        for (int64_t j = tid; j < n; j += blockDim.x) {
            double s = 0.0;
            for (int q = 0; q < W; ++q) s += z_s[static_cast<int64_t>(q) * n + j];
            outp[j] = s;
        }
    if (tid == 0) {
        double s = 0.0;
        for (int q = 0; q < W; ++q) s += red[q];
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
    ChunkCsr cc = build_chunk_csr(ctx, compact, colptr_dev, zeta_max, m, d, false);
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
    SLQ_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
}

namespace {

class SparseOp final : public PassOp {
public:
    SparseOp(slq_ctx* ctx, const slq_sparse* A) : A_(A) {
        m = A->m;
        n = A->n;
        // z copies (one per consumer warp) + p in shared memory; stages take the rest
        const int64_t zrow = n * static_cast<int64_t>(sizeof(double));
        W_ = static_cast<int>(std::min<int64_t>(8, (150 * 1024) / std::max<int64_t>(zrow, 1) - 1));
        if (W_ < 1) fail(SLQ_UNSUPPORTED, "sparse lsqr: n too large for shared-memory z copies");
        R_ = 32;
        S_ = 3;
        // stage capacity = max nnz of a tile (16-byte-rounded range)
        DevBuf mx;
        unsigned long long* dmx = static_cast<unsigned long long*>(mx.ensure(8));
        SLQ_CUDA_CHECK(cudaMemsetAsync(dmx, 0, 8, ctx->stream));
        const int64_t ntiles = ceil_div(std::max<int64_t>(m, 1), R_);
        if (m > 0) {
            max_tile_nnz_kernel<<<static_cast<unsigned>(ceil_div(ntiles, 256)), 256, 0, ctx->stream>>>(A->rowptr, m, R_,
                                                                                                    dmx);
            SLQ_LAUNCH_CHECK(ctx);
        }
        unsigned long long h = 0;
        SLQ_CUDA_CHECK(cudaMemcpyAsync(&h, dmx, 8, cudaMemcpyDeviceToHost, ctx->stream));
        SLQ_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        cap_ = std::max<int64_t>(4, static_cast<int64_t>(h));
        const size_t fixed = static_cast<size_t>(zrow) * (W_ + 1) + 2 * S_ * sizeof(uint64_t) + 64;
        auto stage = [&](int64_t cap) { return static_cast<size_t>(cap * 12 + (R_ + 2) * 8 + R_ * 8); };
        while (fixed + S_ * stage(cap_) > 227 * 1024 && S_ > 2) --S_;
        smem_ = fixed + S_ * stage(cap_);
        if (smem_ > 227 * 1024) fail(SLQ_UNSUPPORTED, "sparse lsqr: row tile too dense for shared memory");
        grid_ = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ctx->num_sms, ntiles)));
        SLQ_CUDA_CHECK(cudaFuncSetAttribute(sparse_pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(smem_)));
    }
    int grid() const override { return grid_; }
    void pass(slq_ctx* ctx, const PassCall& c) const override {
        if (!c.u_in && !A_->b) fail(SLQ_INVALID_ARG, "sparse lsqr: no right-hand side");
        SPassArgs a{A_->rowptr, A_->colidx, A_->vals, A_->b, m, n, c.p, c.u_in, c.u_out, c.coef, c.c_fixed,
                    c.part, c.want_z, c.skip, R_, S_, W_, cap_};
        sparse_pass_kernel<<<grid_, 32 * (W_ + 1), smem_, ctx->stream>>>(a);
        SLQ_LAUNCH_CHECK(ctx);
    }
    std::vector<uint64_t> key() const override {
        return {2, reinterpret_cast<uint64_t>(A_->rowptr), reinterpret_cast<uint64_t>(A_->colidx),
                reinterpret_cast<uint64_t>(A_->vals), reinterpret_cast<uint64_t>(A_->b), static_cast<uint64_t>(m),
                static_cast<uint64_t>(n), static_cast<uint64_t>(cap_), static_cast<uint64_t>(grid_)};
    }
    double pass_bytes() const override { return 12.0 * A_->nnz + 8.0 * (m + 1) + 16.0 * m; }

private:
    const slq_sparse* A_;
    int W_ = 8, R_ = 32, S_ = 3, grid_ = 1;
    int64_t cap_ = 4;
    size_t smem_ = 0;
};

}  // namespace

std::unique_ptr<PassOp> make_sparse_op(slq_ctx* ctx, const slq_sparse* A) {
    return std::unique_ptr<PassOp>(new SparseOp(ctx, A));
}

}  // namespace slq
