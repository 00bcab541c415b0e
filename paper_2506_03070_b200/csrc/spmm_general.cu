// spmm_general.cu -- spmm(csc, dense) / spmm(csc, csc) for a CSC left factor
// with ARBITRARY values (csc_matrix.hpp:103-136), in the reference's
// accumulation order.  The sketch kernels (sketch.cu, sparse.cu) cover the
// sparse-sign case (one magnitude +-v, generated or bucketed per chunk); this
// path serves the rest of the reference's spmm contract (e.g. its
// entry-exact test, test_core_linalg.cpp:192-224).  Not on the solve path.
//
// Order: Y[r, j] = sum over (k ascending, then the stored order within column
// k) of S[r, k] * A[k, j], IEEE multiply then add, starting from +0; the dense
// form skips A[k, j] == 0 like the reference.  The entries of S are sorted by
// row with a STABLE radix sort of their positions p (CSC order = (k, stored
// order)), so each Y entry is one thread's ascending walk: bit-identical.
#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"
#include "spmm_general.cuh"

namespace slq {

namespace {

// flags[0] |= some |value| differs from |values[0]|; flags[1] |= row out of range
__global__ void csc_check_kernel(const int64_t* rows, const double* vals, int64_t nnz, int64_t d, int* flags) {
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= nnz) return;
    if (fabs(vals[e]) != fabs(vals[0])) flags[0] = 1;
    if (rows[e] < 0 || rows[e] >= d) flags[1] = 1;
}

__global__ void iota_kernel(int64_t* p, int64_t n) {
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e < n) p[e] = e;
}

// column index of every stored entry of the CSC
__global__ void expand_cols_kernel(const int64_t* colptr, int64_t m, int64_t* colk) {
    const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= m) return;
    for (int64_t p = colptr[k]; p < colptr[k + 1]; ++p) colk[p] = k;
}

// row pointers of the row-sorted entries: rp[r] = first sorted position with row >= r
__global__ void row_ptr_kernel(const int64_t* srow, int64_t nnz, int64_t d, int64_t* rp) {
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e > nnz) return;
    const int64_t hi = e < nnz ? srow[e] : d;
    const int64_t lo = e > 0 ? srow[e - 1] + 1 : 0;
    for (int64_t r = lo; r <= hi && r <= d; ++r) rp[r] = e;
}

// thread (r, j): Y[r, j] over the row's entries (ascending (k, p)); A row-major (ld)
__global__ void spmm_gen_dense_kernel(int64_t d, int64_t n, const int64_t* rp, const int64_t* perm,
                                      const int64_t* colk, const double* vals, const double* A, int64_t ld,
                                      double* Y) {
    const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t r = blockIdx.y;
    if (j >= n || r >= d) return;
    double acc = 0.0;
    for (int64_t e = rp[r]; e < rp[r + 1]; ++e) {
        const int64_t p = perm[e];
        const double a = A[colk[p] * ld + j];
        if (a != 0.0) acc = __dadd_rn(acc, __dmul_rn(vals[p], a));
    }
    Y[j * d + r] = acc;
}

// thread (r, j): merge S's row r (ascending k) with A's column j (ascending rows)
__global__ void spmm_gen_csc_kernel(int64_t d, int64_t n, const int64_t* rp, const int64_t* perm,
                                    const int64_t* colk, const double* vals, const int64_t* acp,
                                    const int64_t* arows, const double* avals, double* Y) {
    const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t r = blockIdx.y;
    if (j >= n || r >= d) return;
    double acc = 0.0;
    int64_t e = rp[r];
    const int64_t ee = rp[r + 1];
    for (int64_t q = acp[j]; q < acp[j + 1] && e < ee; ++q) {
        const int64_t k = arows[q];
        while (e < ee && colk[perm[e]] < k) ++e;
        for (int64_t f = e; f < ee && colk[perm[f]] == k; ++f) acc = __dadd_rn(acc, __dmul_rn(vals[perm[f]], avals[q]));
    }
    Y[j * d + r] = acc;
}

}  // namespace

SpmmCheck csc_check_dev(slq_ctx* ctx, const int64_t* rows, const double* vals, int64_t nnz, int64_t d) {
    SpmmCheck out{};
    if (nnz == 0) return out;
    DevBuf f;
    int* flags = static_cast<int*>(f.ensure(2 * sizeof(int)));
    SLQ_CUDA_CHECK(cudaMemsetAsync(flags, 0, 2 * sizeof(int), ctx->stream));
    csc_check_kernel<<<static_cast<unsigned>(ceil_div(nnz, 256)), 256, 0, ctx->stream>>>(rows, vals, nnz, d, flags);
    SLQ_LAUNCH_CHECK(ctx);
    int h[2] = {0, 0};
    SLQ_CUDA_CHECK(cudaMemcpyAsync(h, flags, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    SLQ_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    out.mixed_magnitudes = h[0] != 0;
    out.row_out_of_range = h[1] != 0;
    return out;
}

void spmm_general_dev(slq_ctx* ctx, int64_t d, int64_t m, int64_t nnz, const int64_t* rows, const double* vals,
                      const int64_t* colptr, int64_t n, const double* A_rows, int64_t ld, const int64_t* acp,
                      const int64_t* arows, const double* avals, double* Y) {
    if (d == 0 || n == 0) return;
    if (nnz == 0) {
        SLQ_CUDA_CHECK(cudaMemsetAsync(Y, 0, sizeof(double) * d * n, ctx->stream));
        return;
    }
    DevBuf bp, bp2, bk, bk2, bc, brp, btmp;
    int64_t* p_in = static_cast<int64_t*>(bp.ensure(sizeof(int64_t) * nnz));
    int64_t* perm = static_cast<int64_t*>(bp2.ensure(sizeof(int64_t) * nnz));
    int64_t* srow = static_cast<int64_t*>(bk2.ensure(sizeof(int64_t) * nnz));
    int64_t* colk = static_cast<int64_t*>(bc.ensure(sizeof(int64_t) * nnz));
    int64_t* rp = static_cast<int64_t*>(brp.ensure(sizeof(int64_t) * (d + 1)));
    (void)bk;
    const unsigned g = static_cast<unsigned>(ceil_div(nnz, 256));
    iota_kernel<<<g, 256, 0, ctx->stream>>>(p_in, nnz);
    SLQ_LAUNCH_CHECK(ctx);
    expand_cols_kernel<<<static_cast<unsigned>(ceil_div(std::max<int64_t>(m, 1), 256)), 256, 0, ctx->stream>>>(colptr, m,
                                                                                                            colk);
    SLQ_LAUNCH_CHECK(ctx);
    // stable sort of positions by row: equal rows keep (k, stored) order
    int bits = 1;
    while (bits < 63 && (int64_t(1) << bits) <= d) ++bits;
    size_t tb = 0;
    SLQ_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tb, rows, srow, p_in, perm, nnz, 0, bits, ctx->stream));
    void* tmp = btmp.ensure(std::max<size_t>(tb, 16));
    SLQ_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(tmp, tb, rows, srow, p_in, perm, nnz, 0, bits, ctx->stream));
    row_ptr_kernel<<<static_cast<unsigned>(ceil_div(nnz + 1, 256)), 256, 0, ctx->stream>>>(srow, nnz, d, rp);
    SLQ_LAUNCH_CHECK(ctx);
    const dim3 grid(static_cast<unsigned>(ceil_div(n, 128)), static_cast<unsigned>(d));
    if (A_rows) {
        spmm_gen_dense_kernel<<<grid, 128, 0, ctx->stream>>>(d, n, rp, perm, colk, vals, A_rows, ld, Y);
    } else {
        spmm_gen_csc_kernel<<<grid, 128, 0, ctx->stream>>>(d, n, rp, perm, colk, vals, acp, arows, avals, Y);
    }
    SLQ_LAUNCH_CHECK(ctx);
    SLQ_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
}

}  // namespace slq
