// sketch.cuh -- host entry points of the sparse-sign sketch kernels (K1, K2).
#pragma once

#include "common.cuh"

namespace slq {

// Chunk-CSR of a sparse sign sketch (K2's bucketed form): for every chunk of
// K consecutive sketch columns (= A rows), the entries sorted by (target row
// r, column k) as u16 (k_local << 1 | negative) with u16 row pointers.
struct ChunkPlan {
    int K, KB, cap;
    int64_t nchunks, ptr_stride, ent_stride;
};
struct ChunkCsr {
    ChunkPlan plan;
    uint16_t* ptr = nullptr;
    uint16_t* ent = nullptr;
    int* flag = nullptr;
};
// gather_width W = 4 / 2 / 1: entries encoded for the dense gather of W-column
// slabs (smem byte offset | neg); 0: (k_local << 1 | neg) for the sparse path.
ChunkCsr build_chunk_csr(slq_ctx* ctx, const uint32_t* compact, const int64_t* colptr_dev, int64_t zeta_max,
                         int64_t m, int64_t d, int gather_width);
void check_chunk_csr(slq_ctx* ctx, const ChunkCsr& cc);

// K1: sparse-sign generator for global columns [col_begin, col_begin+ncols).
// Outputs (device pointers, each optional): compact u32 entries, reference
// CSC (rows64 / vals / colptr), stats[2] (u64 counters, accumulated).
void generate_sparse_sign_dev(slq_ctx* ctx, int64_t d, int64_t zeta, uint64_t seed,
                              int64_t col_begin, int64_t ncols, uint32_t* compact,
                              int64_t* rows64, double* vals, int64_t* colptr,
                              unsigned long long* stats);

// C4 benchmark harness: CSR rows with nnz distinct random columns each (see sketch.cu)
void generate_sparse_rows_dev(slq_ctx* ctx, int64_t n, int64_t nnz, uint64_t seed, int64_t row_begin, int64_t m,
                              const double* scale, int64_t* rowptr, int32_t* colidx, double* vals);

// K2: Y_aug = S [A b] for the rows of A (S keyed by global row id).  Writes
// d x (n+1) column-major into Y (ldy = d).  exact => single split in the
// reference's accumulation order.
void sketch_apply_dev(slq_ctx* ctx, const slq_dense* A, int64_t d, int64_t zeta, uint64_t seed,
                      bool exact, double* Y);

// K2 in phases, for A arriving in row ranges (the host e2e path applies the
// sketch to each uploaded block while the next one is in flight): plan (chunk-
// CSR, slab width, Y workspace), gather of row ranges aligned to the chunk size
// (later ranges accumulate onto earlier ones, in ascending row order), finish.
struct DenseGather {
    ChunkCsr cc;
    int W = 4, rpt = 1;
    int64_t m = 0, d = 0, ld = 0, ncols_out = 0, ldw = 0, nslabs = 0, nsplit = 1;
    double val = 0.0;
    bool exact = false;
    double* Yw = nullptr;
    double* Y = nullptr;
    size_t smem = 0;
    int chunk_rows() const { return cc.plan.K; }
};
DenseGather dense_gather_plan(slq_ctx* ctx, int64_t m, int64_t n, int64_t ld, int64_t d, const uint32_t* compact,
                              const int64_t* colptr_dev, int64_t zeta, double val, bool exact, double* Y,
                              bool incremental);
void dense_gather_rows(slq_ctx* ctx, const DenseGather& G, const double* A, int64_t row_lo, int64_t row_hi);
void dense_gather_finish(slq_ctx* ctx, const DenseGather& G);

// K2 for a caller CSC sketch already in compact form on the device
// (colptr_dev int64, may be null for uniform zeta) against device A.
void sketch_apply_compact_dev(slq_ctx* ctx, const slq_dense* A, int64_t d, const uint32_t* compact,
                              const int64_t* colptr_dev, int64_t zeta, double val, bool exact,
                              double* Y);

}  // namespace slq
