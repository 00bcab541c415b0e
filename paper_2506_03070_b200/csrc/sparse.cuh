// sparse.cuh -- host entry points of the sparse-A (CSR) path.
#pragma once

#include <memory>

#include "common.cuh"
#include "lsqr.cuh"

namespace slq {

// allocate the CSR arrays of A (m, n, nnz set by the caller) with bulk-copy slack
void sparse_alloc(slq_ctx* ctx, slq_sparse* A, bool with_b);
void sparse_free(slq_sparse* A);
// fill A's CSR from a host CSC (the reference CscMatrix layout), rows sorted
void sparse_from_csc(slq_ctx* ctx, slq_sparse* A, const int64_t* colptr, const int64_t* rows, const double* vals);
// K2s: Y_aug = S [A b] (d x (n+1), column-major), bit-identical to spmm(csc, csc)
void sketch_apply_sparse_dev(slq_ctx* ctx, const slq_sparse* A, int64_t d, int64_t zeta, uint64_t seed, double* Y);
// K2s for a caller-given sketch already in compact form (colptr_dev null = uniform zeta)
void sketch_apply_sparse_compact_dev(slq_ctx* ctx, const slq_sparse* A, int64_t d, const uint32_t* compact,
                                     const int64_t* colptr_dev, int64_t zeta_max, double val, double* Y);
// Build (or rebuild) the row-blocked CSC copy the two-pass operator reads
// (kept with the matrix until its CSR is rewritten).  async: on ctx->aux,
// overlapping what the main stream does next; PassOp::ready joins it.
void prepare_two_pass(slq_ctx* ctx, slq_sparse* A, bool async = false);
// K4s operator for LSQR.  two_pass: u_hat over the CSR, then z = A^T u_hat over
// a row-blocked CSC copy built here (solves: many passes amortise the build);
// false: the single fused pass (one-off products)
std::unique_ptr<PassOp> make_sparse_op(slq_ctx* ctx, const slq_sparse* A, bool two_pass = false);

}  // namespace slq
