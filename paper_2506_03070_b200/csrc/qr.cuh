// qr.cuh -- host entry points of the K3 kernels (QR, R^-1, triangular apply).
#pragma once

#include "common.cuh"

namespace slq {

// Householder QR of the first n columns of Yaug (d x ncols, column-major,
// ldy), in place; columns n..ncols-1 receive H^T (e.g. Q^T Sb).  Outputs
// (device): R (n x n, diag >= 0), qtb (n, sign-corrected Q^T of column n, may
// be null), Q (d x n, formed only if non-null), sign_out (n, may be null).
void qr_factor_dev(slq_ctx* ctx, double* Yaug, int64_t d, int64_t n, int64_t ncols, int64_t ldy,
                   double* R, double* qtb, double* Q, double* sign_out);

// M = R^-1 (column-major) and optionally Mt (row-major copy).
void tri_inverse_dev(slq_ctx* ctx, const double* R, int64_t n, double* M, double* Mt);

// Mt = M^T (n x n, column-major in and out).
void transpose_dev(slq_ctx* ctx, const double* M, int64_t n, double* Mt);

// y = M v for upper-triangular M given as its row-major copy Mt.
void trmv_upper_dev(slq_ctx* ctx, const double* Mt, int64_t n, const double* v, double* y);
// y = M^T v for upper-triangular M given column-major.
void trmv_upper_trans_dev(slq_ctx* ctx, const double* M, int64_t n, const double* v, double* y);

}  // namespace slq
