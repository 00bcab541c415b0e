// spmm_general.cuh -- spmm for a CSC left factor with arbitrary values (see spmm_general.cu).
#pragma once

#include "common.cuh"

namespace slq {

struct SpmmCheck {
    bool mixed_magnitudes = false;  // not a sparse-sign matrix (|values| not all equal)
    bool row_out_of_range = false;
};
// device-side validation of a CSC's entries (one sync)
SpmmCheck csc_check_dev(slq_ctx* ctx, const int64_t* rows, const double* vals, int64_t nnz, int64_t d);

// Y (d x n, column-major) = S A with S (d x m, CSC: rows / vals / colptr on the
// device) and either A_rows (device row-major, leading dimension ld; zero
// entries skipped) or a device CSC A (acp / arows / avals), reference order.
void spmm_general_dev(slq_ctx* ctx, int64_t d, int64_t m, int64_t nnz, const int64_t* rows, const double* vals,
                      const int64_t* colptr, int64_t n, const double* A_rows, int64_t ld, const int64_t* acp,
                      const int64_t* arows, const double* avals, double* Y);

}  // namespace slq
