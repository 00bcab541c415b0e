// sketchlsq/qr.hpp (B200 drop-in) -- householder_qr (qr.hpp:21-89) on the
// B200: thread-block-cluster panel factorization + FP64 tensor-core (DMMA)
// trailing updates, the reference's conventions (rank tolerance
// 1e-12 max|Y|, sign choice, diag(R) >= 0), RankDeficient on rank loss.
#pragma once

#include <algorithm>

#include "sketchlsq/dense_matrix.hpp"
#include "sketchlsq/device.hpp"
#include "sketchlsq/errors.hpp"

namespace sketchlsq {

struct QrResult {
    DenseMatrix Q;  // d x n, orthonormal columns
    DenseMatrix R;  // n x n, upper triangular, diag(R) >= 0
};

inline QrResult householder_qr(const DenseMatrix& Y) {
    const index_t d = Y.rows(), n = Y.cols();
    if (d < n) throw DimensionMismatch("householder_qr: need rows >= cols");
    QrResult f{DenseMatrix(d, n), DenseMatrix(n, n)};
    if (n == 0) return f;
    b200::check(slq_householder_qr(b200::ctx(), Y.data().data(), d, n, std::max<index_t>(d, 1), f.Q.data().data(),
                                   f.R.data().data()));
    return f;
}

}  // namespace sketchlsq
