// sketchlsq/operators.hpp (B200 drop-in) -- the Op concept the solvers are
// templated on (operators.hpp:11-58).  SerialOperator<MatT> keeps the
// reference's surface (VecM = Vector on the host, matvec / rmatvec /
// rmatvec_and_norm / norm / axpy / scal, the uncounted instrumentation
// helpers, sync_snapshot) but its products run on the B200: the matrix is
// uploaded once when the operator is made, and every matvec / rmatvec is one
// HBM pass of the device operand (rmatvec_and_norm fuses A^T y and ||y||^2 in
// that pass).  This is the operator-level drop-in: the generic lsqr /
// lsqr_one_sync / gradient_descent_hbm templates drive it unchanged, with one
// host round trip per product; the DenseMatrix / CscMatrix overloads of those
// solvers run the fused device loop instead (lsqr.hpp).
#pragma once

#include <algorithm>
#include <cmath>
#include <memory>
#include <utility>

#include "sketchlsq/csc_matrix.hpp"
#include "sketchlsq/dense_matrix.hpp"
#include "sketchlsq/device.hpp"
#include "sketchlsq/vector_ops.hpp"

namespace sketchlsq {

namespace detail {

// Device copy of an operand (no right-hand side), owned by the operator.
struct DeviceOperand {
    slq_dense* dense = nullptr;
    slq_sparse* sparse = nullptr;
    DeviceOperand() = default;
    DeviceOperand(const DeviceOperand&) = delete;
    DeviceOperand& operator=(const DeviceOperand&) = delete;
    ~DeviceOperand() {
        if (dense) slq_dense_free(dense);
        if (sparse) slq_sparse_free(sparse);
    }
};

inline std::shared_ptr<DeviceOperand> upload_operand(const DenseMatrix& A) {
    auto d = std::make_shared<DeviceOperand>();
    b200::check(slq_dense_upload(b200::ctx(), A.data().data(), A.rows(), A.cols(), std::max<index_t>(A.rows(), 1),
                                 nullptr, 0, &d->dense));
    return d;
}
inline std::shared_ptr<DeviceOperand> upload_operand(const CscMatrix& A) {
    auto d = std::make_shared<DeviceOperand>();
    b200::check(slq_sparse_upload_csc(b200::ctx(), A.rows, A.cols, A.col_pointers.data(), A.row_indices.data(),
                                      A.values.data(), nullptr, 0, &d->sparse));
    return d;
}

inline void dev_matvec(const DeviceOperand& d, const Vector& x, Vector& y) {
    b200::check(d.dense ? slq_dense_matvec(b200::ctx(), d.dense, x.data(), y.data())
                        : slq_sparse_matvec(b200::ctx(), d.sparse, x.data(), y.data()));
}
inline void dev_rmatvec(const DeviceOperand& d, const Vector& y, Vector& z, double* ynorm2) {
    b200::check(d.dense ? slq_dense_rmatvec(b200::ctx(), d.dense, y.data(), z.data(), ynorm2)
                        : slq_sparse_rmatvec(b200::ctx(), d.sparse, y.data(), z.data(), ynorm2));
}

inline index_t mat_rows(const DenseMatrix& M) { return M.rows(); }
inline index_t mat_cols(const DenseMatrix& M) { return M.cols(); }
inline index_t mat_rows(const CscMatrix& M) { return M.rows; }
inline index_t mat_cols(const CscMatrix& M) { return M.cols; }

}  // namespace detail

template <class MatT>
struct SerialOperator {
    const MatT& A;
    std::shared_ptr<detail::DeviceOperand> dev = detail::upload_operand(A);

    using VecM = Vector;

    index_t rows() const { return detail::mat_rows(A); }
    index_t cols() const { return detail::mat_cols(A); }

    VecM matvec(const Vector& x) const {
        if (static_cast<index_t>(x.size()) != cols()) throw DimensionMismatch("matvec: length mismatch");
        VecM y(static_cast<std::size_t>(rows()));
        detail::dev_matvec(*dev, x, y);
        return y;
    }
    Vector rmatvec(const VecM& y) const {
        if (static_cast<index_t>(y.size()) != rows()) throw DimensionMismatch("rmatvec: length mismatch");
        Vector z(static_cast<std::size_t>(cols()));
        detail::dev_rmatvec(*dev, y, z, nullptr);
        return z;
    }
    // A^T y and ||y|| from one pass (the one-synchronization product)
    std::pair<Vector, double> rmatvec_and_norm(const VecM& y) const {
        if (static_cast<index_t>(y.size()) != rows()) throw DimensionMismatch("rmatvec: length mismatch");
        Vector z(static_cast<std::size_t>(cols()));
        double ss = 0.0;
        detail::dev_rmatvec(*dev, y, z, &ss);
        return {std::move(z), std::sqrt(ss)};
    }
    double norm(const VecM& y) const { return norm2(y); }
    void axpy(double a, const VecM& x, VecM& y) const { sketchlsq::axpy(a, x, y); }
    void scal(double a, VecM& y) const { sketchlsq::scal(a, y); }

    double error_norm(const Vector& xdiff) const { return norm2(matvec(xdiff)); }
    double residual_norm(const VecM& b, const Vector& x) const {
        VecM r = b;
        sketchlsq::axpy(-1.0, matvec(x), r);
        return norm2(r);
    }
    double norm_uncounted(const VecM& y) const { return norm2(y); }
    std::pair<long, long> sync_snapshot() const { return {0, 0}; }
};

template <class MatT>
SerialOperator<MatT> serial_operator(const MatT& A) {
    return SerialOperator<MatT>{A};
}

}  // namespace sketchlsq
