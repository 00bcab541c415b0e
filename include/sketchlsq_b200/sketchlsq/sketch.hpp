// sketchlsq/sketch.hpp (B200 drop-in) -- the sketches of sketch.hpp:16-306.
//
// Sparse sign (the paper's sketch, the hot path): generation and application
// run on the B200 through the C-ABI -- K1, the warp-cooperative rejection
// sampler keyed by global column id (bit-identical row indices, signs and
// RejectionStats for the same seed, sketch.hpp:75-194), and spmm on the
// device in the reference's accumulation order (csc_matrix.hpp).
//
// Gaussian and subsampled-trigonometric sketches and the Fisher-Yates sampler
// are outside the B200 path (comparison sketches / a statistical
// oracle); they are provided on the host with the reference's semantics and
// streams so code written against sketch.hpp keeps compiling and agreeing.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <string>
#include <vector>

#include "sketchlsq/csc_matrix.hpp"
#include "sketchlsq/dense_matrix.hpp"
#include "sketchlsq/device.hpp"
#include "sketchlsq/errors.hpp"
#include "sketchlsq/rng.hpp"
#include "sketchlsq/vector_ops.hpp"

namespace sketchlsq {

enum class SketchKind { SparseSign, Gaussian, Trig };

struct SketchParams {
    index_t d = 0;
    index_t zeta = 8;
    SketchKind kind = SketchKind::SparseSign;
    std::uint64_t seed = 0;

    // sketch.hpp:26-34
    void validate(index_t m, index_t n) const {
        if (!(n < d && d <= m))
            throw InvalidDims("SketchParams: need n < d <= m, got n=" + std::to_string(n) + " d=" + std::to_string(d) +
                              " m=" + std::to_string(m));
        if (kind == SketchKind::SparseSign && !(1 <= zeta && zeta <= d))
            throw InvalidSparsity("SketchParams: need 1 <= zeta <= d");
    }
};

struct SparseSignSketch {
    CscMatrix matrix;  // d x m, zeta entries +-1/sqrt(zeta) per column
    index_t zeta = 0;
    std::uint64_t seed = 0;
};

struct GaussianSketch {
    DenseMatrix matrix;
    std::uint64_t seed = 0;
};

struct TrigSketch {
    index_t d = 0;
    index_t m = 0;
    index_t padded_len = 0;
    std::vector<double> signs;
    std::vector<index_t> permutation;
    std::vector<index_t> selected_rows;
    std::uint64_t seed = 0;
};

struct RejectionStats {
    index_t columns_resampled = 0;
    index_t resample_rounds = 0;
};

namespace detail {

inline void add_stats(RejectionStats* out, const slq_rejection_stats& st) {
    if (!out) return;
    out->columns_resampled += st.columns_resampled;
    out->resample_rounds += st.resample_rounds;
}

// sketch.hpp:149-173: columns [col_begin, col_end) keyed by GLOBAL column id
// (index stream 2j, sign stream 2j+1), generated on the device
inline CscMatrix sparse_sign_block(index_t d, index_t zeta, std::uint64_t seed, index_t col_begin, index_t col_end,
                                   RejectionStats* stats = nullptr) {
    const index_t ncols = col_end - col_begin;
    CscMatrix S(d, ncols);
    S.values.resize(static_cast<std::size_t>(ncols * zeta));
    S.row_indices.resize(static_cast<std::size_t>(ncols * zeta));
    slq_rejection_stats st{0, 0};
    b200::check(slq_generate_sparse_sign(b200::ctx(), d, col_begin, ncols, zeta, seed, S.row_indices.data(),
                                         S.values.data(), S.col_pointers.data(), &st));
    add_stats(stats, st);
    return S;
}

inline index_t next_pow2(index_t m) {
    index_t p = 1;
    while (p < m) p <<= 1;
    return p;
}

// in-place orthonormal Walsh-Hadamard transform, len a power of two
inline void fwht(double* x, index_t len) {
    for (index_t span = 1; span < len; span *= 2)
        for (index_t blk = 0; blk < len; blk += 2 * span)
            for (index_t k = blk; k < blk + span; ++k) {
                const double lo = x[k], hi = x[k + span];
                x[k] = lo + hi;
                x[k + span] = lo - hi;
            }
    const double s = 1.0 / std::sqrt(static_cast<double>(len));
    for (index_t k = 0; k < len; ++k) x[k] *= s;
}

}  // namespace detail

// sketch.hpp:105-124: index matrix of m columns (column j at [j zeta, (j+1) zeta)),
// sorted distinct rows per column, on the device
inline std::vector<index_t> rejection_sample_columns(index_t d, index_t m, index_t zeta, std::uint64_t seed,
                                                     RejectionStats* stats = nullptr) {
    if (zeta < 1 || zeta > d) throw InvalidSparsity("rejection_sample_columns: need 1 <= zeta <= d");
    std::vector<index_t> C(static_cast<std::size_t>(m * zeta));
    slq_rejection_stats st{0, 0};
    b200::check(slq_rejection_sample_columns(b200::ctx(), d, m, zeta, seed, C.data(), &st));
    detail::add_stats(stats, st);
    return C;
}

// sketch.hpp:129-141: zeta distinct indices of [0, d) in selection order
// (swap Fisher-Yates), host -- the statistical oracle of the rejection sampler
inline std::vector<index_t> fisher_yates_sample(index_t d, index_t zeta, Rng& rng) {
    if (zeta < 1 || zeta > d) throw InvalidSparsity("fisher_yates_sample: need 1 <= zeta <= d");
    std::vector<index_t> pool(static_cast<std::size_t>(d));
    std::iota(pool.begin(), pool.end(), index_t{0});
    for (index_t i = 0; i < zeta; ++i) {
        const index_t pick = i + static_cast<index_t>(rng.uniform_below(static_cast<std::uint64_t>(d - i)));
        std::swap(pool[static_cast<std::size_t>(i)], pool[static_cast<std::size_t>(pick)]);
    }
    pool.resize(static_cast<std::size_t>(zeta));
    return pool;
}

// sketch.hpp:178-194
inline SparseSignSketch generate_sparse_sign(index_t d, index_t m, index_t zeta, std::uint64_t seed,
                                             RejectionStats* stats = nullptr) {
    if (zeta < 1 || zeta > d) throw InvalidSparsity("generate_sparse_sign: need 1 <= zeta <= d");
    return SparseSignSketch{detail::sparse_sign_block(d, zeta, seed, 0, m, stats), zeta, seed};
}
inline SparseSignSketch generate_sparse_sign(const SketchParams& p, index_t m, RejectionStats* stats = nullptr) {
    return generate_sparse_sign(p.d, m, p.zeta, p.seed, stats);
}

// sketch.hpp:199-216: N(0, 1/d) entries, column j from substream (seed, j)
inline GaussianSketch generate_gaussian(index_t d, index_t m, std::uint64_t seed,
                                        std::size_t max_entries = std::size_t{1} << 28) {
    if (static_cast<std::size_t>(d) * static_cast<std::size_t>(m) > max_entries)
        throw AllocationTooLarge("generate_gaussian: " + std::to_string(d) + "x" + std::to_string(m) +
                                 " exceeds the configured cap of " + std::to_string(max_entries) + " entries");
    GaussianSketch g{DenseMatrix(d, m), seed};
    const double inv_sqrt_d = 1.0 / std::sqrt(static_cast<double>(d));
    for (index_t j = 0; j < m; ++j) {
        Rng col_rng(seed, static_cast<std::uint64_t>(j));
        double* c = g.matrix.col(j);
        for (index_t i = 0; i < d; ++i) c[i] = col_rng.normal() * inv_sqrt_d;
    }
    return g;
}

// sketch.hpp:224-242: signs from substream 0, full permutation from 1, row selection from 2
inline TrigSketch generate_trig(index_t d, index_t m, std::uint64_t seed) {
    const index_t padded = detail::next_pow2(m);
    if (d > padded) throw InvalidDims("generate_trig: d exceeds padded length");
    TrigSketch t;
    t.d = d;
    t.m = m;
    t.padded_len = padded;
    t.seed = seed;
    Rng sgn(seed, 0);
    t.signs.resize(static_cast<std::size_t>(padded));
    for (double& s : t.signs) s = sgn.sign();
    Rng perm(seed, 1);
    t.permutation = fisher_yates_sample(m, m, perm);
    Rng sel(seed, 2);
    t.selected_rows = fisher_yates_sample(padded, d, sel);
    return t;
}

// sketch.hpp:267-291: permute, sign-flip, orthonormal WHT of the padded column,
// restrict to the selected rows, scale by sqrt(padded/d)
inline DenseMatrix apply_trig(const TrigSketch& t, const DenseMatrix& A) {
    if (A.rows() != t.m) throw DimensionMismatch("apply_trig: row count mismatch");
    DenseMatrix Y(t.d, A.cols());
    std::vector<double> work(static_cast<std::size_t>(t.padded_len));
    const double scale = std::sqrt(static_cast<double>(t.padded_len) / static_cast<double>(t.d));
    for (index_t j = 0; j < A.cols(); ++j) {
        const double* a = A.col(j);
        std::fill(work.begin(), work.end(), 0.0);
        for (index_t i = 0; i < t.m; ++i) work[static_cast<std::size_t>(i)] = a[t.permutation[static_cast<std::size_t>(i)]];
        for (index_t i = 0; i < t.padded_len; ++i) work[static_cast<std::size_t>(i)] *= t.signs[static_cast<std::size_t>(i)];
        detail::fwht(work.data(), t.padded_len);
        double* y = Y.col(j);
        for (index_t i = 0; i < t.d; ++i) y[i] = scale * work[static_cast<std::size_t>(t.selected_rows[static_cast<std::size_t>(i)])];
    }
    return Y;
}
inline Vector apply_trig(const TrigSketch& t, const Vector& x) {
    DenseMatrix X(t.m, 1, x);
    DenseMatrix Y = apply_trig(t, X);
    return Vector(Y.data().begin(), Y.data().end());
}

// sketch.hpp:297-306: the uniform apply / sketch_vector interface
inline DenseMatrix apply(const SparseSignSketch& s, const DenseMatrix& A) { return spmm(s.matrix, A); }
inline DenseMatrix apply(const SparseSignSketch& s, const CscMatrix& A) { return spmm(s.matrix, A); }
inline DenseMatrix apply(const GaussianSketch& s, const DenseMatrix& A) { return matmul(s.matrix, A); }
inline DenseMatrix apply(const GaussianSketch& s, const CscMatrix& A) { return matmul(s.matrix, densify(A)); }
inline DenseMatrix apply(const TrigSketch& s, const DenseMatrix& A) { return apply_trig(s, A); }
inline DenseMatrix apply(const TrigSketch& s, const CscMatrix& A) { return apply_trig(s, densify(A)); }

// S b on the device (csc_matrix.hpp:71-82 order, bit-identical)
inline Vector sketch_vector(const SparseSignSketch& s, const Vector& b) {
    if (static_cast<index_t>(b.size()) != s.matrix.cols) throw DimensionMismatch("matvec(csc): length mismatch");
    DenseMatrix Y = spmm(s.matrix, DenseMatrix(static_cast<index_t>(b.size()), 1, b));
    return Vector(Y.data().begin(), Y.data().end());
}
inline Vector sketch_vector(const GaussianSketch& s, const Vector& b) { return matvec(s.matrix, b); }
inline Vector sketch_vector(const TrigSketch& s, const Vector& b) { return apply_trig(s, b); }

}  // namespace sketchlsq
