// dropin_solve.cpp -- the reference's serial solve sequence (as in
// proj/tests/test_solvers.cpp:25-37), unchanged except for the include: the
// calls below resolve to the B200 drop-in (include/sketchlsq_b200/sketchlsq.hpp).
//
// Build (make -C examples):
//   g++ -std=c++20 -O2 -Iinclude examples/dropin_solve.cpp -Lpaper_2506_03070_b200 -lslq_b200
#include <cmath>
#include <cstdio>
#include <random>

#include "sketchlsq_b200/sketchlsq.hpp"

using namespace sketchlsq;

int main() {
    const index_t m = 20000, n = 50, d = 4 * n, zeta = 8;
    DenseMatrix A(m, n);
    std::mt19937_64 g(7);
    std::normal_distribution<double> N;
    for (double& v : A.data()) v = N(g);
    Vector b(static_cast<std::size_t>(m));
    for (double& v : b) v = N(g);

    SparseSignSketch S = generate_sparse_sign(d, m, zeta, /*seed=*/3);
    Preconditioner P = build_preconditioner(apply(S, A));
    Vector x0 = initial_guess(P, sketch_vector(S, b));
    SolveOptions opts;
    opts.eps = 0.0;
    opts.maxit = 40;
    auto [x, rep] = lsqr(A, P, b, x0, opts);

    // backward error ||A^T r|| / (||A||_F ||r||) on the host
    Vector r = b;
    for (index_t j = 0; j < n; ++j)
        for (index_t i = 0; i < m; ++i) r[i] -= A(i, j) * x[j];
    double atr = 0, rn = 0, af = 0;
    for (index_t j = 0; j < n; ++j) {
        double s = 0;
        for (index_t i = 0; i < m; ++i) s += A(i, j) * r[i];
        atr += s * s;
    }
    for (double v : r) rn += v * v;
    for (double v : A.data()) af += v * v;
    const double eta = std::sqrt(atr) / (std::sqrt(af) * std::sqrt(rn));
    std::printf("iterations=%ld termination=%s eta_F=%.3e\n", rep.iterations, to_string(rep.termination).c_str(), eta);
    try {
        generate_sparse_sign(3, 1, 4, 0);
    } catch (const InvalidSparsity& e) {
        std::printf("InvalidSparsity ok\n");
    }
    // the gradient family (gradient.hpp) on the same preconditioner
    SolveOptions gopts;
    gopts.eps = 1e-10;
    gopts.maxit = 400;
    auto [xh, rh] = gradient_descent_hbm(A, P, b, x0, hbm_params(std::sqrt(double(n) / double(d))), gopts);
    double dx = 0, xn = 0;
    for (index_t j = 0; j < n; ++j) {
        dx += (xh[j] - x[j]) * (xh[j] - x[j]);
        xn += x[j] * x[j];
    }
    std::printf("hbm iterations=%ld termination=%s |x_hbm - x_lsqr|/|x|=%.3e\n", rh.iterations,
                to_string(rh.termination).c_str(), std::sqrt(dx / xn));
    try {
        hbm_params(1.0);
    } catch (const InvalidDistortion& e) {
        std::printf("InvalidDistortion ok\n");
    }
    return (eta < 1e-10 && std::sqrt(dx / xn) < 1e-8) ? 0 : 1;
}
