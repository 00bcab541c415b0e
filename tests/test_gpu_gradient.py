"""GPU parity of the gradient family (gradient.hpp:27-126)
against the CPU oracle (bit-identical to the compiled reference, see
tests/test_oracle.py::test_gradient_golden).

Bars: iterates within 1e-10 relative, ||M^T A^T r|| histories rtol 1e-9,
same termination and iteration count under the reference stopping rule,
Divergence raised where the reference raises it."""
import numpy as np
import pytest
import scipy.sparse as sp

import oracle

pytestmark = pytest.mark.gpu

slq = pytest.importorskip("paper_2506_03070_b200")
C = oracle.C()


def test_params_match_reference(golden):
    meta = golden["meta"]["gradient"]
    h = slq.hbm_params(meta["eta"])
    g = slq.gd_params(meta["eta"])
    assert (h.alpha, h.beta) == tuple(meta["hbm"]) and (g.alpha, g.beta) == tuple(meta["gd"])
    assert slq.gd_step_size(0.0) == 1.0 and abs(slq.gd_step_size(0.5) - 0.45) <= 1e-15
    for bad in (1.0, 1.5, -0.1):
        with pytest.raises(slq.InvalidDistortion):
            slq.hbm_params(bad)
        with pytest.raises(slq.InvalidDistortion):
            slq.gd_params(bad)


@pytest.mark.parametrize("which", ["hbm", "gd"])
def test_gradient_dense_vs_golden(golden, which):
    p, g = golden["pipeline"], golden["gradient"]
    meta = golden["meta"]["gradient"]
    params = slq.hbm_params(meta["eta"]) if which == "hbm" else slq.gd_params(meta["eta"])
    opts = slq.SolveOptions(eps=0.0, maxit=meta["maxit"], x_star=p["x_star"], track_true_residual=True)
    x, rep = slq.gradient_descent_hbm(p["A"], p["M"], p["b"], p["x0"], params, opts)
    xo, repo = C.gd_hbm(p["A"], p["M"], p["b"], p["x0"], params.alpha, params.beta, eps=0.0, maxit=meta["maxit"],
                        x_star=p["x_star"], track_true=True)
    assert np.array_equal(xo, g[f"x_{which}"])
    assert rep.iterations == meta["maxit"] and rep.termination == slq.Termination.MaxIter
    assert np.linalg.norm(x - xo) <= 1e-10 * np.linalg.norm(xo)
    assert np.allclose(rep.residual_estimate, repo.residual_estimate, rtol=1e-9)
    assert np.allclose(rep.iterates_error, repo.iterates_error, rtol=1e-6, atol=1e-13)
    assert np.allclose(rep.residual_true, repo.residual_true, rtol=1e-9)


def test_gradient_tolerance_rule(golden):
    p, g = golden["pipeline"], golden["gradient"]
    meta = golden["meta"]["gradient"]
    params = slq.hbm_params(meta["eta"])
    x, rep = slq.gradient_descent_hbm(p["A"], p["M"], p["b"], p["x0"], params,
                                      slq.SolveOptions(eps=meta["tol_run"]["eps"], maxit=200))
    assert rep.iterations == meta["tol_run"]["iterations"]
    assert rep.termination.name.lower() == meta["tol_run"]["termination"]
    assert np.linalg.norm(x - g["x_ht"]) <= 1e-9 * np.linalg.norm(g["x_ht"])
    # plain gradient descent needs more iterations than heavy ball (test_solvers.cpp:253-272)
    _, rg = slq.gradient_descent_hbm(p["A"], p["M"], p["b"], p["x0"], slq.gd_params(meta["eta"]),
                                     slq.SolveOptions(eps=meta["tol_run"]["eps"], maxit=400))
    assert rg.iterations > rep.iterations


def test_gradient_device_matrix_batches():
    """Long device-resident run (batched iterations, device stop flag)."""
    rng = np.random.default_rng(4)
    m, n, d = 20000, 60, 240
    A = rng.standard_normal((m, n)) @ np.diag(np.logspace(0, -3, n))
    b = rng.standard_normal(m)
    Y, Sb = C.sketch_apply(d, 8, 5, A, b)
    M, Q = C.build_preconditioner(Y)
    x0 = C.initial_guess(M, Q, Sb)
    eta = float(np.sqrt(n / d))
    prm = slq.hbm_params(eta)
    dm = slq.DeviceMatrix.from_numpy(A, b)
    for eps, maxit in ((0.0, 37), (1e-9, 300)):
        x, rep = slq.gradient_descent_hbm(dm, M, None, x0, prm, slq.SolveOptions(eps=eps, maxit=maxit))
        xo, repo = C.gd_hbm(A, M, b, x0, prm.alpha, prm.beta, eps=eps, maxit=maxit)
        assert rep.iterations == repo.iterations and rep.termination.name.lower() == repo.termination
        assert np.linalg.norm(x - xo) <= 1e-10 * np.linalg.norm(xo)
        assert np.allclose(rep.residual_estimate, repo.residual_estimate, rtol=1e-8)


def test_gradient_sparse_vs_oracle():
    rng = np.random.default_rng(7)
    m, n, d = 5000, 40, 200
    A = sp.random(m, n, density=0.05, format="csc", random_state=3, data_rvs=rng.standard_normal)
    A.sort_indices()
    rows, vals, cp = A.indices.astype(np.int64), A.data.copy(), A.indptr.astype(np.int64)
    b = rng.standard_normal(m)
    Y, Sb = C.sketch_apply_csc(d, 8, 9, m, n, rows, vals, cp, b)
    M, Q = C.build_preconditioner(Y)
    x0 = C.initial_guess(M, Q, Sb)
    prm = slq.hbm_params(float(np.sqrt(n / d)))
    Acsc = slq.CscMatrix(m, n, vals, rows, cp)
    x, rep = slq.gradient_descent_hbm(Acsc, M, b, x0, prm, slq.SolveOptions(eps=0.0, maxit=20))
    xo, repo = C.gd_hbm_csc(m, n, rows, vals, cp, M, b, x0, prm.alpha, prm.beta, eps=0.0, maxit=20)
    assert rep.iterations == 20
    assert np.linalg.norm(x - xo) <= 1e-10 * np.linalg.norm(xo)
    assert np.allclose(rep.residual_estimate, repo.residual_estimate, rtol=1e-9)


def test_gradient_one_step_and_divergence():
    # perfectly preconditioned gradient step solves in one iteration (test_solvers.cpp:208-222)
    rng = np.random.default_rng(19)
    Qa, _ = np.linalg.qr(rng.standard_normal((50, 8)))
    xs = rng.standard_normal(8)
    x, rep = slq.gradient_descent_hbm(Qa, np.eye(8), Qa @ xs, np.zeros(8), slq.GradientParams(1.0, 0.0, 0.0),
                                      slq.SolveOptions(maxit=3, x_star=xs))
    assert rep.iterates_error[1] <= 1e-12 * rep.iterates_error[0]
    # too large a step grows ||M^T A^T r|| by 1e6 -> Divergence (gradient.hpp:82-85)
    A = rng.standard_normal((40, 5))
    bb = rng.standard_normal(40)
    with pytest.raises(oracle.OracleError):
        C.gd_hbm(A, np.eye(5), bb, np.zeros(5), 10.0, 0.0, eps=0.0, maxit=200)
    with pytest.raises(slq.Divergence):
        slq.gradient_descent_hbm(A, np.eye(5), bb, np.zeros(5), slq.GradientParams(10.0, 0.0, 0.0),
                                 slq.SolveOptions(eps=0.0, maxit=200))
