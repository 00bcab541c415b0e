"""CPU tests: pin the C restatement (oracle/) against the reference's golden
vectors (tests/golden/, made from the compiled reference) and, when the
compiled reference is present, against it directly on random cases."""
import numpy as np
import pytest

import oracle

C = oracle.C()


def test_rng_kats(golden):
    g = golden["rng"]
    # SURVEY Appendix A
    assert [hex(v) for v in C.rng_draws(0, None, 3)] == ["0xa706dd2f4d197e6f", "0xb382a305f4414f5e", "0x631a9154fbabf717"]
    assert np.array_equal(C.rng_draws(0, None, 8), g["seed0"])
    assert np.array_equal(C.rng_draws(42, 0, 8), g["s42_0"])
    assert np.array_equal(C.rng_draws(42, 1, 8), g["s42_1"])
    assert np.array_equal(C.uniform_below(7, 10, 16, 64), g["ub_7_10_16"])
    assert list(C.uniform_below(7, 10, 16, 6)) == [7, 9, 2, 2, 6, 13]
    assert np.array_equal(C.uniform_below(3, 4, 4000, 64), g["ub_3_4_4000"])


def test_sparse_sign_golden(golden):
    meta = golden["meta"]["sketch_cases"]
    arr = golden["sketch"]
    for i, c in enumerate(meta):
        rows, vals, colptr, st = C.generate_sparse_sign(c["d"], c["m"], c["zeta"], c["seed"], c["col_begin"])
        assert np.array_equal(rows, arr[f"rows_{i}"]), c
        assert np.array_equal(vals, arr[f"vals_{i}"]), c
        assert np.array_equal(colptr, arr[f"colptr_{i}"]), c
        assert st == (c["columns_resampled"], c["resample_rounds"]), c


def test_appendix_a_duplicate_path():
    rows, _, _, _ = C.generate_sparse_sign(400, 3, 8, 3)
    assert list(rows[16:24]) == [28, 53, 64, 92, 219, 254, 278, 301]


def test_rejection_stats_golden(golden):
    for c in golden["meta"]["stats_cases"]:
        if c["m"] > 100000:
            continue  # the 1e6-column cases are checked in test_sketch_stats (slow)
        _, _, _, st = C.generate_sparse_sign(c["d"], c["m"], c["zeta"], c["seed"])
        assert st == (c["columns_resampled"], c["resample_rounds"])


def test_invalid_sparsity():
    with pytest.raises(oracle.OracleError) as e:
        C.generate_sparse_sign(3, 1, 4, 0)
    assert e.value.kind == "InvalidSparsity"
    with pytest.raises(oracle.OracleError):
        C.generate_sparse_sign(3, 1, 0, 0)


def test_pipeline_golden(golden):
    p = golden["pipeline"]
    meta = golden["meta"]["pipeline"]
    A = C.gen_dense(meta["m"], meta["n"], meta["cond"], meta["seed_A"])
    assert np.array_equal(A, p["A"])
    b, xs = C.gen_rhs(A, meta["rho"], meta["seed_b"])
    assert np.array_equal(b, p["b"]) and np.array_equal(xs, p["x_star"])
    Y, Sb = C.sketch_apply(meta["d"], meta["zeta"], meta["seed_S"], A, b)
    assert np.array_equal(Y, p["Y"]) and np.array_equal(Sb, p["Sb"])
    Q, R = C.householder_qr(Y)
    assert np.array_equal(Q, p["Q"]) and np.array_equal(R, p["R"])
    M = C.tri_inverse(R)
    assert np.array_equal(M, p["M"])
    x0 = C.initial_guess(M, Q, Sb)
    assert np.array_equal(x0, p["x0"])
    x, rep = C.lsqr(A, M, b, x0, eps=0.0, maxit=meta["maxit"], x_star=xs, track_true=True)
    assert np.array_equal(x, p["x_std"])
    assert np.array_equal(rep.residual_estimate, p["est_std"])
    assert np.array_equal(rep.iterates_error, p["err_std"])
    assert np.array_equal(rep.residual_true, p["true_std"])
    x1, rep1 = C.lsqr(A, M, b, x0, eps=0.0, maxit=meta["maxit"], one_sync=True)
    assert np.array_equal(x1, p["x_one"]) and np.array_equal(rep1.residual_estimate, p["est_one"])
    xt, rept = C.lsqr(A, M, b, np.zeros(meta["n"]), eps=1e-10, maxit=100)
    assert rept.iterations == meta["tol_run"]["iterations"]
    assert rept.termination == meta["tol_run"]["termination"]
    assert np.array_equal(xt, p["x_tol"])


def test_partition_rows_golden(golden):
    parts = golden["meta"]["partition_rows"]
    for p in (1, 2, 4, 8):
        assert C.partition_rows(333, p).tolist() == parts[str(p)]
    assert C.partition_rows(4_000_000, 8).tolist() == parts["4000000/8"]
    assert C.partition_rows(1 << 20, 3).tolist() == parts["1048576/3"]
    with pytest.raises(oracle.OracleError):
        C.partition_rows(3, 4)


def test_lsqr_edge_cases():
    # lsqr on identity converges in one iteration (test_solvers.cpp:41-53)
    n = 5
    b = np.array([1.0, -2.0, 0.5, 3.0, 0.25])
    x, rep = C.lsqr(np.eye(n), np.eye(n), b, np.zeros(n))
    assert rep.iterations == 1 and rep.termination != "maxiter"
    assert np.allclose(x, b, rtol=1e-12)
    # breakdown (test_solvers.cpp:132-147)
    x, rep = C.lsqr(np.eye(4), np.eye(4), np.array([2.0, 0, 0, 0]), np.zeros(4), eps=0.0, maxit=5)
    assert rep.termination == "breakdown" and rep.iterations == 1
    # 3x2 hand instance (test_solvers.cpp:55-70)
    A = np.array([[1.0, 0], [0, 1], [1, 1]])
    x, rep = C.lsqr(A, np.eye(2), np.array([1.0, 2, 0]), np.zeros(2), eps=1e-14, maxit=2)
    assert abs(x[0]) <= 1e-10 and abs(x[1] - 1) <= 1e-10
    # beta1 == 0 -> tolerance at 0 iterations
    x, rep = C.lsqr(np.eye(3), np.eye(3), np.zeros(3), np.zeros(3))
    assert rep.iterations == 0 and rep.termination == "tolerance"


@pytest.mark.skipif(not oracle.ref_available(), reason="compiled reference absent")
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_restatement_matches_reference_random(seed):
    R = oracle.REF()
    rng = np.random.default_rng(seed)
    d = int(rng.integers(8, 300))
    zeta = int(rng.integers(1, min(d, 20) + 1))
    m = int(rng.integers(1, 500))
    s = int(rng.integers(0, 2**63))
    a = C.generate_sparse_sign(d, m, zeta, s)
    r = R.generate_sparse_sign(d, m, zeta, s)
    for u, v in zip(a[:3], r[:3]):
        assert np.array_equal(u, v)
    assert a[3] == r[3]
    m, n = 300, 10
    A = rng.standard_normal((m, n))
    A[rng.random((m, n)) < 0.1] = 0.0
    b = rng.standard_normal(m)
    Y1, S1 = C.sketch_apply(40, 4, s, A, b)
    Y2, S2 = R.sketch_apply(40, 4, s, A, b)
    assert np.array_equal(Y1, Y2) and np.array_equal(S1, S2)


def test_gradient_golden(golden):
    """gradient.hpp:27-126 (hbm_params / gd_params / gradient_descent_hbm)
    restated in C, bit-identical to the compiled reference's fixtures."""
    p, g = golden["pipeline"], golden["gradient"]
    meta = golden["meta"]["gradient"]
    assert C.gradient_params(meta["eta"], True) == tuple(meta["hbm"])
    assert C.gradient_params(meta["eta"], False) == tuple(meta["gd"])
    a, b = meta["hbm"]
    x, rep = C.gd_hbm(p["A"], p["M"], p["b"], p["x0"], a, b, eps=0.0, maxit=meta["maxit"], x_star=p["x_star"],
                      track_true=True)
    assert np.array_equal(x, g["x_hbm"]) and rep.iterations == meta["maxit"]
    assert np.array_equal(rep.residual_estimate, g["est_hbm"])
    assert np.array_equal(rep.iterates_error, g["err_hbm"])
    assert np.array_equal(rep.residual_true, g["true_hbm"])
    a, b = meta["gd"]
    x, rep = C.gd_hbm(p["A"], p["M"], p["b"], p["x0"], a, b, eps=0.0, maxit=meta["maxit"])
    assert np.array_equal(x, g["x_gd"]) and np.array_equal(rep.residual_estimate, g["est_gd"])
    a, b = meta["hbm"]
    x, rep = C.gd_hbm(p["A"], p["M"], p["b"], p["x0"], a, b, eps=meta["tol_run"]["eps"], maxit=200)
    assert np.array_equal(x, g["x_ht"])
    assert rep.iterations == meta["tol_run"]["iterations"] and rep.termination == meta["tol_run"]["termination"]


def test_gradient_edge_cases():
    # hbm_params / gd_step_size domain (test_solvers.cpp:187-206)
    assert C.gradient_params(0.5, True) == (0.5625, 0.25)
    assert C.gradient_params(0.0, False) == (1.0, 0.0)
    assert abs(C.gradient_params(0.5, False)[0] - 0.45) <= 1e-15
    for eta, hbm in ((1.0, True), (1.5, False), (-0.1, True)):
        with pytest.raises(oracle.OracleError) as e:
            C.gradient_params(eta, hbm)
        assert e.value.kind == "InvalidDistortion"
    # perfectly preconditioned gradient step solves in one iteration (test_solvers.cpp:208-222)
    rng = np.random.default_rng(19)
    Qa, _ = np.linalg.qr(rng.standard_normal((50, 8)))
    xs = rng.standard_normal(8)
    x, rep = C.gd_hbm(Qa, np.eye(8), Qa @ xs, np.zeros(8), 1.0, 0.0, maxit=3, x_star=xs)
    assert rep.iterates_error[1] <= 1e-12 * rep.iterates_error[0]
    # a step size far too large diverges (Divergence, gradient.hpp:82-85)
    A = rng.standard_normal((40, 5))
    with pytest.raises(oracle.OracleError) as e:
        C.gd_hbm(A, np.eye(5), rng.standard_normal(40), np.zeros(5), 10.0, 0.0, eps=0.0, maxit=200)
    assert e.value.kind == "Divergence"
