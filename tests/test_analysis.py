"""CPU tests of the host-side companions (paper_2506_03070_b200/analysis.py):
embedding-dimension planner (embedding.hpp), scalar metrics (metrics.hpp) and
Matrix Market exchange (matrix_market.hpp), checked against the compiled
reference (oracle/_ref) -- files written by either side are read by the other."""
import os

import numpy as np
import pytest

import oracle

slq = pytest.importorskip("paper_2506_03070_b200")
A = slq.analysis

needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="compiled reference (oracle/_ref) absent")


@needs_ref
@pytest.mark.parametrize("m,n,d,eps,x", [(4_000_000, 1000, 4000, 1e-10, 3.0), (100_000, 100, 400, 1e-8, 0.5),
                                         (2**20, 500, 1000, 1e-6, 1e6), (1000, 999, 1000, 0.5, 1e-12),
                                         (10_000, 100, 10_000, 1e-10, 7.0)])
def test_embedding_matches_reference(m, n, d, eps, x):
    R = oracle.REF()
    ref = R.embedding(m, n, d, eps, x)
    r = A.estimate_rate(n, d)
    plan = A.select_embedding_dim(m, n, eps)
    got = [r.rate_per_iter, r.kappa, A.iterations_for(eps, n, d), A.lambert_w(x), A.balance_dimension_real(m, n, eps),
           plan.d, plan.predicted_iters, plan.predicted_kappa]
    np.testing.assert_allclose(got, ref, rtol=1e-14, atol=0)


def test_embedding_edge_cases():
    # test_sketch_stats / embedding tests: lambert_w(e) = 1, W(0) = 0, domain errors
    assert abs(A.lambert_w(np.e) - 1.0) <= 1e-13 and A.lambert_w(0.0) == 0.0
    w = A.lambert_w(1e12)
    assert abs(w * np.exp(w) - 1e12) <= 1e-12 * 1e12
    with pytest.raises(slq.NegativeArgument):
        A.lambert_w(-1.0)
    with pytest.raises(slq.InvalidDims):
        A.estimate_rate(10, 10)
    with pytest.raises(slq.InvalidDims):
        A.balance_dimension_real(10, 10, 1e-3)
    assert A.iterations_for(1e-10, 1, 100) == 5 and A.iterations_for(2.0, 5, 10) == 1
    p = A.select_embedding_dim(50, 40, 1e-12)
    assert p.d == 50  # clamped to m


@needs_ref
def test_metric_scalars_match_reference():
    R = oracle.REF()
    for x, ratio, eta, rh, rs in [(1.0, 0.25, 0.5, 2.0, 1.0), (0.3, 1.0, 0.0, 1.0, 1.0), (3.0, 0.1, 0.9, 5.0, 4.0)]:
        ref = R.metric_scalars(x, ratio, eta, rh, rs)
        got = (A.marchenko_pastur_pdf(x, ratio), A.cond_bound(eta), A.forward_error_from_residuals(rh, rs))
        np.testing.assert_allclose(got, ref, rtol=1e-15)
    with pytest.raises(slq.InvalidDistortion):
        A.cond_bound(1.0)
    with pytest.raises(slq.InvalidResidual):
        A.forward_error_from_residuals(0.5, 1.0)
    assert A.quantile([3.0, 1.0, 2.0], 0.5) == 2.0 and A.quantile([], 0.3) == 0.0


@needs_ref
def test_matrix_market_exchange(tmp_path):
    R = oracle.REF()
    rng = np.random.default_rng(0)
    # a sketch (CSC) written by the reference, read here -- and back
    rows, vals, cp, _ = oracle.C().generate_sparse_sign(64, 300, 8, 5)
    p1 = str(tmp_path / "S_ref.mtx")
    R.mm_write_csc(p1, 64, 300, rows, vals, cp)
    S = A.read_csc(p1)
    assert (S.rows, S.cols) == (64, 300)
    assert np.array_equal(S.row_indices, rows) and np.array_equal(S.values, vals) and np.array_equal(S.col_pointers, cp)
    p2 = str(tmp_path / "S_ours.mtx")
    A.write_csc(p2, S)
    assert open(p1).read() == open(p2).read()
    m, n, r2, v2, c2 = R.mm_read_csc(p2)
    assert np.array_equal(r2, rows) and np.array_equal(v2, vals) and np.array_equal(c2, cp)
    # dense, full precision round trip both ways
    D = rng.standard_normal((17, 5)) * 10.0 ** rng.integers(-300, 300, (17, 5))
    p3, p4 = str(tmp_path / "D_ref.mtx"), str(tmp_path / "D_ours.mtx")
    R.mm_write_dense(p3, D)
    A.write_dense(p4, D)
    assert open(p3).read() == open(p4).read()
    assert np.array_equal(A.read_dense(p3), D) and np.array_equal(R.mm_read_dense(p4), D)
    assert isinstance(A.load_matrix(p1), slq.CscMatrix) and A.load_matrix(p3).shape == (17, 5)
    # duplicates sum, unsorted input, 1-based indices, comments
    p5 = str(tmp_path / "dup.mtx")
    with open(p5, "w") as f:
        f.write("%%MatrixMarket matrix coordinate real general\n% comment\n3 2 4\n3 2 1.5\n1 1 2\n3 2 0.25\n2 1 -1\n")
    S5 = A.read_csc(p5)
    _, _, r5, v5, c5 = R.mm_read_csc(p5)
    assert np.array_equal(S5.row_indices, r5) and np.array_equal(S5.values, v5) and np.array_equal(S5.col_pointers, c5)
    assert list(S5.values) == [2.0, -1.0, 1.75]
    for bad in ("%%MatrixMarket matrix coordinate complex general\n1 1 0\n",
                "%%MatrixMarket matrix coordinate real symmetric\n1 1 0\n",
                "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n",
                "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n",
                "not a banner\n"):
        p6 = str(tmp_path / "bad.mtx")
        open(p6, "w").write(bad)
        with pytest.raises(slq.UnsupportedFormat):
            A.read_csc(p6)
        with pytest.raises(oracle.OracleError):
            R.mm_read_csc(p6)
