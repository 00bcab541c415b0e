"""GPU parity of the sparse-A path (BASELINE config C4)
against the CPU oracle's CSC restatement (itself bit-identical to the
reference's spmm(csc, csc) / SerialOperator<CscMatrix>, tests/test_oracle.py).

Bars: S A and S b bit-exact (reference accumulation order); LSQR iterates
within 1e-10 at moderate conditioning, residual histories 1e-9; the
pipeline's backward error no worse than 2x the reference's at fixed T."""
import numpy as np
import pytest
import scipy.sparse as sp

import oracle

pytestmark = pytest.mark.gpu

slq = pytest.importorskip("paper_2506_03070_b200")
C = oracle.C()


def rand_csc(m, n, density, seed, long_rows=0, empty_rows=0):
    rng = np.random.default_rng(seed)
    A = sp.random(m, n, density=density, format="lil", random_state=seed, data_rvs=rng.standard_normal)
    for r in range(long_rows):  # rows longer than one warp pass (64 nnz)
        A[r, :] = rng.standard_normal(n) * (rng.random(n) < 0.9)
    for r in range(empty_rows):
        A[m - 1 - r, :] = 0.0
    A = A.tocsc()
    A.sort_indices()
    A.eliminate_zeros()
    return slq.CscMatrix(m, n, A.data.astype(np.float64), A.indices.astype(np.int64), A.indptr.astype(np.int64)), A


@pytest.mark.parametrize("m,n,d,zeta,density,long_rows", [(3000, 40, 200, 8, 0.05, 0), (5000, 100, 400, 4, 0.02, 3),
                                                          (2000, 70, 300, 16, 0.3, 5), (1500, 8, 64, 1, 0.1, 0)])
def test_sparse_apply_bit_exact(m, n, d, zeta, density, long_rows):
    Acsc, A = rand_csc(m, n, density, m + n, long_rows=long_rows, empty_rows=2)
    b = np.random.default_rng(1).standard_normal(m)
    S = slq.generate_sparse_sign(d, m, zeta, 77)
    Y = slq.apply(S, Acsc)
    Yo, Sbo = C.sketch_apply_csc(d, zeta, 77, m, n, Acsc.row_indices, Acsc.values, Acsc.col_pointers, b)
    assert np.array_equal(Y, Yo)
    dm = slq.SparseDeviceMatrix.from_csc(Acsc, b)
    Yd, Sbd = dm.sketch(d, zeta, 77)
    assert np.array_equal(Yd, Yo) and np.array_equal(Sbd, Sbo)


def test_sparse_apply_matches_dense_apply():
    Acsc, A = rand_csc(4000, 30, 0.1, 5)
    S = slq.generate_sparse_sign(160, 4000, 8, 3)
    assert np.array_equal(slq.apply(S, Acsc), slq.apply(S, A.toarray()))


def test_sparse_lsqr_vs_oracle():
    m, n, d, zeta = 6000, 50, 300, 8
    Acsc, A = rand_csc(m, n, 0.05, 11)
    Ad = A.toarray()
    b = np.random.default_rng(2).standard_normal(m)
    Y, Sb = C.sketch_apply_csc(d, zeta, 5, m, n, Acsc.row_indices, Acsc.values, Acsc.col_pointers, b)
    M, Q = C.build_preconditioner(Y)
    x0 = C.initial_guess(M, Q, Sb)
    xs = np.linalg.lstsq(Ad, b, rcond=None)[0]
    for one_sync in (False, True):
        fn = slq.lsqr_one_sync if one_sync else slq.lsqr
        x, rep = fn(Acsc, M, b, x0, slq.SolveOptions(eps=0.0, maxit=12, x_star=xs, track_true_residual=True))
        xo, repo = C.lsqr_csc(m, n, Acsc.row_indices, Acsc.values, Acsc.col_pointers, M, b, x0, eps=0.0, maxit=12,
                              one_sync=one_sync, x_star=xs, track_true=True)
        assert rep.iterations == 12
        assert np.linalg.norm(x - xo) <= 1e-10 * np.linalg.norm(xo)
        assert np.allclose(rep.residual_estimate, repo.residual_estimate, rtol=1e-9)
        assert np.allclose(rep.residual_true, repo.residual_true, rtol=1e-9)
        assert np.allclose(rep.iterates_error, repo.iterates_error, rtol=1e-6, atol=1e-12)


def test_sparse_solve_pipeline():
    m, n, d, zeta = 20000, 60, 240, 8
    Acsc, A = rand_csc(m, n, 0.03, 21)
    Ad = A.toarray()
    b = np.random.default_rng(3).standard_normal(m)
    x, rep, times = slq.solve(Acsc, d, zeta, 9, slq.SolveOptions(eps=0.0, maxit=25), b=b)
    Y, Sb = C.sketch_apply_csc(d, zeta, 9, m, n, Acsc.row_indices, Acsc.values, Acsc.col_pointers, b)
    M, Q = C.build_preconditioner(Y)
    x0 = C.initial_guess(M, Q, Sb)
    xo, repo = C.lsqr_csc(m, n, Acsc.row_indices, Acsc.values, Acsc.col_pointers, M, b, x0, eps=0.0, maxit=25,
                          one_sync=True)

    def eta(v):
        r = b - Ad @ v
        return np.linalg.norm(Ad.T @ r) / (np.linalg.norm(Ad, 2) * np.linalg.norm(r))

    assert rep.iterations == 25
    assert eta(x) <= max(2 * eta(xo), 1e-14)
    assert np.linalg.norm(x - xo) <= 1e-8 * np.linalg.norm(xo)
    # fixed-order reductions throughout: a repeat solve is bit-identical
    x2, rep2, _ = slq.solve(Acsc, d, zeta, 9, slq.SolveOptions(eps=0.0, maxit=25), b=b)
    assert np.array_equal(x, x2) and np.array_equal(rep.residual_estimate, rep2.residual_estimate)


def test_sparse_lsqr_long_rows():
    """Rows longer than 64 and 255 entries take the pass's tail path."""
    m, n, d, zeta = 3000, 600, 1200, 8
    Acsc, A = rand_csc(m, n, 0.01, 5, long_rows=4)
    Ad = A.toarray()
    Ad[10, :500] = np.random.default_rng(9).standard_normal(500)  # 500-entry row
    Ad[11, ::7] = 1.0
    As = sp.csc_matrix(Ad)
    As.sort_indices()
    Acsc = slq.CscMatrix(m, n, As.data.copy(), As.indices.astype(np.int64), As.indptr.astype(np.int64))
    b = np.random.default_rng(2).standard_normal(m)
    Y, Sb = C.sketch_apply_csc(d, zeta, 5, m, n, Acsc.row_indices, Acsc.values, Acsc.col_pointers, b)
    M, Q = C.build_preconditioner(Y)
    x0 = C.initial_guess(M, Q, Sb)
    x, rep = slq.lsqr_one_sync(Acsc, M, b, x0, slq.SolveOptions(eps=0.0, maxit=8))
    xo, repo = C.lsqr_csc(m, n, Acsc.row_indices, Acsc.values, Acsc.col_pointers, M, b, x0, eps=0.0, maxit=8,
                          one_sync=True)
    assert np.linalg.norm(x - xo) <= 1e-10 * np.linalg.norm(xo)
    assert np.allclose(rep.residual_estimate, repo.residual_estimate, rtol=1e-9)


@pytest.mark.parametrize("m,n,dens", [(50, 13, 0.08), (400, 13, 0.08), (7, 3, 0.5), (1000, 40, 0.02), (3000, 200, 0.3)])
def test_sparse_operator_products(m, n, dens):
    """slq_sparse_matvec / slq_sparse_rmatvec (the Op surface of operators.hpp
    over a CSC operand): A x and A^T y (+ ||y||^2) against numpy, including
    empty rows and columns."""
    import ctypes as ct

    from paper_2506_03070_b200 import _capi as CA

    rng = np.random.default_rng(m * 31 + n)
    D = np.where(rng.random((m, n)) < dens, rng.standard_normal((m, n)), 0.0)
    cols = [np.nonzero(D[:, j])[0] for j in range(n)]
    rows = np.concatenate(cols).astype(np.int64)
    vals = np.concatenate([D[c, j] for j, c in enumerate(cols)])
    cp = np.concatenate([[0], np.cumsum([len(c) for c in cols])]).astype(np.int64)
    A = slq.SparseDeviceMatrix.from_csc(slq.CscMatrix(m, n, vals, rows, cp))
    x = rng.standard_normal(n)
    y = rng.standard_normal(m)
    ax = np.zeros(m)
    aty = np.zeros(n)
    ss = ct.c_double(0.0)
    assert CA.lib.slq_sparse_matvec(A.ctx.handle, A.handle, x.ctypes.data_as(CA.dp), ax.ctypes.data_as(CA.dp)) == 0
    assert CA.lib.slq_sparse_rmatvec(A.ctx.handle, A.handle, y.ctypes.data_as(CA.dp), aty.ctypes.data_as(CA.dp),
                                     ct.byref(ss)) == 0
    assert np.allclose(ax, D @ x, rtol=1e-13, atol=1e-13)
    assert np.allclose(aty, D.T @ y, rtol=1e-12, atol=1e-13), np.abs(aty - D.T @ y).max()
    assert abs(ss.value - y @ y) <= 1e-12 * (y @ y)
    Dd = np.asfortranarray(D)
    dm = slq.DeviceMatrix.from_numpy(Dd)
    assert CA.lib.slq_dense_matvec(dm.ctx.handle, dm.handle, x.ctypes.data_as(CA.dp), ax.ctypes.data_as(CA.dp)) == 0
    assert CA.lib.slq_dense_rmatvec(dm.ctx.handle, dm.handle, y.ctypes.data_as(CA.dp), aty.ctypes.data_as(CA.dp),
                                    ct.byref(ss)) == 0
    assert np.allclose(ax, D @ x, rtol=1e-13, atol=1e-13)
    assert np.allclose(aty, D.T @ y, rtol=1e-12, atol=1e-13)


def test_sparse_two_pass_multiblock(monkeypatch):
    """The two-pass LSQR operator (u_hat over the CSR, z = A^T u_hat over the
    row-blocked CSC copy, blocks of 16384 rows) across several blocks with a
    partial last block, rows longer than 64 entries and empty rows: against the
    oracle's CSC LSQR and the single fused pass (SLQ_SPARSE_ONEPASS=1)."""
    m, n, d, zeta = 50_001, 300, 1200, 8
    # 40 long rows in the first 128-row chunk: > 8192 entries, so that chunk takes the
    # u_hat pass's direct (unstaged) path
    Acsc, A = rand_csc(m, n, 0.02, 31, long_rows=40, empty_rows=5)
    assert Acsc.col_pointers[-1] > 0 and (A.tocsr()[:128].nnz > 8192)
    b = np.random.default_rng(4).standard_normal(m)
    Y, Sb = C.sketch_apply_csc(d, zeta, 5, m, n, Acsc.row_indices, Acsc.values, Acsc.col_pointers, b)
    M, Q = C.build_preconditioner(Y)
    x0 = C.initial_guess(M, Q, Sb)
    xo, repo = C.lsqr_csc(m, n, Acsc.row_indices, Acsc.values, Acsc.col_pointers, M, b, x0, eps=0.0, maxit=10,
                          one_sync=True)
    x2, rep2 = slq.lsqr_one_sync(Acsc, M, b, x0, slq.SolveOptions(eps=0.0, maxit=10))
    monkeypatch.setenv("SLQ_SPARSE_ONEPASS", "1")
    x1, rep1 = slq.lsqr_one_sync(Acsc, M, b, x0, slq.SolveOptions(eps=0.0, maxit=10))
    for x, rep in ((x2, rep2), (x1, rep1)):
        assert np.linalg.norm(x - xo) <= 1e-10 * np.linalg.norm(xo)
        assert np.allclose(rep.residual_estimate, repo.residual_estimate, rtol=1e-9)
    # the gradient family runs its passes without keeping u_hat (scratch vector path)
    monkeypatch.delenv("SLQ_SPARSE_ONEPASS")
    P = slq.hbm_params(float(np.sqrt(n / d)))
    xg, _ = slq.gradient_descent_hbm(Acsc, M, b, x0, P, slq.SolveOptions(eps=0.0, maxit=6))
    xgo, _ = C.gd_hbm_csc(m, n, Acsc.row_indices, Acsc.values, Acsc.col_pointers, M, b, x0, P.alpha, P.beta,
                          eps=0.0, maxit=6)
    assert np.linalg.norm(xg - xgo) <= 1e-10 * np.linalg.norm(xgo)


@pytest.mark.parametrize("m,n,dens", [(100, 12, 0.3), (37, 1, 0.6), (300, 24, 0.02)])
def test_sparse_two_pass_small_shapes(m, n, dens):
    """The two-pass operator at shapes below one 128-row chunk / one 16384-row
    block, with empty rows (and n = 1): LSQR against the oracle's CSC LSQR.
    For n <= maxit the Krylov space is exhausted: whether beta / alpha land on
    an exact zero (Breakdown) or on a rounding-level value depends on the
    summation order, so only x is compared there."""
    Acsc, A = rand_csc(m, n, dens, m + 7 * n, empty_rows=3)
    b = np.random.default_rng(m).standard_normal(m)
    M = np.triu(np.random.default_rng(n).standard_normal((n, n))) + 3.0 * np.eye(n)
    x0 = np.zeros(n)
    xo, repo = C.lsqr_csc(m, n, Acsc.row_indices, Acsc.values, Acsc.col_pointers, M, b, x0, eps=0.0, maxit=4,
                          one_sync=True)
    x, rep = slq.lsqr_one_sync(Acsc, M, b, x0, slq.SolveOptions(eps=0.0, maxit=4))
    if n > 4:
        assert rep.iterations == repo.iterations
    assert np.linalg.norm(x - xo) <= 1e-10 * max(np.linalg.norm(xo), 1e-300)


@pytest.mark.parametrize("m,n,dens", [(40_000, 9000, 0.002), (20_000, 3000, 0.005)])
def test_sparse_two_pass_wide_n(m, n, dens):
    """Wide sparse rows: at n = 9000 the u_hat pass runs its smaller ring (p
    takes 72 KB of shared memory) and the A^T u_hat pass accumulates z in the
    global partials; at n = 3000 both keep their shared-memory layouts."""
    Acsc, A = rand_csc(m, n, dens, n, empty_rows=2)
    b = np.random.default_rng(n).standard_normal(m)
    rng = np.random.default_rng(1)
    M = np.asfortranarray(np.diag(1.0 / np.maximum(np.sqrt(np.asarray(A.multiply(A).sum(axis=0)).ravel()), 1e-3))
                          + np.triu(rng.standard_normal((n, n)), 1) * (1e-3 / np.sqrt(n)))
    x0 = np.zeros(n)
    xo, repo = C.lsqr_csc(m, n, Acsc.row_indices, Acsc.values, Acsc.col_pointers, M, b, x0, eps=0.0, maxit=5,
                          one_sync=True)
    x, rep = slq.lsqr_one_sync(Acsc, M, b, x0, slq.SolveOptions(eps=0.0, maxit=5))
    assert rep.iterations == repo.iterations == 5
    assert np.linalg.norm(x - xo) <= 1e-10 * np.linalg.norm(xo)
    assert np.allclose(rep.residual_estimate, repo.residual_estimate, rtol=1e-9)


# ----------------------------------------------- K2s column-slab gather


def _sketch_vs_oracle(Acsc, b, d, zeta, seed):
    Yo, Sbo = C.sketch_apply_csc(d, zeta, seed, Acsc.rows, Acsc.cols, Acsc.row_indices, Acsc.values,
                                 Acsc.col_pointers, b)
    dm = slq.SparseDeviceMatrix.from_csc(Acsc, b)
    Yd, Sbd = dm.sketch(d, zeta, seed)
    dm.free()
    return np.array_equal(Yd, Yo) and np.array_equal(Sbd, Sbo)


@pytest.mark.parametrize("wcap,kwin,lag", [(None, None, None), ("32", None, None), ("48", "512", "1"),
                                           ("100", "700", "3"), ("32", "64", "1")])
def test_sparse_apply_slab_gather(monkeypatch, wcap, kwin, lag):
    """S [A b] through the column-slab gather (every Y row resident, A walked in
    k windows under a soft grid barrier): bit-exact against the oracle's
    spmm(csc, csc) for slab widths down to 32 columns (segments longer than one
    group pass come from the long rows), several windows and lags, and the row
    gather (SLQ_K2S=row) on the same matrix."""
    for k, v in (("SLQ_K2S_W", wcap), ("SLQ_K2S_KWIN", kwin), ("SLQ_K2S_LAG", lag)):
        if v is not None:
            monkeypatch.setenv(k, v)
    Acsc, A = rand_csc(5000, 150, 0.1, 21, long_rows=4, empty_rows=3)
    b = np.random.default_rng(3).standard_normal(5000)
    assert _sketch_vs_oracle(Acsc, b, 600, 8, 19)
    monkeypatch.setenv("SLQ_K2S", "row")
    assert _sketch_vs_oracle(Acsc, b, 600, 8, 19)


def test_sparse_apply_slab_gather_two_slabs_natural():
    """d large enough that the Y rows of one CTA fill its shared memory: the
    slab count comes out > 1 without any override (d = 9000 on 148 SMs ->
    61 rows per CTA, ~417-column slabs for n + 1 = 601)."""
    Acsc, A = rand_csc(30_000, 600, 0.015, 8, long_rows=2, empty_rows=1)
    b = np.random.default_rng(5).standard_normal(30_000)
    assert _sketch_vs_oracle(Acsc, b, 9000, 4, 23)


def _cudart():
    import ctypes as ct
    import os

    import nvidia.cuda_runtime as cr
    lib = ct.CDLL(os.path.join(list(cr.__path__)[0], "lib", "libcudart.so.12"))
    lib.cudaMemcpy.argtypes = [ct.c_void_p, ct.c_void_p, ct.c_size_t, ct.c_int]
    return lib


def test_sparse_apply_slab_gather_unsorted_rows(monkeypatch):
    """A CSR written in place (slq_sparse_create_csr) whose rows are NOT sorted by
    column: the slab table marks those rows and the gather filters their
    entries by column -- still bit-exact (the per-element order is ascending
    k, whatever the order inside a row)."""
    m, n, d, zeta = 3000, 120, 500, 8
    Acsc, A = rand_csc(m, n, 0.08, 41, long_rows=2)
    R = A.tocsr()
    rng = np.random.default_rng(9)
    cols, vals = R.indices.astype(np.int32).copy(), R.data.copy()
    for r in range(0, m, 3):  # every third row shuffled
        lo, hi = R.indptr[r], R.indptr[r + 1]
        p = rng.permutation(hi - lo)
        cols[lo:hi], vals[lo:hi] = cols[lo:hi][p], vals[lo:hi][p]
    b = rng.standard_normal(m)
    dm, (rp, ci, vl, bp) = slq.SparseDeviceMatrix.create_csr(m, n, R.nnz)
    cu = _cudart()
    H2D = 1
    rowptr = R.indptr.astype(np.int64)
    for dst, src in ((rp, rowptr), (ci, cols), (vl, vals), (bp, b)):
        assert cu.cudaMemcpy(dst, src.ctypes.data, src.nbytes, H2D) == 0
    Yo, Sbo = C.sketch_apply_csc(d, zeta, 13, m, n, Acsc.row_indices, Acsc.values, Acsc.col_pointers, b)
    for wcap in ("32", "64", None):
        if wcap:
            monkeypatch.setenv("SLQ_K2S_W", wcap)
        else:
            monkeypatch.delenv("SLQ_K2S_W", raising=False)
        Yd, Sbd = dm.sketch(d, zeta, 13)
        assert np.array_equal(Yd, Yo) and np.array_equal(Sbd, Sbo)
    dm.free()


@pytest.mark.parametrize("d,zeta", [(600, 8), (20_000, 3), (64, 1)])
def test_sparse_apply_wide_and_narrow_sketches(d, zeta):
    """S [A b] bit-exact against the oracle for a sketch far taller than one
    CTA's shared memory holds per row set (d = 20000: 136 rows per CTA, slabs
    of ~180 columns) and for zeta = 1."""
    m = 25_000 if d > 1000 else 5000
    Acsc, A = rand_csc(m, 90, 0.05, d + zeta, long_rows=2, empty_rows=2)
    b = np.random.default_rng(d).standard_normal(m)
    assert _sketch_vs_oracle(Acsc, b, d, zeta, 31)


def test_sparse_apply_slab_tables_per_geometry(monkeypatch):
    """One matrix sketched under six slab geometries (the per-matrix cache holds
    four: the oldest is retired), then again after its right-hand side changed
    and after prepare() (tables dropped and rebuilt): bit-exact every time."""
    m, n, d, zeta = 4000, 130, 500, 8
    Acsc, A = rand_csc(m, n, 0.06, 77, long_rows=1)
    b = np.random.default_rng(7).standard_normal(m)
    Yo, Sbo = C.sketch_apply_csc(d, zeta, 9, m, n, Acsc.row_indices, Acsc.values, Acsc.col_pointers, b)
    dm = slq.SparseDeviceMatrix.from_csc(Acsc, b)
    for wcap in ("32", "40", "48", "64", "100", None, "32"):
        if wcap:
            monkeypatch.setenv("SLQ_K2S_W", wcap)
        else:
            monkeypatch.delenv("SLQ_K2S_W", raising=False)
        Yd, Sbd = dm.sketch(d, zeta, 9)
        assert np.array_equal(Yd, Yo) and np.array_equal(Sbd, Sbo)
    b2 = np.random.default_rng(8).standard_normal(m)
    dm.set_rhs(b2)
    dm.prepare()
    Yo2, Sbo2 = C.sketch_apply_csc(d, zeta, 9, m, n, Acsc.row_indices, Acsc.values, Acsc.col_pointers, b2)
    Yd, Sbd = dm.sketch(d, zeta, 9)
    assert np.array_equal(Yd, Yo2) and np.array_equal(Sbd, Sbo2)
    dm.free()
