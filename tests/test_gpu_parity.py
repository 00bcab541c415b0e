"""GPU parity tests: the sm_100a path through the C-ABI vs the CPU oracle.

Bars:
  * sketch row indices / values / col pointers / RejectionStats: bit-exact;
  * S A and S b: bit-exact in exact (serial-order) mode, else 1e-12 max|Y|
    (test_distsim.cpp:169);
  * QR / R^-1 / x0: relative 1e-12 cond(Y) on R, orthonormality 1e-12 d
    (test_core_linalg.cpp:29-87, test_preconditioning.cpp:30-46);
  * LSQR: same termination / iteration count; iterates within 1e-10 of the
    oracle at cond <= 1e3 (reduction order only), residual histories 1e-10.
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

slq = pytest.importorskip("paper_2506_03070_b200")
C = oracle.C()


def _csc_equal(S, rows, vals, colptr):
    assert np.array_equal(S.matrix.row_indices, rows)
    assert np.array_equal(S.matrix.values, vals)
    assert np.array_equal(S.matrix.col_pointers, colptr)


# ------------------------------------------------------------------ K1


def test_generator_golden(golden):
    arr = golden["sketch"]
    for i, c in enumerate(golden["meta"]["sketch_cases"]):
        st = slq.RejectionStats()
        M = slq.sparse_sign_block(c["d"], c["zeta"], c["seed"], c["col_begin"], c["col_begin"] + c["m"], st)
        assert np.array_equal(M.row_indices, arr[f"rows_{i}"]), c
        assert np.array_equal(M.values, arr[f"vals_{i}"]), c
        assert np.array_equal(M.col_pointers, arr[f"colptr_{i}"]), c
        assert (st.columns_resampled, st.resample_rounds) == (c["columns_resampled"], c["resample_rounds"]), c


@pytest.mark.parametrize("d,zeta", [(4000, 8), (400, 8), (64, 16), (33, 32), (2000, 2), (8000, 4), (12, 12), (5, 3)])
def test_generator_vs_oracle_sweep(d, zeta):
    m = 20000
    for seed in (0, 3, 2**63 + 5):
        S = slq.generate_sparse_sign(d, m, zeta, seed)
        rows, vals, colptr, st = C.generate_sparse_sign(d, m, zeta, seed)
        _csc_equal(S, rows, vals, colptr)


def test_rejection_stats_large(golden):
    for c in golden["meta"]["stats_cases"]:
        st = slq.RejectionStats()
        slq.generate_sparse_sign(c["d"], c["m"], c["zeta"], c["seed"], stats=st)
        assert (st.columns_resampled, st.resample_rounds) == (c["columns_resampled"], c["resample_rounds"])


def test_rejection_sample_columns():
    st = slq.RejectionStats()
    got = slq.rejection_sample_columns(400, 5000, 8, 77, st)
    ref, rst = C.rejection_sample_columns(400, 5000, 8, 77)
    assert np.array_equal(got, ref)
    assert (st.columns_resampled, st.resample_rounds) == rst


def test_partitioned_generation_bit_identical():
    # test_distsim.cpp:136-149: any partition of the columns reproduces the sketch
    d, m, zeta, seed = 96, 333, 5, 271828
    full = slq.generate_sparse_sign(d, m, zeta, seed)
    for p in (1, 2, 4, 8):
        part = slq.partition_rows(m, p)
        blocks = [slq.sparse_sign_block(d, zeta, seed, part.begin(k), part.end(k)) for k in range(p)]
        rows = np.concatenate([b.row_indices for b in blocks])
        vals = np.concatenate([b.values for b in blocks])
        assert np.array_equal(rows, full.matrix.row_indices)
        assert np.array_equal(vals, full.matrix.values)


def test_generator_errors():
    with pytest.raises(slq.InvalidSparsity):
        slq.generate_sparse_sign(3, 1, 4, 0)
    with pytest.raises(slq.InvalidSparsity):
        slq.rejection_sample_columns(3, 1, 0, 0)


# ------------------------------------------------------------------ K2


@pytest.mark.parametrize("m,n,d,zeta", [(600, 24, 96, 6), (5000, 37, 200, 8), (3000, 3, 64, 1), (4096, 64, 512, 16),
                                        (3000, 40, 6000, 8), (2500, 12, 12000, 4)])
def test_apply_exact(m, n, d, zeta):
    rng = np.random.default_rng(m + n)
    A = np.asfortranarray(rng.standard_normal((m, n)))
    A[rng.random((m, n)) < 0.05] = 0.0
    b = rng.standard_normal(m)
    S = slq.generate_sparse_sign(d, m, zeta, 93)
    Y = slq.apply(S, A)
    Yo, Sbo = C.sketch_apply(d, zeta, 93, A, b)
    assert np.array_equal(Y, Yo)  # bit-identical: same order, IEEE mul+add
    assert np.array_equal(slq.sketch_vector(S, b), Sbo)
    # fused device path (generate + apply on resident [A | b])
    dm = slq.DeviceMatrix.from_numpy(A, b)
    Ye, Sbe = dm.sketch(d, zeta, 93, exact=True)
    assert np.array_equal(Ye, Yo) and np.array_equal(Sbe, Sbo)
    Yf, Sbf = dm.sketch(d, zeta, 93, exact=False)
    tol = 1e-12 * max(1.0, np.abs(Yo).max())
    assert np.abs(Yf - Yo).max() <= tol and np.abs(Sbf - Sbo).max() <= tol


@pytest.mark.parametrize("m,n,d,zeta", [(513, 16, 1030, 8), (1, 5, 40, 3), (2000, 47, 8, 8), (7000, 15, 2100, 32),
                                        (1537, 33, 1500, 2), (2000, 10, 3000, 64), (900, 6, 700, 1)])
def test_apply_fast_tile_gather(m, n, d, zeta, monkeypatch):
    """Fast mode runs the DMMA tile gather (K2d); it must agree with the
    reference order to 1e-12 and with the register gather (SLQ_ROW_GATHER=1):
    partial chunks, partial 16-column slabs, several 1024-row blocks, zeta up
    to 32."""
    rng = np.random.default_rng(m * 7 + d)
    A = np.asfortranarray(rng.standard_normal((m, n)))
    b = rng.standard_normal(m)
    Yo, Sbo = C.sketch_apply(d, zeta, 29, A, b)
    dm = slq.DeviceMatrix.from_numpy(A, b)
    Yf, Sbf = dm.sketch(d, zeta, 29, exact=False)
    monkeypatch.setenv("SLQ_ROW_GATHER", "1")
    Yr, Sbr = dm.sketch(d, zeta, 29, exact=False)
    tol = 1e-12 * max(1.0, np.abs(Yo).max())
    assert np.abs(Yf - Yo).max() <= tol and np.abs(Sbf - Sbo).max() <= tol
    assert np.abs(Yf - Yr).max() <= tol and np.abs(Sbf - Sbr).max() <= tol


def test_apply_fast_tile_gather_overflow_falls_back(monkeypatch):
    """A row block whose entries overflow the tile bucket (forced with a tiny
    SLQ_TD_CAP) is detected and the apply is redone by the register gather."""
    m, n, d, zeta = 3000, 20, 600, 8
    rng = np.random.default_rng(9)
    A = np.asfortranarray(rng.standard_normal((m, n)))
    b = rng.standard_normal(m)
    Yo, Sbo = C.sketch_apply(d, zeta, 41, A, b)
    monkeypatch.setenv("SLQ_TD_CAP", "64")
    Yf, Sbf = slq.DeviceMatrix.from_numpy(A, b).sketch(d, zeta, 41, exact=False)
    tol = 1e-12 * max(1.0, np.abs(Yo).max())
    assert np.abs(Yf - Yo).max() <= tol and np.abs(Sbf - Sbo).max() <= tol


def test_apply_fast_tile_gather_tall_sketch():
    """d = 20000 is past the register gather's envelope (d <= 16384); the
    tile gather covers it in fast mode (20 row blocks of 1024)."""
    m, n, d, zeta = 6000, 9, 20000, 4
    rng = np.random.default_rng(5)
    A = np.asfortranarray(rng.standard_normal((m, n)))
    b = rng.standard_normal(m)
    Yo, Sbo = C.sketch_apply(d, zeta, 31, A, b)
    Yf, Sbf = slq.DeviceMatrix.from_numpy(A, b).sketch(d, zeta, 31, exact=False)
    tol = 1e-12 * max(1.0, np.abs(Yo).max())
    assert np.abs(Yf - Yo).max() <= tol and np.abs(Sbf - Sbo).max() <= tol


def test_apply_golden(golden):
    p = golden["pipeline"]
    meta = golden["meta"]["pipeline"]
    dm = slq.DeviceMatrix.from_numpy(p["A"], p["b"])
    Y, Sb = dm.sketch(meta["d"], meta["zeta"], meta["seed_S"], exact=True)
    assert np.array_equal(Y, p["Y"]) and np.array_equal(Sb, p["Sb"])


def test_apply_identity_sketch():
    # test_core_linalg.cpp:178-190: identity S reproduces A
    m, n = 50, 7
    A = np.asfortranarray(np.random.default_rng(1).standard_normal((m, n)))
    I = slq.CscMatrix(m, m, np.ones(m), np.arange(m, dtype=np.int64), np.arange(m + 1, dtype=np.int64))
    Y = slq.apply(slq.SparseSignSketch(I, 1, 0), A)
    assert np.array_equal(Y, A)


@pytest.mark.parametrize("d,m,n,dens", [(9, 12, 5, 0.3), (300, 2000, 17, 0.01), (64, 5000, 40, 0.05)])
def test_spmm_general_values_bit_exact(d, m, n, dens):
    """spmm(csc, dense) / spmm(csc, csc) with arbitrary S values (not a sparse
    sign matrix) -- the reference's order, bit for bit (test_core_linalg.cpp:192-224)."""
    rng = np.random.default_rng(d + m)
    mask = rng.random((d, m)) < dens
    Sd = np.where(mask, rng.standard_normal((d, m)), 0.0)
    cols = [np.nonzero(mask[:, k])[0] for k in range(m)]
    rows = np.concatenate(cols).astype(np.int64) if cols else np.zeros(0, np.int64)
    vals = np.concatenate([Sd[c, k] for k, c in enumerate(cols)])
    colptr = np.concatenate([[0], np.cumsum([len(c) for c in cols])]).astype(np.int64)
    A = np.asfortranarray(rng.standard_normal((m, n)))
    A[rng.random((m, n)) < 0.2] = 0.0
    S = slq.CscMatrix(d, m, vals, rows, colptr)
    Y = slq.apply(slq.SparseSignSketch(S, 1, 0), A)
    assert np.array_equal(Y, C.spmm(d, rows, vals, colptr, A))
    amask = rng.random((m, n)) < 0.1
    acols = [np.nonzero(amask[:, j])[0] for j in range(n)]
    arows = np.concatenate(acols).astype(np.int64)
    avals = rng.standard_normal(arows.size)
    acp = np.concatenate([[0], np.cumsum([len(c) for c in acols])]).astype(np.int64)
    Ya = slq.apply(slq.SparseSignSketch(S, 1, 0), slq.CscMatrix(m, n, avals, arows, acp))
    assert np.array_equal(Ya, C.spmm_csc(d, rows, vals, colptr, m, n, arows, avals, acp))


def test_apply_dimension_mismatch():
    S = slq.generate_sparse_sign(10, 20, 2, 1)
    with pytest.raises(slq.DimensionMismatch):
        slq.apply(S, np.zeros((21, 3)))


# ------------------------------------------------------------------ K3


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


# (5000, 70) / (9000, 40): taller than one 16-CTA cluster x 256 rows, so the
# narrow next-panel update restages its rows in chunks; (9000, 40) also takes
# the shared-memory panel
@pytest.mark.parametrize("d,n", [(96, 24), (400, 100), (130, 33), (1000, 250), (64, 64), (2000, 40), (5000, 70),
                                 (9000, 40)])
def test_qr_vs_oracle(d, n):
    rng = np.random.default_rng(d * n)
    Y = np.asfortranarray(rng.standard_normal((d, n)) @ np.diag(np.logspace(0, -4, n)))
    got = slq.householder_qr(Y)
    Qo, Ro = C.householder_qr(Y)
    cond = np.linalg.cond(Y)
    assert np.all(np.diag(got.R) >= 0)
    assert np.allclose(np.tril(got.R, -1), 0.0)
    assert _rel(got.R, Ro) <= 1e-12 * cond
    assert np.abs(got.Q.T @ got.Q - np.eye(n)).max() <= 1e-12 * d
    assert np.linalg.norm(got.Q @ got.R - Y) <= 1e-13 * np.sqrt(d * n) * np.linalg.norm(Y)


def test_qr_known_answers():
    # test_core_linalg.cpp:29-60: identity and R00 = 5
    I = np.eye(6)
    qr = slq.householder_qr(I)
    assert np.allclose(qr.R, np.eye(6), atol=1e-15) and np.allclose(qr.Q, np.eye(6), atol=1e-15)
    Y = np.array([[3.0, 1.0], [4.0, 2.0], [0.0, 1.0]])
    assert abs(slq.householder_qr(Y).R[0, 0] - 5.0) <= 1e-14


def test_qr_rank_deficient():
    Y = np.ones((10, 3))
    with pytest.raises(slq.RankDeficient):
        slq.householder_qr(Y)
    with pytest.raises(slq.DimensionMismatch):
        slq.householder_qr(np.ones((2, 3)))


def test_tri_inverse():
    rng = np.random.default_rng(5)
    for n in (1, 7, 100, 333):
        R = np.triu(rng.standard_normal((n, n))) + 3 * np.eye(n)
        M = slq.tri_inverse(R)
        Mo = C.tri_inverse(R)
        cond = np.linalg.cond(R)
        assert np.allclose(np.tril(M, -1), 0.0)
        assert np.abs(M @ R - np.eye(n)).max() <= 1e-10 * cond  # test_core_linalg.cpp:120-136
        assert _rel(M, Mo) <= 1e-13 * cond
    R = np.eye(3)
    R[1, 1] = 0.0
    with pytest.raises(slq.SingularTriangular):
        slq.tri_inverse(R)


def test_preconditioner_and_x0(golden):
    p = golden["pipeline"]
    P, x0 = slq.build_preconditioner(p["Y"], Sb=p["Sb"])
    cond = np.linalg.cond(p["Y"])
    assert _rel(P.M, p["M"]) <= 1e-12 * cond
    assert np.abs(P.Q.T @ P.Q - np.eye(P.M.shape[0])).max() <= 1e-10  # test_preconditioning.cpp:30-46
    assert np.abs(p["Y"] @ P.M - P.Q).max() <= 1e-10
    assert _rel(x0, p["x0"]) <= 1e-12 * cond
    x0b = slq.initial_guess(P, p["Sb"])
    assert _rel(x0b, p["x0"]) <= 1e-12 * cond
    v = np.random.default_rng(2).standard_normal(P.M.shape[0])
    assert np.allclose(slq.apply_M(P, v), C.apply_M(P.M, v), rtol=1e-12, atol=1e-12 * np.abs(P.M).max())
    assert np.allclose(slq.apply_Mt(P, v), C.apply_Mt(P.M, v), rtol=1e-12, atol=1e-12 * np.abs(P.M).max())


# ------------------------------------------------------------------ K4/K5


def test_lsqr_golden(golden):
    p = golden["pipeline"]
    meta = golden["meta"]["pipeline"]
    for one_sync in (False, True):
        fn = slq.lsqr_one_sync if one_sync else slq.lsqr
        x, rep = fn(p["A"], p["M"], p["b"], p["x0"], slq.SolveOptions(eps=0.0, maxit=meta["maxit"], x_star=p["x_star"],
                                                                      track_true_residual=True))
        xref = p["x_one"] if one_sync else p["x_std"]
        assert rep.iterations == meta["maxit"] and rep.termination == slq.Termination.MaxIter
        assert np.linalg.norm(x - xref) <= 1e-10 * np.linalg.norm(xref)
        est_ref = p["est_one"] if one_sync else p["est_std"]
        assert np.allclose(rep.residual_estimate, est_ref, rtol=1e-9, atol=1e-14)
        if not one_sync:
            assert np.allclose(rep.iterates_error, p["err_std"], rtol=1e-6, atol=1e-13)
            assert np.allclose(rep.residual_true, p["true_std"], rtol=1e-10, atol=1e-14)
    x, rep = slq.lsqr(p["A"], p["M"], p["b"], np.zeros(meta["n"]), slq.SolveOptions(eps=1e-10, maxit=100))
    assert str(rep.termination) == meta["tol_run"]["termination"]
    assert abs(rep.iterations - meta["tol_run"]["iterations"]) <= 1
    assert np.linalg.norm(x - p["x_tol"]) <= 1e-9 * np.linalg.norm(p["x_tol"])


def test_lsqr_identity_one_iteration():
    n = 5
    b = np.array([1.0, -2.0, 0.5, 3.0, 0.25])
    x, rep = slq.lsqr(np.eye(n), slq.Preconditioner.identity(n), b, np.zeros(n))
    assert rep.iterations == 1 and rep.termination != slq.Termination.MaxIter
    assert np.allclose(x, b, rtol=1e-12)


def test_lsqr_hand_instance_and_breakdown():
    A = np.array([[1.0, 0], [0, 1], [1, 1]])
    x, rep = slq.lsqr(A, np.eye(2), np.array([1.0, 2, 0]), np.zeros(2), slq.SolveOptions(eps=1e-14, maxit=2))
    assert abs(x[0]) <= 1e-10 and abs(x[1] - 1) <= 1e-10 and rep.iterations <= 2
    x, rep = slq.lsqr(np.eye(4), np.eye(4), np.array([2.0, 0, 0, 0]), np.zeros(4), slq.SolveOptions(eps=0.0, maxit=5))
    assert rep.termination == slq.Termination.Breakdown and rep.iterations == 1
    assert np.allclose(x, [2.0, 0, 0, 0], atol=1e-14)
    x, rep = slq.lsqr(np.eye(3), np.eye(3), np.zeros(3), np.zeros(3))
    assert rep.iterations == 0 and rep.termination == slq.Termination.Tolerance


def test_lsqr_bidiag_unit_vectors():
    A = C.gen_dense(400, 20, 50.0, 900)
    b, xs = C.gen_rhs(A, 0.5, 901)
    Y, Sb = C.sketch_apply(120, 6, 902, A, b)
    M, Q = C.build_preconditioner(Y)
    x0 = C.initial_guess(M, Q, Sb)
    worst = [0.0, 0.0]

    def hook(t, un, vn):
        worst[0] = max(worst[0], abs(un - 1))
        worst[1] = max(worst[1], abs(vn - 1))

    slq.lsqr(A, M, b, x0, slq.SolveOptions(eps=0.0, maxit=15, on_bidiag=hook))
    assert worst[0] <= 1e-10 and worst[1] <= 1e-10


def test_solve_pipeline_c1_small():
    # end-to-end device pipeline vs the oracle pipeline at a C1-like shape
    m, n, d, zeta = 20000, 50, 200, 8
    A = C.gen_dense(m, n, 1e3, 1)
    b, xs = C.gen_rhs(A, 0.5, 2)
    x, rep, times = slq.solve(A, d, zeta, 3, slq.SolveOptions(eps=0.0, maxit=20), b=b)
    Y, Sb = C.sketch_apply(d, zeta, 3, A, b)
    M, Q = C.build_preconditioner(Y)
    x0 = C.initial_guess(M, Q, Sb)
    xo, repo = C.lsqr(A, M, b, x0, eps=0.0, maxit=20, one_sync=True)
    assert rep.iterations == 20
    assert np.linalg.norm(x - xo) <= 1e-9 * np.linalg.norm(xo)
    assert np.allclose(rep.residual_estimate, repo.residual_estimate, rtol=1e-8)
    def eta(v):
        r = b - A @ v
        return np.linalg.norm(A.T @ r) / (np.linalg.norm(A, 2) * np.linalg.norm(r))

    # backward error no worse than the reference's at fixed T
    assert eta(x) <= max(2 * eta(xo), 1e-14)
    assert times["kernel_launches"] > 0


def test_solve_deterministic_across_runs_and_contexts():
    """Every reduction is in a fixed order (no atomics on floating-point data):
    repeated fast-mode solves -- same context and a fresh one -- return
    bit-identical x and residual histories."""
    m, n, d, zeta = 60000, 120, 480, 8
    rng = np.random.default_rng(17)
    A = np.asfortranarray(rng.standard_normal((m, n)))
    b = rng.standard_normal(m)
    opts = slq.SolveOptions(eps=0.0, maxit=15)
    x1, r1, _ = slq.solve(A, d, zeta, 5, opts, b=b)
    x2, r2, _ = slq.solve(A, d, zeta, 5, opts, b=b)
    x3, r3, _ = slq.solve(A, d, zeta, 5, opts, b=b, ctx=slq.Context(0))
    assert np.array_equal(x1, x2) and np.array_equal(x1, x3)
    assert np.array_equal(r1.residual_estimate, r2.residual_estimate)
    assert np.array_equal(r1.residual_estimate, r3.residual_estimate)


@pytest.mark.parametrize("block_rows", [None, "5000"])
def test_solve_host_streams_blocks(block_rows, monkeypatch):
    """slq_solve_host (e2e path): A uploaded block by block from a column-major
    host buffer with the sketch applied to each block as it lands; same solve as
    the device-resident path up to summation order."""
    import ctypes as ct
    from paper_2506_03070_b200 import _capi as CA
    if block_rows:
        monkeypatch.setenv("SLQ_UPLOAD_ROWS", block_rows)  # several blocks (rounded to the chunk size)
    rng = np.random.default_rng(8)
    m, n, d, zeta, T = 30000, 40, 160, 8, 20
    A = np.asfortranarray(rng.standard_normal((m, n)) @ np.diag(np.logspace(0, -3, n)))
    b = rng.standard_normal(m)
    ctx = slq.Context(0)
    co = CA.SolveOpts()
    CA.lib.slq_solve_opts_default(ct.byref(co))
    co.eps, co.maxit, co.one_sync = 0.0, T, 1
    x = np.zeros(n)
    rep = CA.Report()
    st = CA.lib.slq_solve_host(ctx.handle, A.ctypes.data_as(CA.dp), m, n, m, b.ctypes.data_as(CA.dp), 0, d, zeta, 5,
                               ct.byref(co), x.ctypes.data_as(CA.dp), ct.byref(rep), None, None)
    assert st == 0, CA.lib.slq_last_error()
    xr, repr_, _ = slq.solve(slq.DeviceMatrix.from_numpy(A, b), d, zeta, 5, slq.SolveOptions(eps=0.0, maxit=T))
    assert rep.iterations == repr_.iterations == T
    assert np.linalg.norm(x - xr) <= 1e-9 * np.linalg.norm(xr)
    Y, Sb = C.sketch_apply(d, zeta, 5, A, b)
    M, Q = C.build_preconditioner(Y)
    xo, _ = C.lsqr(A, M, b, C.initial_guess(M, Q, Sb), eps=0.0, maxit=T, one_sync=True)
    assert np.linalg.norm(x - xo) <= 1e-9 * np.linalg.norm(xo)
