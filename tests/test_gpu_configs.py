"""Parity at the BASELINE.json configurations: the device path against the
compiled reference (oracle/_ref: the unmodified sketchlsq headers) on the SAME
bytes.

Bars:
  (i)  sketch bits equal (checked in test_gpu_parity.py; here through S A);
  (ii) S A within 1e-12 max|Y| (fast mode), bit-identical in exact mode;
  (iii) R: diag >= 0, ||R - R_ref||_F / ||R_ref||_F <= 1e-12 cond(Y);
       Y M orthonormal no worse than the reference's own (10x, floor 1e-12);
  (iv) LSQR: same termination and iteration count under the reference rule;
       at fixed T, eta_gpu <= max(2 eta_ref, 1e-14) with
       eta(x) = ||A^T r|| / (||A||_2 ||r||), and
       ||A (x_gpu - x_ref)|| / ||b|| <= 1e-12 cond(A).
At cond 1e8 the solution itself moves ~1e-6 under a change of summation
order alone (the reference's serial vs threaded LSQR), so
parity is stated in backward-error / residual space there.

Every measured delta is appended to gpurun_out/parity_configs.jsonl (kept
under profiles/ per round).
"""
import json
import os

import numpy as np
import pytest

import oracle

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

slq = pytest.importorskip("paper_2506_03070_b200")
C = oracle.C()
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CORES = os.cpu_count() or 1


@pytest.fixture(scope="module")
def REF():
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    return oracle.REF()


def _log(case, **kv):
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "parity_configs.jsonl"), "a") as f:
        f.write(json.dumps({"case": case, **{k: (float(v) if isinstance(v, (np.floating, float)) else v)
                                            for k, v in kv.items()}}) + "\n")


def _eta(A, b, x, anorm=1.0):
    r = b - A @ x
    return float(np.linalg.norm(A.T @ r) / (anorm * np.linalg.norm(r)))


# ------------------------------------------------------------------ C1


@pytest.fixture(scope="module")
def c1(REF):
    """Config C1 verbatim: gen_dense(1e5, 100, 1e3, seed 1) (problems.hpp:45-66),
    gen_rhs(A, 0.5, seed 2) (problems.hpp:137-167), d = 4n, zeta = 8, seed 3."""
    A = REF.gen_dense(100_000, 100, 1e3, 1)
    b, xs = REF.gen_rhs(A, 0.5, 2)
    return A, b, xs


@pytest.mark.parametrize("one_sync", [True, False])
def test_c1_pipeline_vs_reference(c1, REF, one_sync):
    A, b, _ = c1
    m, n = A.shape
    d, zeta, seed = 4 * n, 8, 3
    # reference pipeline: generate_sparse_sign, apply, sketch_vector, build_preconditioner,
    # initial_guess, lsqr[_one_sync] with the default options (eps 1e-10, maxit 100)
    Y, Sb = REF.sketch_apply(d, zeta, seed, A, b)
    M, Q, x0, _ = REF.build_preconditioner(Y, Sb)
    xr, rr = REF.lsqr(A, M, b, x0, eps=1e-10, maxit=100, one_sync=one_sync)
    # device: the whole pipeline (sketch on the device, QR, LSQR) ...
    x, rep, _ = slq.solve(A, d, zeta, seed, slq.SolveOptions(eps=1e-10, maxit=100), b=b, one_sync=one_sync)
    assert str(rep.termination) == rr.termination and rep.iterations == rr.iterations, (rep, rr.iterations)
    anorm = np.linalg.norm(A, 2)
    eg, er = _eta(A, b, x, anorm), _eta(A, b, xr, anorm)
    dx = np.linalg.norm(x - xr) / np.linalg.norm(xr)
    assert dx <= 1e-10
    assert eg <= max(2 * er, 1e-14)
    assert np.allclose(rep.residual_estimate, rr.residual_estimate, rtol=1e-9, atol=1e-15)
    # ... and LSQR alone from the reference's own M, x0 (drop-in lsqr)
    fn = slq.lsqr_one_sync if one_sync else slq.lsqr
    x2, rep2 = fn(A, M, b, x0, slq.SolveOptions(eps=1e-10, maxit=100))
    assert rep2.iterations == rr.iterations and str(rep2.termination) == rr.termination
    dx2 = np.linalg.norm(x2 - xr) / np.linalg.norm(xr)
    assert dx2 <= 1e-10
    _log("C1 pipeline", one_sync=one_sync, iterations=rep.iterations, termination=str(rep.termination),
         rel_dx=dx, eta_gpu=eg, eta_ref=er, lsqr_only_rel_dx=dx2)


def test_c1_consistent_tolerance_rule(c1, REF):
    """Consistent variant (rho = 0, x0 = 0, test_solvers.cpp:360-373): the
    reference rule phi_bar <= eps beta_1 fires; same termination, iteration
    count within one (the last comparison sits at rounding level).  Both
    stop at a relative residual ~eps, so the iterates agree to ~eps cond(A)
    in x and ~eps in residual space."""
    A, _, xs = c1
    n = A.shape[1]
    b = A @ xs
    Y, _ = REF.sketch_apply(4 * n, 8, 3, A)
    M, _, _, _ = REF.build_preconditioner(Y)
    xr, rr = REF.lsqr(A, M, b, np.zeros(n), eps=1e-10, maxit=100, one_sync=True)
    x, rep = slq.lsqr_one_sync(A, M, b, np.zeros(n), slq.SolveOptions(eps=1e-10, maxit=100))
    assert rr.termination == "tolerance"
    assert str(rep.termination) == rr.termination and abs(rep.iterations - rr.iterations) <= 1
    dx = np.linalg.norm(x - xr) / np.linalg.norm(xr)
    dres = np.linalg.norm(A @ (x - xr)) / np.linalg.norm(b)
    assert dx <= 1e-10 * 1e3
    assert dres <= 2e-10
    _log("C1 consistent", iterations=rep.iterations, iterations_ref=rr.iterations, rel_dx=dx, res_delta=dres)


# ------------------------------------------------------- C2 (cond 1e8)


def test_c2_cond1e8_vs_reference_threaded(REF):
    """C2 shape: m = 2^20, n = 500, cond 1e8, rho = 0.5, d = 4n, zeta = 8.
    A comes from the device generator (bench.py make_problem) and the same
    bytes are copied to the host; the reference runs its threaded backend
    (WorkerPool(nproc): dist_generate_sparse_sign + dist_sketch_apply + serial
    QR + lsqr_one_sync(dist_operator)) for the same T."""
    import torch

    import bench

    m, n, T = 1 << 20, 500, 30
    d, zeta, seed = 4 * n, 8, 3
    dev = torch.device("cuda", 0)
    Abuf, ld, _ = bench.make_problem(torch, m, n, 1e8, 0.5, 0, m, dev)
    Ah = np.asfortranarray(Abuf[:, :n].cpu().numpy())
    bh = Abuf[:, n].cpu().numpy().copy()
    dm = slq.DeviceMatrix.wrap(Abuf.data_ptr(), m, n, ld, owner=Abuf)
    x, rep, _ = slq.solve(dm, d, zeta, seed, slq.SolveOptions(eps=0.0, maxit=T))
    xr, rr, _ = REF.solve_timed(Ah, bh, d, zeta, seed, 0.0, T, CORES)
    assert rep.iterations == rr.iterations == T
    At = Abuf[:, :n]
    bt = Abuf[:, n]

    def eta(v):  # ||A||_2 = 1 by construction (sigma_max = 1)
        r = bt - At @ torch.from_numpy(v).to(dev)
        return float(torch.linalg.norm(At.T @ r) / torch.linalg.norm(r))

    eg, er = eta(x), eta(xr)
    dres = float(torch.linalg.norm(At @ torch.from_numpy(x - xr).to(dev)) / torch.linalg.norm(bt))
    dx = np.linalg.norm(x - xr) / np.linalg.norm(xr)
    _log("C2 cond1e8 vs reference threaded", m=m, n=n, T=T, eta_gpu=eg, eta_ref=er, res_delta=dres, rel_dx=dx,
         ref_cores=CORES)
    assert eg <= max(2 * er, 1e-14)
    assert dres <= 1e-12 * 1e8
    assert eg <= 1e-9  # both reach the backward-error regime at T = 30


# ------------------------------------------------------- QR at C3 / C4


@pytest.mark.parametrize("d,n", [(4000, 1000), (8000, 2000)])
def test_qr_inverse_at_config_shapes(d, n):
    """K3 at the shapes the C3 / C4 solves factor: Y (d x n) with cond 1e8
    against the oracle's householder_qr + tri_inverse."""
    rng = np.random.default_rng(d + n)
    U, _ = np.linalg.qr(rng.standard_normal((d, n)))
    V, _ = np.linalg.qr(rng.standard_normal((n, n)))
    s = 10.0 ** (-8.0 * np.arange(n) / (n - 1))
    Y = np.asfortranarray((U * s) @ V.T)
    cond = 1e8
    got = slq.householder_qr(Y)
    _, Ro = C.householder_qr(Y, want_q=False)
    assert np.all(np.diag(got.R) >= 0) and np.allclose(np.tril(got.R, -1), 0.0)
    dR = np.linalg.norm(got.R - Ro) / np.linalg.norm(Ro)
    assert dR <= 1e-12 * cond
    M = slq.tri_inverse(got.R)
    Mo = C.tri_inverse(Ro)

    def orth(Mx):
        W = Y @ Mx
        return float(np.abs(W.T @ W - np.eye(n)).max())

    og, oo = orth(M), orth(Mo)
    assert og <= max(10 * oo, 1e-12)
    assert np.abs(got.Q.T @ got.Q - np.eye(n)).max() <= 1e-12 * d
    _log("QR+inverse", d=d, n=n, cond=cond, rel_dR=dR, orth_gpu=og, orth_ref=oo)


# ------------------------------------------------ S A at m >= 2^20


def test_sketch_apply_large_fast_vs_exact_vs_oracle():
    m, n, d, zeta, seed = 1 << 20, 128, 512, 8, 3
    rng = np.random.default_rng(20)
    A = np.asfortranarray(rng.standard_normal((m, n)))
    b = rng.standard_normal(m)
    dm = slq.DeviceMatrix.from_numpy(A, b)
    Ye, Sbe = dm.sketch(d, zeta, seed, exact=True)
    Yf, Sbf = dm.sketch(d, zeta, seed, exact=False)
    Yo, Sbo = C.sketch_apply(d, zeta, seed, A, b)
    assert np.array_equal(Ye, Yo) and np.array_equal(Sbe, Sbo)
    tol = 1e-12 * max(1.0, np.abs(Yo).max())
    dmax = float(max(np.abs(Yf - Yo).max(), np.abs(Sbf - Sbo).max()))
    assert dmax <= tol
    _log("S A m=2^20", m=m, n=n, d=d, zeta=zeta, exact_bitwise=True, fast_max_abs_delta=dmax,
         fast_rel_delta=dmax / np.abs(Yo).max())


# ------------------------------------------------ sparse A at 2^20 rows


def test_sparse_2p20_vs_reference(REF):
    """C4-like operand at m = 2^20 rows: n = 200, ~50 nnz per row (each entry
    present with probability 1/4), values +-sigma_j, sigma log-spaced in
    [1e-6, 1] (cond ~1e6); d = 4n, zeta = 8.  S A bit-identical to the
    reference spmm(csc, csc); LSQR (T = 25) in backward-error space against
    the reference lsqr_one_sync over its threaded CscMatrix operator."""
    import scipy.sparse as sp

    m, n, T = 1 << 20, 200, 25
    d, zeta, seed = 4 * n, 8, 3
    rng = np.random.default_rng(44)
    mask = rng.random((m, n), dtype=np.float32) < 0.25
    sigma = 10.0 ** (-6.0 * np.arange(n) / (n - 1))
    As = sp.csc_matrix(mask, dtype=np.float64)
    del mask
    As.data = np.where(rng.random(As.nnz) < 0.5, -1.0, 1.0) * sigma[np.repeat(np.arange(n), np.diff(As.indptr))]
    As.sort_indices()
    rows, colptr = As.indices.astype(np.int64), As.indptr.astype(np.int64)
    b = rng.uniform(-1, 1, m)
    Acsc = slq.CscMatrix(m, n, As.data, rows, colptr)
    # S A: bit-identical to the reference's spmm(csc, csc)
    Yr = REF.sketch_apply_csc(d, zeta, seed, m, n, rows, As.data, colptr)
    Y, Sb = slq.SparseDeviceMatrix.from_csc(Acsc, b).sketch(d, zeta, seed)
    assert np.array_equal(Y, Yr)
    _, Sbo = C.sketch_apply_csc(d, zeta, seed, m, n, rows, As.data, colptr, b)
    assert np.array_equal(Sb, Sbo)
    # LSQR from the reference's preconditioner and x0
    M, Q, x0, _ = REF.build_preconditioner(Yr, Sbo)
    xr, rr = REF.lsqr_csc(m, n, rows, As.data, colptr, M, b, x0, eps=0.0, maxit=T, one_sync=True, workers=CORES)
    x, rep, _ = slq.solve(Acsc, d, zeta, seed, slq.SolveOptions(eps=0.0, maxit=T), b=b)
    assert rep.iterations == rr.iterations == T
    # ||A||_2 by power iteration (shared by both etas)
    v = np.ones(n) / np.sqrt(n)
    for _ in range(30):
        v = As.T @ (As @ v)
        v /= np.linalg.norm(v)
    anorm = float(np.sqrt(np.linalg.norm(As.T @ (As @ v))))
    eg, er = _eta(As, b, x, anorm), _eta(As, b, xr, anorm)
    dres = float(np.linalg.norm(As @ (x - xr)) / np.linalg.norm(b))
    dx = np.linalg.norm(x - xr) / np.linalg.norm(xr)
    _log("sparse m=2^20", m=m, n=n, nnz=int(As.nnz), T=T, eta_gpu=eg, eta_ref=er, res_delta=dres, rel_dx=dx)
    assert eg <= max(2 * er, 1e-14)
    assert dres <= 1e-12 * 1e6
