"""The shape envelope beyond round 1's limits, against the oracle:
  * n > 2046: the wide-row LSQR pass (columns split across the consumer warps);
  * d > 12400: TSQR of tall sketches (row blocks factored independently, R's
    stacked and factored again), R / x0 against householder_qr /
    initial_guess of the reference;
  * the paper's strong-scaling shape family (n = 4000,
    d = 8n, zeta = 12) end to end at a reduced m, in backward-error space."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

slq = pytest.importorskip("paper_2506_03070_b200")
C = oracle.C()


def _eta(A, b, x):
    r = b - A @ x
    return np.linalg.norm(A.T @ r) / (np.linalg.norm(A, 2) * np.linalg.norm(r))


@pytest.mark.parametrize("m,n", [(6000, 2100), (5000, 3000), (6000, 4500), (8500, 8000),
                                 (3000, 150), (4000, 700), (5000, 1100), (5000, 1500), (4000, 2000)])
def test_wide_pass_lsqr_vs_oracle(m, n):
    """K4 at every slot count: wide rows (ld > 2048, NQ = 6 / 9 / 12 / 18) and
    the one-warp-per-row pass at NP = 4 (quad path), 12, 24 (row re-read for
    the z update), 32: LSQR iterates against the oracle's lsqr_one_sync at a
    fixed T from the same M and x0."""
    rng = np.random.default_rng(n)
    A = np.asfortranarray(rng.standard_normal((m, n)) * np.logspace(0, -2, n))
    b = rng.standard_normal(m)
    # any upper-triangular preconditioner exercises the same machinery: column
    # scaling plus a small strictly upper part
    M = np.asfortranarray(np.diag(1.0 / np.linalg.norm(A, axis=0))
                          + np.triu(rng.standard_normal((n, n)), 1) * (1e-3 / np.sqrt(n)))
    x0 = np.zeros(n)
    T = 6
    x, rep = slq.lsqr_one_sync(A, M, b, x0, slq.SolveOptions(eps=0.0, maxit=T))
    xo, repo = C.lsqr(A, M, b, x0, eps=0.0, maxit=T, one_sync=True)
    assert rep.iterations == T
    assert np.linalg.norm(x - xo) <= 1e-9 * np.linalg.norm(xo)
    assert np.allclose(rep.residual_estimate, repo.residual_estimate, rtol=1e-9)


@pytest.mark.parametrize("d,n", [(20000, 40), (30000, 120), (60000, 64)])
def test_tsqr_tall_sketch_vs_oracle(d, n):
    rng = np.random.default_rng(d + n)
    Y = np.asfortranarray(rng.standard_normal((d, n)) @ np.diag(np.logspace(0, -6, n)))
    Sb = rng.standard_normal(d)
    P, x0 = slq.build_preconditioner(Y, Sb=Sb, want_q=False)
    _, Ro = C.householder_qr(Y, want_q=False)
    Mo = C.tri_inverse(Ro)
    cond = np.linalg.cond(Y)
    Rg = np.linalg.inv(P.M)
    assert np.linalg.norm(Rg - Ro) / np.linalg.norm(Ro) <= 1e-12 * cond
    # x0 = M Q^T Sb: the sketched least-squares solution
    x0o = np.linalg.lstsq(Y, Sb, rcond=None)[0]
    assert np.linalg.norm(x0 - x0o) <= 1e-12 * cond * np.linalg.norm(x0o)
    W = Y @ P.M
    assert np.abs(W.T @ W - np.eye(n)).max() <= max(10 * np.abs((Y @ Mo).T @ (Y @ Mo) - np.eye(n)).max(), 1e-12)


def test_tsqr_wide_leaves():
    """n > 4096 with d > 12400: TSQR leaves of 2n rows (here 2 leaves of 8400),
    R against LAPACK's (numpy) QR with the diagonal made nonnegative."""
    d, n = 16800, 4200
    rng = np.random.default_rng(7)
    Y = np.asfortranarray(rng.standard_normal((d, n)) * np.logspace(0, -3, n))
    P, _ = slq.build_preconditioner(Y, Sb=rng.standard_normal(d), want_q=False)
    Rn = np.linalg.qr(Y, mode="r")
    Rn *= np.sign(np.diag(Rn))[:, None]
    Rg = np.linalg.inv(P.M)
    assert np.linalg.norm(Rg - Rn) / np.linalg.norm(Rn) <= 1e-12 * np.linalg.cond(Rn)


def test_tsqr_rank_deficient_detected():
    rng = np.random.default_rng(2)
    Y = np.asfortranarray(rng.standard_normal((20000, 10)))
    Y[:, 7] = Y[:, 3]
    with pytest.raises(slq.RankDeficient):
        slq.build_preconditioner(Y, Sb=np.ones(20000), want_q=False)


def test_paper_shape_family_reduced_m():
    """n = 4000 is the paper's strong-scaling width; d = 8n = 32000 > 12400
    (TSQR) and zeta = 12.  At m = 60000 the whole pipeline runs on the device
    (wide-row pass, TSQR, K2d with 32 row blocks) and reaches the backward
    error target; against a lstsq solution of the same system."""
    import torch

    import bench

    m, n = 60000, 4000
    d, zeta, T = 8 * n, 12, 24  # ~sqrt(n/d) = 0.35 per iteration
    dev = torch.device("cuda", 0)
    Abuf, ld, _ = bench.make_problem(torch, m, n, 1e4, 0.5, 0, m, dev)
    dm = slq.DeviceMatrix.wrap(Abuf.data_ptr(), m, n, ld, owner=Abuf)
    x, rep, ph = slq.solve(dm, d, zeta, 3, slq.SolveOptions(eps=0.0, maxit=T, a_norm_est=1.0))
    assert rep.iterations == T
    assert rep.backward_error <= 1e-10, rep.backward_error
    A = Abuf[:, :n]
    b = Abuf[:, n]
    xl = torch.linalg.lstsq(A, b.unsqueeze(1)).solution.squeeze(1)
    dres = float(torch.linalg.norm(A @ (torch.from_numpy(x).to(dev) - xl)) / torch.linalg.norm(b))
    assert dres <= 1e-8
