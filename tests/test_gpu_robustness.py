"""GPU tests for boundary robustness: the opt-in backward-error stop, the
on_bidiag hook on breakdown, missing right-hand sides and non-finite padding
in wrapped caller storage."""
import ctypes as ct

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

slq = pytest.importorskip("paper_2506_03070_b200")
C = oracle.C()


def _eta(A, b, x):
    r = b - A @ x
    return np.linalg.norm(A.T @ r) / (np.linalg.norm(A, 2) * np.linalg.norm(r))


def test_backward_tol_stops_early_and_is_confirmed():
    # inconsistent system: the reference rule phi_bar <= eps beta_1 never fires
    # (SURVEY 0.1); the opt-in backward-error rule stops once eta <= tol.
    m, n, d, zeta = 30000, 60, 240, 8
    A = C.gen_dense(m, n, 1e4, 11)
    b, _ = C.gen_rhs(A, 0.5, 12)
    anorm = np.linalg.norm(A, 2)
    full, rep_full, _ = slq.solve(A, d, zeta, 3, slq.SolveOptions(eps=1e-10, maxit=80), b=b)
    assert rep_full.termination == slq.Termination.MaxIter and rep_full.iterations == 80
    for tol in (1e-6, 1e-10):
        x, rep, _ = slq.solve(A, d, zeta, 3, slq.SolveOptions(eps=1e-10, maxit=80, backward_tol=tol,
                                                              a_norm_est=anorm), b=b)
        assert rep.termination == slq.Termination.Tolerance, (tol, rep)
        assert rep.iterations < 80
        assert 0 <= rep.backward_error <= tol
        assert _eta(A, b, x) <= 1.01 * tol
        # the first iterates agree with the full run (same recurrence)
        assert np.allclose(rep.residual_estimate, rep_full.residual_estimate[: rep.iterations], rtol=1e-12)


def test_backward_tol_unreachable_runs_to_maxit():
    m, n, d, zeta = 8000, 20, 80, 8
    A = C.gen_dense(m, n, 1e2, 5)
    b, _ = C.gen_rhs(A, 0.5, 6)
    x, rep, _ = slq.solve(A, d, zeta, 3, slq.SolveOptions(eps=0.0, maxit=15, backward_tol=1e-30, a_norm_est=1.0), b=b)
    assert rep.iterations == 15 and rep.termination == slq.Termination.MaxIter


def test_on_bidiag_not_called_on_breakdown():
    # lsqr.hpp:120-141: a breakdown returns before the hook
    calls = []
    x, rep = slq.lsqr(np.eye(4), np.eye(4), np.array([2.0, 0, 0, 0]), np.zeros(4),
                      slq.SolveOptions(eps=0.0, maxit=5, on_bidiag=lambda t, un, vn: calls.append((t, un, vn))))
    assert rep.termination == slq.Termination.Breakdown
    assert all(np.isfinite(c[1]) and np.isfinite(c[2]) for c in calls)
    assert len(calls) == 0


def test_solve_without_rhs_is_an_error():
    from paper_2506_03070_b200 import _capi as CA

    A = np.asfortranarray(np.random.default_rng(0).standard_normal((500, 6)))
    dm = slq.DeviceMatrix.from_numpy(A)  # no b
    x = np.zeros(6)
    st = CA.lib.slq_solve(dm.ctx.handle, dm.handle, 24, 4, 1, None, x.ctypes.data_as(CA.dp), None, None, None)
    assert st == 10  # SLQ_INVALID_ARG
    assert b"right-hand side" in CA.lib.slq_last_error()


def test_wrap_zeroes_nonfinite_padding():
    import torch

    m, n = 3000, 5
    ld = slq.DeviceMatrix.ld_for(n)
    assert ld > n + 1
    rng = np.random.default_rng(3)
    A = rng.standard_normal((m, n))
    b = rng.standard_normal(m)
    buf = torch.full((m, ld), float("nan"), dtype=torch.float64, device="cuda")
    buf[:, :n] = torch.from_numpy(A)
    buf[:, n] = torch.from_numpy(b)
    dm = slq.DeviceMatrix.wrap(buf.data_ptr(), m, n, ld, owner=buf)
    x, rep, _ = slq.solve(dm, 24, 4, 7, slq.SolveOptions(eps=0.0, maxit=10))
    assert np.all(np.isfinite(x))
    xr, _, _ = slq.solve(np.asfortranarray(A), 24, 4, 7, slq.SolveOptions(eps=0.0, maxit=10), b=b)
    assert np.linalg.norm(x - xr) <= 1e-12 * np.linalg.norm(xr)


def test_solve_on_legacy_and_user_streams():
    """The same solve on a context bound to the legacy default stream (which
    cannot be captured: no CUDA graphs there), on a caller's stream and on the
    library's own stream, three times each (first use, graph capture, graph
    replay): bit-identical solutions."""
    import torch

    m, n, d, zeta = 20000, 70, 280, 8
    A = C.gen_dense(m, n, 1e3, 5)
    b, _ = C.gen_rhs(A, 0.5, 6)
    opts = slq.SolveOptions(eps=0.0, maxit=12)
    dm0 = slq.DeviceMatrix.from_numpy(A, b)
    ref, _, _ = slq.solve(dm0, d, zeta, 3, opts)
    dm0.free()
    user = torch.cuda.Stream()
    for ptr in (0, user.cuda_stream, None):
        ctx = slq.Context(0)
        if ptr is not None:
            ctx.set_stream(ptr)
        dm = slq.DeviceMatrix.from_numpy(A, b, ctx=ctx)
        for _ in range(3):
            x, rep, _ = slq.solve(dm, d, zeta, 3, opts, ctx=ctx)
            assert rep.iterations == 12
            assert np.array_equal(x, ref)
        dm.free()
