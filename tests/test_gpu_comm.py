"""The NCCL code path on one GPU: a single-rank communicator drives every
collective of the multi-GPU solve (ncclReduce of S[A b], status / M / x0
broadcasts, one ncclAllReduce of n+1 doubles per LSQR iteration, captured in
the iteration graph) and of the gradient family.  With one rank the
collectives are identities, so results must equal the communicator-free run
bit for bit, while the counters show the collectives were issued."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

slq = pytest.importorskip("paper_2506_03070_b200")
C = oracle.C()


def _problem(m=20000, n=40, seed=3):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((m, n)) @ np.diag(np.logspace(0, -4, n))
    b = rng.standard_normal(m)
    return A, b


def test_single_rank_nccl_solve_matches(monkeypatch):
    monkeypatch.setenv("SLQ_FORCE_NCCL", "1")
    A, b = _problem()
    d, zeta, T = 160, 8, 25
    opts = slq.SolveOptions(eps=0.0, maxit=T)
    ref_ctx = slq.Context(0)
    x0, rep0, ph0 = slq.solve(slq.DeviceMatrix.from_numpy(A, b, ctx=ref_ctx), d, zeta, 7, opts, ctx=ref_ctx)
    ctx = slq.Context(0)
    ctx.init_comm(slq.Context.unique_id(), 0, 1)
    x1, rep1, ph1 = slq.solve(slq.DeviceMatrix.from_numpy(A, b, ctx=ctx), d, zeta, 7, opts, ctx=ctx)
    assert np.array_equal(x0, x1)
    assert rep1.iterations == rep0.iterations == T
    assert ph0["nccl_calls"] == 0 and ph1["nccl_calls"] > 0
    # one allreduce per LSQR iteration (+ the init pass), as dist_rmatvec_and_norm (distsim.hpp:312-331)
    assert rep1.sync_count - rep1.init_reductions == T
    assert rep0.sync_count == 0


def test_single_rank_nccl_gradient_matches(monkeypatch):
    monkeypatch.setenv("SLQ_FORCE_NCCL", "1")
    A, b = _problem(8000, 30, 5)
    d = 120
    Y, Sb = C.sketch_apply(d, 8, 9, A, b)
    M, Q = C.build_preconditioner(Y)
    x0 = C.initial_guess(M, Q, Sb)
    prm = slq.hbm_params(float(np.sqrt(30 / d)))
    opts = slq.SolveOptions(eps=0.0, maxit=20)
    c0 = slq.Context(0)
    xa, ra = slq.gradient_descent_hbm(slq.DeviceMatrix.from_numpy(A, b, ctx=c0), M, None, x0, prm, opts, ctx=c0)
    c1 = slq.Context(0)
    c1.init_comm(slq.Context.unique_id(), 0, 1)
    xb, rb = slq.gradient_descent_hbm(slq.DeviceMatrix.from_numpy(A, b, ctx=c1), M, None, x0, prm, opts, ctx=c1)
    assert np.array_equal(xa, xb) and rb.iterations == 20
    assert rb.sync_count == 20 and ra.sync_count == 0
