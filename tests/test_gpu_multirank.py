"""The multi-rank decomposition driven through the library's own per-rank
entry points, with N ranks sharing one B200: every rank is a thread with its
own context (own stream) and row block, and the collectives go through
host-side callbacks (slq_ctx_set_host_comm) instead of NCCL -- the same
per-rank sequence as the NCCL path (reduce of S[A_k b_k] partials, rank-0 QR /
R^-1 / x0, status / M / M^T / x0 broadcasts, one allreduce of n+1 doubles per
LSQR iteration), with the device work of all ranks running concurrently and
no rank's kernels waiting on another's (the ranks meet only in host barriers).
The collectives sum in rank order, identically on every rank, as
distsim.hpp's fixed-order tree_reduce does for its workers."""
import threading

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

slq = pytest.importorskip("paper_2506_03070_b200")
C = oracle.C()


class ThreadGroup:
    """In-process collectives among p rank threads (fixed rank order)."""

    def __init__(self, p):
        self.p = p
        self.bar = threading.Barrier(p, timeout=120)  # a mismatched collective sequence fails, not hangs
        self.slots = [None] * p
        self.calls = [0] * p

    def comm(self, r):
        g = self

        class Rank:
            def _sum(self, buf, root_only):
                g.calls[r] += 1
                g.slots[r] = buf.copy()
                g.bar.wait()
                if r == 0 or not root_only:
                    tot = g.slots[0].copy()
                    for k in range(1, g.p):
                        tot += g.slots[k]
                    buf[:] = tot
                g.bar.wait()

            def allreduce_sum(self, buf):
                self._sum(buf, False)

            def reduce_sum_root(self, buf):
                self._sum(buf, True)

            def broadcast_root(self, buf):
                g.calls[r] += 1
                if r == 0:
                    g.slots[0] = buf.copy()
                g.bar.wait()
                buf[:] = g.slots[0]
                g.bar.wait()

        return Rank()


def _run_ranks(p, body):
    group = ThreadGroup(p)
    out = [None] * p
    errs = [None] * p

    def worker(r):
        try:
            ctx = slq.Context(0)
            ctx.set_host_comm(group.comm(r), r, p)
            out[r] = body(r, ctx)
        except BaseException as e:  # noqa: BLE001 -- reported below
            # no barrier abort here: a rank that finished (even with an error)
            # has passed all its collectives; aborting could break a peer that
            # was released from the last barrier but not yet woken
            errs[r] = e

    ts = [threading.Thread(target=worker, args=(r,)) for r in range(p)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    return out, errs, group


def _problem(m, n, cond, seed):
    A = C.gen_dense(m, n, cond, seed)
    b, _ = C.gen_rhs(A, 0.5, seed + 1)
    return A, b


def _eta(A, b, x):
    r = b - A @ x
    return np.linalg.norm(A.T @ r) / (np.linalg.norm(A, 2) * np.linalg.norm(r))


@pytest.mark.parametrize("p", [2, 3, 5])
def test_multirank_solve_matches_single_rank(p):
    m, n, d, zeta, T = 24000, 40, 160, 8, 25
    A, b = _problem(m, n, 1e4, 7)
    part = slq.partition_rows(m, p)
    opts = slq.SolveOptions(eps=0.0, maxit=T)

    def body(r, ctx):
        r0, r1 = part.begin(r), part.end(r)
        dm = slq.DeviceMatrix.from_numpy(A[r0:r1], b[r0:r1], row_begin=r0, ctx=ctx)
        return slq.solve(dm, d, zeta, 11, opts, ctx=ctx)

    out, errs, group = _run_ranks(p, body)
    assert not any(errs), errs
    xs = [o[0] for o in out]
    for x in xs[1:]:
        assert np.array_equal(x, xs[0])  # replicated n-vector work: identical bits on every rank
    for x, rep, ph in out:
        assert rep.iterations == T
        assert rep.sync_count - rep.init_reductions == T  # one allreduce per iteration
        assert ph["nccl_calls"] > 0
    # collectives per rank: reduce + status/M/M^T/x0 broadcasts + init allreduce + T + no-op tail of the last batch
    assert len(set(group.calls)) == 1 and group.calls[0] >= 1 + 4 + 1 + T
    # against one rank: the sketch partials are summed in another order, which
    # moves x by ~1e-8 at cond 1e4 -- compared in residual / backward-error space
    x1, rep1, _ = slq.solve(A, d, zeta, 11, opts, b=b)
    assert np.linalg.norm(A @ (xs[0] - x1)) <= 1e-10 * np.linalg.norm(b)
    assert _eta(A, b, xs[0]) <= max(2 * _eta(A, b, x1), 1e-14)
    # the reference's distributed sketch (distsim.hpp:383-396) + serial pipeline, same seed
    Yr, Sbr = oracle.REF().dist_sketch_apply(d, zeta, 11, A, b, p) if oracle.ref_available() else C.sketch_apply(
        d, zeta, 11, A, b)
    M, Q = C.build_preconditioner(Yr)
    xo, _ = C.lsqr(A, M, b, C.initial_guess(M, Q, Sbr), eps=0.0, maxit=T, one_sync=True)
    assert np.linalg.norm(A @ (xs[0] - xo)) <= 1e-10 * np.linalg.norm(b)
    assert _eta(A, b, xs[0]) <= max(2 * _eta(A, b, xo), 1e-14)


def test_multirank_gradient_descent():
    p, m, n, d = 3, 9000, 30, 120
    A, b = _problem(m, n, 1e2, 21)
    Y, Sb = C.sketch_apply(d, 8, 9, A, b)
    M, Q = C.build_preconditioner(Y)
    x0 = C.initial_guess(M, Q, Sb)
    prm = slq.hbm_params(float(np.sqrt(n / d)))
    opts = slq.SolveOptions(eps=0.0, maxit=15)
    part = slq.partition_rows(m, p)

    def body(r, ctx):
        r0, r1 = part.begin(r), part.end(r)
        dm = slq.DeviceMatrix.from_numpy(A[r0:r1], b[r0:r1], row_begin=r0, ctx=ctx)
        return slq.gradient_descent_hbm(dm, M, None, x0, prm, opts, ctx=ctx)

    out, errs, _ = _run_ranks(p, body)
    assert not any(errs), errs
    assert all(np.array_equal(o[0], out[0][0]) for o in out)
    xs, rs = slq.gradient_descent_hbm(A, M, b, x0, prm, opts)
    assert np.linalg.norm(out[0][0] - xs) <= 1e-10 * np.linalg.norm(xs)
    assert out[0][1].sync_count == 15


def test_multirank_rank0_failure_reaches_every_rank():
    """A rank-deficient sketch on rank 0 (duplicate columns): every rank raises
    RankDeficient from the broadcast status word -- no rank hangs."""
    p, m, n, d = 2, 4000, 12, 48
    rng = np.random.default_rng(3)
    A = rng.standard_normal((m, n))
    A[:, 5] = A[:, 4]
    b = rng.standard_normal(m)
    part = slq.partition_rows(m, p)

    def body(r, ctx):
        r0, r1 = part.begin(r), part.end(r)
        dm = slq.DeviceMatrix.from_numpy(np.asfortranarray(A[r0:r1]), b[r0:r1], row_begin=r0, ctx=ctx)
        return slq.solve(dm, d, 4, 1, slq.SolveOptions(eps=0.0, maxit=10), ctx=ctx)

    out, errs, _ = _run_ranks(p, body)
    assert all(isinstance(e, slq.RankDeficient) for e in errs), errs
