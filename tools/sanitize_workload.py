"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck) and for
the library's guard-band mode (SLQ_GUARD=1: prints guards_corrupted=N at the end):
every hot kernel family at shapes that exercise its synchronisation protocol
  * K1 generator (warp path + generic path for zeta > 32),
  * K2d DMMA tile gather (stage refill by the last warp, 2-3 stage ring) and
    the exact-order register gather (TMA double buffer),
  * K3 cluster QR panel (DSMEM st.async pushes, several CTAs per cluster),
    narrow / wide updates, blocked inverse,
  * K4 fused pass (producer warp + mbarrier ring) and K5, one-sync LSQR,
  * K2s / K4s sparse path, gradient family.
usage: compute-sanitizer --tool racecheck python tools/sanitize_workload.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2506_03070_b200 as slq

rng = np.random.default_rng(0)
# K1
slq.generate_sparse_sign(400, 3000, 8, 3)
slq.generate_sparse_sign(100, 500, 40, 3)
# K2d (fast) + register gather (exact), several row blocks and chunks
m, n, d, zeta = 6000, 20, 1100, 8
A = np.asfortranarray(rng.standard_normal((m, n)))
b = rng.standard_normal(m)
dm = slq.DeviceMatrix.from_numpy(A, b)
dm.sketch(d, zeta, 5, exact=False)
dm.sketch(d, zeta, 5, exact=True)
# K3: cluster panel over several CTAs (tall Y), inverse
Y = np.asfortranarray(rng.standard_normal((3000, 70)))
qr = slq.householder_qr(Y)
slq.tri_inverse(qr.R)
# K4/K5: full pipeline, one-sync, graph batches
x, rep, _ = slq.solve(A, 4 * n, zeta, 7, slq.SolveOptions(eps=0.0, maxit=10), b=b)
# sparse path
cols = [np.unique(rng.integers(0, m, 30)) for _ in range(n)]
rr = np.concatenate(cols)
colptr = np.concatenate([[0], np.cumsum([len(c) for c in cols])]).astype(np.int64)
S = slq.CscMatrix(m, n, rng.standard_normal(rr.size), rr.astype(np.int64), colptr)
slq.solve(S, 4 * n, zeta, 7, slq.SolveOptions(eps=0.0, maxit=5), b=b)
# gradient family
Ys, Sbs = dm.sketch(4 * n, zeta, 9)
P, x0 = slq.build_preconditioner(Ys, Sb=Sbs)
slq.gradient_descent_hbm(A, P, b, x0, slq.hbm_params(0.5), slq.SolveOptions(eps=0.0, maxit=5))
# round-2 paths: two-pass sparse operator over several 16384-row blocks (+ the
# transposed-copy build), wide-row LSQR pass (n > 2046), TSQR (d > 12400)
m2, n2 = 40_000, 90
cols2 = [np.unique(rng.integers(0, m2, 700)) for _ in range(n2)]
rr2 = np.concatenate(cols2)
cp2 = np.concatenate([[0], np.cumsum([len(c) for c in cols2])]).astype(np.int64)
S2 = slq.CscMatrix(m2, n2, rng.standard_normal(rr2.size), rr2.astype(np.int64), cp2)
slq.solve(S2, 4 * n2, zeta, 7, slq.SolveOptions(eps=0.0, maxit=4), b=rng.standard_normal(m2))
mw, nw = 3000, 2100
Aw = np.asfortranarray(rng.standard_normal((mw, nw)))
slq.solve(Aw, nw + 100, zeta, 7, slq.SolveOptions(eps=0.0, maxit=2), b=rng.standard_normal(mw))
At = np.asfortranarray(rng.standard_normal((20000, 24)))
slq.solve(At, 13000, 4, 7, slq.SolveOptions(eps=0.0, maxit=2), b=rng.standard_normal(20000))
print("sanitize workload done", rep.iterations)
if os.environ.get("SLQ_GUARD"):
    import ctypes as ct

    bad = ct.c_int64(-1)
    assert slq._capi.lib.slq_debug_check_guards(ct.byref(bad)) == 0
    print(f"guards_corrupted={bad.value}")
