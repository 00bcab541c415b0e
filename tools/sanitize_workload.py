"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
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
print("sanitize workload done", rep.iterations)
