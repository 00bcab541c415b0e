"""Stress / race check: repeat full solves at C3 (dense) and C4 (sparse) shapes
and require bit-identical solutions every time (every kernel on the path is
deterministic; a race in an mbarrier ring, a stage refill or a DSMEM exchange
would show up as a differing bit).  usage: python tools/stress_determinism.py [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2506_03070_b200 as slq

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
dev = torch.device("cuda", 0)
ctx = slq.Context(0)
# dense, C3 width at 1/4 of the rows
m, n = 1_000_000, 1000
ld = (n + 1 + 3) // 4 * 4
g = torch.Generator(device=dev).manual_seed(5)
Abuf = torch.randn(m, ld, device=dev, dtype=torch.float64, generator=g)
Abuf[:, n + 1:] = 0
A = slq.DeviceMatrix.wrap(Abuf.data_ptr(), m, n, ld, ctx=ctx, owner=Abuf)
ref = None
for r in range(reps):
    x, rep, _ = slq.solve(A, 4 * n, 8, 3, slq.SolveOptions(eps=0.0, maxit=20), ctx=ctx)
    if ref is None:
        ref = x.copy()
    assert np.array_equal(x, ref), f"dense solve {r} differs"
print(f"dense {m}x{n}: {reps} solves bit-identical", flush=True)
del A, Abuf
torch.cuda.empty_cache()
# sparse, C4 shape at 1/4 of the rows
ms, ns, k = 1 << 22, 2000, 50
S, _ = slq.SparseDeviceMatrix.create_csr(ms, ns, ms * k, with_b=True, ctx=ctx)
S.fill_random(k, 4, np.power(10.0, -6.0 * np.arange(ns) / (ns - 1)))
S.set_rhs(np.random.default_rng(1).uniform(-1, 1, ms))
ref = None
for r in range(reps):
    x, rep, _ = slq.solve(S, 4 * ns, 8, 3, slq.SolveOptions(eps=0.0, maxit=20), ctx=ctx)
    if ref is None:
        ref = x.copy()
    assert np.array_equal(x, ref), f"sparse solve {r} differs"
print(f"sparse {ms}x{ns}: {reps} solves bit-identical", flush=True)
