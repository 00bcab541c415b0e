"""Per-iteration LSQR time with the fused cooperative K5 vs the three-kernel K5
(SLQ_NO_FUSED_K5=1, read once per process: run this script twice).
usage: python tools/diag_k5.py [m] [n] [T]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2506_03070_b200 as slq

m = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100
T = int(sys.argv[3]) if len(sys.argv) > 3 else 30
dev = torch.device("cuda", 0)
ld = (n + 1 + 3) // 4 * 4
g = torch.Generator(device=dev).manual_seed(0)
Abuf = torch.randn(m, ld, device=dev, dtype=torch.float64, generator=g)
Abuf[:, n + 1:] = 0
ctx = slq.Context(0)
s = torch.cuda.Stream()
ctx.set_stream(s.cuda_stream)
A = slq.DeviceMatrix.wrap(Abuf.data_ptr(), m, n, ld, ctx=ctx, owner=Abuf)
opts = slq.SolveOptions(eps=0.0, maxit=T)
for _ in range(3):
    slq.solve(A, 4 * n, 8, 3, opts, ctx=ctx)
res = [slq.solve(A, 4 * n, 8, 3, opts, ctx=ctx) for _ in range(10)]
tot = np.median([r[2]["total"] for r in res]) * 1e3
it = np.median([r[2]["lsqr_per_iteration"] for r in res]) * 1e6
x = res[-1][0]
print(f"m={m} n={n} T={T} fused={'SLQ_NO_FUSED_K5' not in os.environ}: solve {tot:.3f} ms, "
      f"lsqr {it:.1f} us/iteration, launches {res[-1][2]['kernel_launches']:.0f}, |x| {np.linalg.norm(x):.15e}",
      flush=True)
