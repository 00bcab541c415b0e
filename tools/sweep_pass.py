"""K4 dense pass efficiency across row lengths: average device time of the
fused pass (slq_time_kernels, live-data form) for A of ~4 GB at n in a sweep,
as GB/s of the algorithmic bytes (8 m n + 16 m).
usage: python tools/sweep_pass.py [gb]"""
import ctypes as ct
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2506_03070_b200 as slq

gb = float(sys.argv[1]) if len(sys.argv) > 1 else 4.0
dev = torch.device("cuda", 0)
ctx = slq.Context(0)
NS = [int(v) for v in os.environ.get("NS", "20,50,100,200,300,500,700,1000,1500,2000,3000,4000").split(",")]
for n in NS:
    ld = (n + 1 + 3) // 4 * 4
    m = int(gb * 1e9 / (8 * ld))
    Abuf = torch.randn(m, ld, device=dev, dtype=torch.float64)
    Abuf[:, n + 1:] = 0
    A = slq.DeviceMatrix.wrap(Abuf.data_ptr(), m, n, ld, ctx=ctx, owner=Abuf)
    # one short solve so the pass runs on live vectors, then the pass timing
    slq.solve(A, 4 * n, 8, 3, slq.SolveOptions(eps=0.0, maxit=3), ctx=ctx)
    out = np.zeros(4)
    assert slq._capi.lib.slq_time_kernels(ctx.handle, A.handle, 4 * n, 8, 3, 10, out.ctypes.data_as(ct.POINTER(ct.c_double))) == 0
    t = out[0]
    print(f"n={n:5d} m={m:9d}: pass {t * 1e3:.3f} ms  {(8.0 * m * n + 16.0 * m) / t / 1e9:.0f} GB/s", flush=True)
    del A, Abuf
    torch.cuda.empty_cache()
