"""K4 pass time vs run length: average device time per launch over 10 / 30 / 90
back-to-back launches on a C3-sized A (power / clock effects of a sustained
stream).  usage: python tools/diag_pass_sustained.py [m] [n]"""
import ctypes as ct
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2506_03070_b200 as slq

m = int(sys.argv[1]) if len(sys.argv) > 1 else 4_000_000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
dev = torch.device("cuda", 0)
ld = (n + 1 + 3) // 4 * 4
Abuf = torch.empty(m, ld, device=dev, dtype=torch.float64)
for r in range(0, m, 500_000):
    Abuf[r:r + 500_000].normal_()
ctx = slq.Context(0)
A = slq.DeviceMatrix.wrap(Abuf.data_ptr(), m, n, ld, ctx=ctx, owner=Abuf)
out = np.zeros(8)
for reps in (10, 30, 90, 10):
    slq._capi.lib.slq_time_kernels(ctx.handle, A.handle, 4 * n, 8, 3, reps, out.ctypes.data_as(ct.POINTER(ct.c_double)))
    gb = (8.0 * m * n + 16.0 * m) / 1e9
    print(f"reps {reps:3d}: {out[0] * 1e3:.3f} ms per pass = {gb / out[0]:.0f} GB/s", flush=True)
