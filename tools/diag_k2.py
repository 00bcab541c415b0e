"""K2 diagnostics: fast-mode sketch apply S.[A b] by kernel family.
    K2d  DMMA tile gather (default),
    reg  register gather (SLQ_ROW_GATHER=1)
Times generate+apply and generate alone with slq_time_kernels (CUDA events on
the library stream; apply = difference), and checks each against exact mode
at a reduced m.
usage: python tools/diag_k2.py [m] [n] [d] [zeta] [families, comma-separated]"""
import ctypes as ct
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2506_03070_b200 as slq
from paper_2506_03070_b200 import _capi as CA

m = int(sys.argv[1]) if len(sys.argv) > 1 else 4_000_000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
d = int(sys.argv[3]) if len(sys.argv) > 3 else 4 * n
zeta = int(sys.argv[4]) if len(sys.argv) > 4 else 8
fams = (sys.argv[5] if len(sys.argv) > 5 else "K2d,reg").split(",")
ENV = {"K2d": {}, "reg": {"SLQ_ROW_GATHER": "1"}}
dev = torch.device("cuda", 0)
ld = (n + 1 + 3) // 4 * 4
g = torch.Generator(device=dev).manual_seed(0)
Abuf = torch.randn(m, ld, device=dev, dtype=torch.float64, generator=g)
Abuf[:, n + 1:] = 0
ctx = slq.Context(0)
s = torch.cuda.Stream()
ctx.set_stream(s.cuda_stream)
A = slq.DeviceMatrix.wrap(Abuf.data_ptr(), m, n, ld, ctx=ctx, owner=Abuf)


def setenv(f):
    for k in ("SLQ_ROW_GATHER",):
        os.environ.pop(k, None)
    os.environ.update(ENV[f])


def timed(f, reps=3):
    setenv(f)
    best = 1e9
    for _ in range(reps):
        out = np.zeros(4)
        st = CA.lib.slq_time_kernels(ctx.handle, A.handle, d, zeta, 7, 1, out.ctypes.data_as(CA.dp))
        assert st == 0, CA.lib.slq_last_error()
        best = min(best, out[1] - out[2])
    return best


# parity at a reduced m (exact mode = the reference's serial order)
ms = min(m, 300_000)
Asub = slq.DeviceMatrix.wrap(Abuf.data_ptr(), ms, n, ld, ctx=ctx, owner=Abuf)
Ye, Sbe = Asub.sketch(d, zeta, 7, exact=True)
sc = np.abs(Ye).max()
res = {}
for f in fams:
    setenv(f)
    Yf, Sbf = Asub.sketch(d, zeta, 7, exact=False)
    rel = max(np.abs(Yf - Ye).max(), np.abs(Sbf - Sbe).max()) / sc
    t = timed(f)
    res[f] = (t, rel)
gb = 8.0 * m * ld / 1e9
print(f"m={m} n={n} d={d} zeta={zeta}: " + "  ".join(
    f"{f} {t * 1e3:.2f} ms ({gb / t:.0f} GB/s of A, rel diff {rel:.1e})" for f, (t, rel) in res.items()), flush=True)
