"""K2 diagnostics: the DMMA tile gather (fast-mode default) vs the register
gather (SLQ_ROW_GATHER=1) and the exact serial-order gather.
usage: python tools/diag_k2d.py [m] [n] [d] [zeta]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2506_03070_b200 as slq

m = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
d = int(sys.argv[3]) if len(sys.argv) > 3 else 4 * n
zeta = int(sys.argv[4]) if len(sys.argv) > 4 else 8
dev = torch.device("cuda", 0)
ld = (n + 1 + 3) // 4 * 4
g = torch.Generator(device=dev).manual_seed(0)
Abuf = torch.randn(m, ld, device=dev, dtype=torch.float64, generator=g)
Abuf[:, n + 1:] = 0
ctx = slq.Context(0)
s = torch.cuda.Stream()
ctx.set_stream(s.cuda_stream)
A = slq.DeviceMatrix.wrap(Abuf.data_ptr(), m, n, ld, ctx=ctx, owner=Abuf)


def run(exact, row, reps=3):
    if row:
        os.environ["SLQ_ROW_GATHER"] = "1"
    else:
        os.environ.pop("SLQ_ROW_GATHER", None)
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        Y, Sb = A.sketch(d, zeta, 7, exact=exact)
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return np.column_stack([Y, Sb]), min(ts)


Ye, te = run(True, True)
Yr, tr = run(False, True)
Yd, td = run(False, False)
sc = np.abs(Ye).max()
print(f"m={m} n={n} d={d} zeta={zeta}: exact {te:.2f} ms  row(fast) {tr:.2f} ms  dmma(fast) {td:.2f} ms  "
      f"rel diff row {np.abs(Yr - Ye).max() / sc:.2e}  dmma {np.abs(Yd - Ye).max() / sc:.2e}", flush=True)
