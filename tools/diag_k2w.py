"""K2 diagnostics: the lane-column warp gather (K2w, SLQ_K2W=1, SLQ_KW_NW=8|16)
against the DMMA tile gather (K2d) and the exact register gather; checks K2w
exact mode bit for bit against the exact register gather and fast mode
against it within 1e-12 max|Y|.
usage: python tools/diag_k2w.py [m] [n] [d] [zeta] [config (profile one)]"""
import ctypes as ct
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
A = slq.DeviceMatrix.wrap(Abuf.data_ptr(), m, n, ld, ctx=ctx, owner=Abuf)
CFG = {"dmma": {}, "row": {"SLQ_ROW_GATHER": "1"}, "k2w16": {"SLQ_K2W": "1", "SLQ_KW_NW": "16"}, "k2w24": {"SLQ_K2W": "1", "SLQ_KW_NW": "24"},
       "k2w8": {"SLQ_K2W": "1", "SLQ_KW_NW": "8"}}


def setenv(cfg):
    for k in ("SLQ_ROW_GATHER", "SLQ_K2W", "SLQ_KW_NW"):
        os.environ.pop(k, None)
    os.environ.update(CFG[cfg])


def timed(cfg, reps=3):
    setenv(cfg)
    out = np.zeros(4)
    best = 1e9
    for _ in range(reps):
        rc = slq._capi.lib.slq_time_kernels(ctx.handle, A.handle, d, zeta, 7, 1, out.ctypes.data_as(ct.POINTER(ct.c_double)))
        assert rc == 0, slq._capi.lib.slq_last_error()
        best = min(best, out[1] - out[2])
    return best * 1e3


def sketch(cfg, exact):
    setenv(cfg)
    Y, Sb = A.sketch(d, zeta, 7, exact=exact)
    return np.column_stack([Y, Sb])


if len(sys.argv) > 5:  # profile one configuration: one timed call
    print(sys.argv[5], timed(sys.argv[5], reps=1))
    sys.exit(0)
res = {}
Ye = sketch("row", True)
sc = np.abs(Ye).max()
for cfg in ("k2w16", "k2w24"):
    Yx = sketch(cfg, True)
    Yf = sketch(cfg, False)
    res[cfg + "_exact_bitwise"] = bool(np.array_equal(Yx, Ye))
    res[cfg + "_fast_rel"] = float(np.abs(Yf - Ye).max() / sc)
res["dmma_fast_rel"] = float(np.abs(sketch("dmma", False) - Ye).max() / sc)
for cfg in ("dmma", "k2w16", "k2w24", "k2w8"):
    res[cfg + "_ms"] = timed(cfg)
print(f"m={m} n={n} d={d} zeta={zeta}", {k: (round(v, 3) if isinstance(v, float) and v > 1e-6 else v) for k, v in res.items()},
      flush=True)


def timed_host(cfg, exact, reps=3):
    best = 1e9
    for _ in range(reps):
        setenv(cfg)
        torch.cuda.synchronize()
        import time
        t = time.perf_counter()
        A.sketch(d, zeta, 7, exact=exact)
        best = min(best, time.perf_counter() - t)
    return best * 1e3


print("exact mode, host-timed incl. 32 MB D2H:", {c: round(timed_host(c, True), 2) for c in ("row", "k2w16")}, flush=True)
