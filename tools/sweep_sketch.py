"""Config C5: sketch-only sweep -- K1 generation and K2 S*[A b]
throughput vs d/n in {2,4,8} and zeta in {2,4,8,16}, n = 500, device-resident A.

usage: python tools/sweep_sketch.py [log2_m ...]   (default 20 22 24)
Prints one JSON line per (m, d, zeta): K1 seconds / Gnnz/s, K2 seconds / GB/s of A."""
import ctypes as ct
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2506_03070_b200 as slq

n = 500
dev = torch.device("cuda", 0)
ctx = slq.Context(0)
s = torch.cuda.Stream()
ctx.set_stream(s.cuda_stream)
for lm in [int(a) for a in sys.argv[1:]] or [20, 22, 24]:
    m = 1 << lm
    ld = (n + 1 + 3) // 4 * 4
    A = torch.empty((m, ld), dtype=torch.float64, device=dev)
    A.normal_()
    A[:, n + 1:] = 0
    dm = slq.DeviceMatrix.wrap(A.data_ptr(), m, n, ld, ctx=ctx, owner=A)
    for dfac in (2, 4, 8):
        d = dfac * n
        for zeta in (2, 4, 8, 16):
            out = np.zeros(4)
            for _ in range(2):  # warm, then measure
                rc = slq._capi.lib.slq_time_kernels(ctx.handle, dm.handle, d, zeta, 3, 1,
                                                    out.ctypes.data_as(ct.POINTER(ct.c_double)))
                assert rc == 0, slq._capi.lib.slq_last_error()
            k1, k12 = out[2], out[1]
            k2 = k12 - k1
            print(json.dumps({"m": m, "n": n, "d": d, "zeta": zeta, "k1_s": k1, "k1_gnnz_s": m * zeta / k1 / 1e9,
                              "k2_s": k2, "k2_gbs_of_A": 8.0 * m * ld / k2 / 1e9,
                              "k2_gfma_s": m * zeta * (n + 1) / k2 / 1e9}), flush=True)
    del dm, A
    torch.cuda.empty_cache()
