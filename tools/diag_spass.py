"""K4s timing: average device time of the sparse LSQR pass (slq_time_sparse_pass)
on a C4-shaped synthetic CSR.  usage: [GEOMS=0,1,2] python tools/diag_spass.py [m] [n] [nnz_per_row]"""
import ctypes as ct
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2506_03070_b200 as slq

m = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
k = int(sys.argv[3]) if len(sys.argv) > 3 else 50
ctx = slq.Context(0)
A, _ = slq.SparseDeviceMatrix.create_csr(m, n, m * k, with_b=True, ctx=ctx)
A.fill_random(k, 4, np.power(10.0, -6.0 * np.arange(n) / (n - 1)))
A.set_rhs(np.ones(m))
A.prepare()
t = ct.c_double(0.0)
gb = (12.0 * m * k + 8.0 * (m + 1) + 16.0 * m) / 1e9
for geom in os.environ.get("GEOMS", "0").split(","):
    os.environ["SLQ_UPASS_GEOM"] = geom
    for _ in range(2):
        assert slq._capi.lib.slq_time_sparse_pass(ctx.handle, A.handle, 10, ct.byref(t)) == 0
    print(f"K4s m={m} n={n} nnz/row={k} upass geometry {geom}: {t.value * 1e3:.3f} ms  {gb / t.value:.0f} GB/s "
          f"(algorithmic)", flush=True)
