"""K2s (sparse S.[A b]) timing on a C4-shaped CSR for several k-range launch
counts (SLQ_K2S_CHUNKS); host-timed, includes the 128 MB D2H of Y.
usage: [CHUNKS=1,64,150] python tools/diag_k2s.py [m] [n] [nnz_per_row]"""
import os
import sys
import time

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
ref = None
for ch in os.environ.get("CHUNKS", "1,64,150").split(","):
    os.environ["SLQ_K2S_CHUNKS"] = ch
    best = 1e9
    for _ in range(3):
        t = time.perf_counter()
        Y, Sb = A.sketch(4 * n, 8, 3)
        best = min(best, time.perf_counter() - t)
    same = ref is None or (np.array_equal(Y, ref[0]) and np.array_equal(Sb, ref[1]))
    if ref is None:
        ref = (Y, Sb)
    print(f"K2s m={m} n={n} chunks={ch}: {best * 1e3:.1f} ms (bitwise equal to chunks=first: {same})", flush=True)
