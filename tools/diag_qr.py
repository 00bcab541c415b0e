"""QR-only driver for profiling the K3 kernels (4000 x 1000 by default)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2506_03070_b200 as slq
d = int(sys.argv[1]) if len(sys.argv) > 1 else 4000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
rng = np.random.default_rng(0)
Y = np.asfortranarray(rng.standard_normal((d, n)) @ np.diag(np.logspace(0, -6, n)))
for i in range(3):
    t = time.perf_counter()
    P = slq.build_preconditioner(Y)
    print(f"build_preconditioner {d}x{n}: host {1e3*(time.perf_counter()-t):.2f} ms, device build_time {1e3*P.build_time:.2f} ms")
