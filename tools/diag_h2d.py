"""H2D bandwidth diagnostics for the e2e path: plain pinned copies, 2D
column-block copies (the slq_dense_upload pattern) and slq_dense_upload."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2506_03070_b200 as slq

dev = torch.device("cuda", 0)
GB = 1 << 30
h = torch.empty(4 * GB // 8, dtype=torch.float64, pin_memory=True)
h.fill_(1.0)
d = torch.empty_like(h, device=dev)
for name, nbytes in (("1 GB", GB), ("4 GB", 4 * GB)):
    n = nbytes // 8
    torch.cuda.synchronize()
    for _ in range(2):
        t = time.perf_counter()
        d[:n].copy_(h[:n], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    print(f"pinned 1D H2D {name}: {nbytes / dt / 1e9:.1f} GB/s", flush=True)
# D2H for reference
t = time.perf_counter(); h[: GB // 8].copy_(d[: GB // 8], non_blocking=True); torch.cuda.synchronize()
print(f"pinned 1D D2H 1 GB: {GB / (time.perf_counter() - t) / 1e9:.1f} GB/s", flush=True)
# slq_dense_upload of a 4 GB column-major block (m = 500k, n = 1000)
m, n = 500_000, 1000
Ah = torch.empty((n, m), dtype=torch.float64, pin_memory=True)
Ah.normal_()
bh = torch.empty(m, dtype=torch.float64, pin_memory=True)
ctx = slq.Context(0)
import ctypes as ct
from paper_2506_03070_b200 import _capi as C
for _ in range(3):
    out = ct.c_void_p()
    torch.cuda.synchronize()
    t = time.perf_counter()
    rc = C.lib.slq_dense_upload(ctx.handle, ct.cast(Ah.data_ptr(), C.dp), m, n, m, ct.cast(bh.data_ptr(), C.dp), 0,
                                ct.byref(out))
    dt = time.perf_counter() - t
    assert rc == 0, C.lib.slq_last_error()
    C.lib.slq_dense_free(out)
    print(f"slq_dense_upload 4 GB: {dt * 1e3:.1f} ms = {8 * m * (n + 1) / dt / 1e9:.1f} GB/s", flush=True)
