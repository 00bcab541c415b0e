"""Diagnostics: host vs device time of repeated device-resident solves."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("SLQ_TRACE", "1")
import torch
import bench
import paper_2506_03070_b200 as slq

m = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
n, d, zeta = 1000, 4000, 8
dev = torch.device("cuda", 0)
Abuf, ld, _ = bench.make_problem(torch, m, n, 1e8, 0.5, 0, m, dev)
ctx = slq.Context(0)
s = torch.cuda.Stream()
ctx.set_stream(s.cuda_stream)
A = slq.DeviceMatrix.wrap(Abuf.data_ptr(), m, n, ld, ctx=ctx, owner=Abuf)
for i in range(4):
    t = time.perf_counter()
    x, rep, ph = slq.solve(A, d, zeta, 3, slq.SolveOptions(eps=0.0, maxit=30), ctx=ctx)
    print(f"solve {i}: host {1e3*(time.perf_counter()-t):.1f} ms, device total {1e3*ph['total']:.1f} ms, "
          f"apply {1e3*ph['apply']:.1f} qr {1e3*ph['qr']:.1f} lsqr {1e3*ph['lsqr']:.1f}", file=sys.stderr, flush=True)
