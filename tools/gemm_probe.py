import torch, time
dev = torch.device("cuda")
for rows, nc in [(8000, 1936), (4000, 968), (8000, 1000)]:
    V = torch.randn(rows, 32, dtype=torch.float64, device=dev)
    C = torch.randn(nc, rows, dtype=torch.float64, device=dev).t()  # column-major rows x nc
    W2 = torch.randn(32, nc, dtype=torch.float64, device=dev)
    for f, name in [(lambda: V.t() @ C, "W=VtC"), (lambda: C.sub_(V @ W2), "C-=VW2"), (lambda: torch.addmm(C, V, W2, alpha=-1.0, out=C), "addmm")]:
        for _ in range(3): f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): f()
        e1.record(); torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 20 * 1e3
        print(f"rows={rows} nc={nc} {name}: {t:.1f} us  {2*rows*nc*32/t/1e6:.1f} TF/s", flush=True)
