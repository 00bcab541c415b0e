"""Print the shared objects a profiler injected into this process (diagnostics for the QR-graph opt-out)."""
import torch

torch.zeros(1, device="cuda")
libs = set()
for line in open("/proc/self/maps"):
    path = line.split()[-1]
    if "/" in path and any(x in path.lower() for x in ("nsight", "ncu", "inject", "intercept", "nvperf", "cupti", "target")):
        libs.add(path)
print("INJECTED", sorted(libs))
