"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list.

usage: python tools/summarize_launches.py launches.csv "title" > profiles/<name>.txt
Groups launches by kernel; reports count, total, average and the share of the
library's (slq) kernels."""
import collections
import csv
import sys

path, title = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
h, data = rows[0], rows[1:]
ik, iv = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in data:
    k = r[ik].split("(")[0]
    k = k.replace("void ", "").replace("slq::(anonymous namespace)::", "").replace("slq::<unnamed>::", "")
    agg[k][0] += 1
    agg[k][1] += float(r[iv].replace(",", ""))
# library kernels = the __global__ functions defined in paper_2506_03070_b200/csrc
import glob
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
names = set()
for f in glob.glob(os.path.join(ROOT, "paper_2506_03070_b200", "csrc", "*.cu")):
    names.update(re.findall(r"__global__\s+void\s+(?:__launch_bounds__\([^)]*\)\s+)?(\w+)", open(f).read()))
ours = {k: v for k, v in agg.items() if re.sub(r"<.*", "", k).split("::")[-1] in names}
tot_all = sum(v[1] for v in agg.values()) / 1e6
tot = sum(v[1] for v in ours.values()) / 1e6
print(title)
print(f"ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialized launches)")
print(f"all kernels total {tot_all:.1f} ms; library kernels total {tot:.1f} ms")
for k, (c, t) in sorted(ours.items(), key=lambda x: -x[1][1]):
    print(f"{k[:44]:44s} launches={c:6d} total_ms={t / 1e6:10.2f} avg_us={t / c / 1e3:11.2f} share={t / 1e6 / tot:.3f}")
