"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list by kernel: launches, total and mean time.
usage: python tools/launch_agg.py launches.csv [first-kernel-regex-of-the-last-solve]"""
import collections
import csv
import io
import re
import sys

txt = open(sys.argv[1]).read()
rows = list(csv.reader(io.StringIO(txt[txt.index('"ID"'):])))
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
L = []
for r in rows[1:]:
    if len(r) < len(h) or r[h.index("Metric Name")] != "gpu__time_duration.sum":
        continue
    t = float(r[vi].replace(",", ""))
    u = r[ui]
    t = t / 1e3 if u in ("us", "usecond") else t if u in ("ms", "msecond") else t / 1e6
    L.append((re.sub(r"\(.*", "", r[ki]).replace("(anonymous namespace)::", "")[-48:], t))
if len(sys.argv) > 2:
    starts = [i for i, (k, _) in enumerate(L) if re.search(sys.argv[2], k)]
    if starts:
        L = L[starts[-1]:]
agg = collections.OrderedDict()
for k, t in L:
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += t
tot = sum(v[1] for v in agg.values())
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:50s} n={n:5d} total={t:9.3f} ms mean={1e3 * t / n:9.1f} us")
print(f"total {tot:.3f} ms")
