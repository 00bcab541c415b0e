#!/bin/bash
# slab gather pacing sweep on the final kernel: window rows x lag (C4)
mkdir -p gpurun_out
for kw in 65536 131072 262144 524288; do
  for lag in 1 2 4; do
    SLQ_K2S_KWIN=$kw SLQ_K2S_LAG=$lag timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv -k regex:"sparse_gather_slab" -c 1 python bench.py --config c4 --steps 1 --warmup 1 --no-cpu --no-e2e --iters 2 > gpurun_out/pace.csv 2>&1
    python - "$kw" "$lag" <<'PY'
import csv, io, sys
txt = open('gpurun_out/pace.csv').read()
i = txt.find('"ID"')
rows = list(csv.reader(io.StringIO(txt[i:]))) if i >= 0 else []
h = rows[0] if rows else []
vals = {}
for r in rows[1:]:
    if len(r) == len(h):
        vals[r[h.index('Metric Name')]] = (r[h.index('Metric Value')], r[h.index('Metric Unit')])
print('kwin', sys.argv[1], 'lag', sys.argv[2], vals)
PY
  done
done
