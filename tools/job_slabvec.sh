#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sparse.py -x -q > gpurun_out/sv_tests.log 2>&1; echo "tests rc $?"; tail -1 gpurun_out/sv_tests.log
timeout 300 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/sv.jsonl 2>gpurun_out/sv.err
python -c "
import json; d=json.loads(open('gpurun_out/sv.jsonl').read().strip().splitlines()[-1]); p=d['phases_s']; print(round(d['value']*1e3,2), 'apply', round(p['apply']*1e3,2), d['clocks']['reasons'])"
timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,dram__bytes_read.sum --clock-control none --csv -k regex:"slab" python bench.py --config c4 --steps 1 --warmup 1 --no-cpu --no-e2e --iters 2 > gpurun_out/sv_launch.csv 2>&1
grep -v "^==" gpurun_out/sv_launch.csv | grep -i "slab" | head -6 | awk -F'","' '{print $5, $13, $14, $15}' | cut -c1-200
