#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sparse.py -x -q -k "apply" > gpurun_out/k2s_tests.log 2>&1; echo "tests rc $?"
tail -2 gpurun_out/k2s_tests.log
run() {  # tag, env...
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/k2s_$tag.jsonl 2>gpurun_out/k2s_$tag.err
  python -c "
import json; d=json.loads(open('gpurun_out/k2s_$tag.jsonl').read().strip().splitlines()[-1]); print('$tag', round(d['value'],4), 'apply', round(d['phases_s']['apply']*1e3,2), 'ms', d['clocks']['reasons'])" || tail -3 gpurun_out/k2s_$tag.err
}
run slab
run row SLQ_K2S=row
run kw18 SLQ_K2S_KWIN=262144
run kw16 SLQ_K2S_KWIN=65536
run nolag SLQ_K2S_LAG=100000
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sparse_gather" -c 1 -o gpurun_out/k2slab4_full python bench.py --config c4 --steps 1 --warmup 3 --no-cpu --no-e2e --iters 4 > gpurun_out/ncu_k2slab4.log 2>&1
ncu -i gpurun_out/k2slab4_full.ncu-rep --page raw --csv > gpurun_out/k2slab4_raw.csv 2>&1
SLQ_K2S=row timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sparse_gather" -c 1 -o gpurun_out/k2row4_full python bench.py --config c4 --steps 1 --warmup 3 --no-cpu --no-e2e --iters 4 > gpurun_out/ncu_k2row4.log 2>&1
ncu -i gpurun_out/k2row4_full.ncu-rep --page raw --csv > gpurun_out/k2row4_raw.csv 2>&1
