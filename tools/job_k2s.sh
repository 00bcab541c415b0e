#!/bin/bash
# K2s: sparse sketch-gather parity + C4 timing of the slab gather vs the row gather and pacing variants
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sparse.py -x -q > gpurun_out/k2s_tests.log 2>&1; echo "tests rc $?"
tail -3 gpurun_out/k2s_tests.log
run() {  # tag, env...
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/k2s_$tag.jsonl 2>gpurun_out/k2s_$tag.err
  python -c "
import json; d=json.loads(open('gpurun_out/k2s_$tag.jsonl').read().strip().splitlines()[-1]); print('$tag', round(d['value'],4), 'apply', round(d['phases_s']['apply']*1e3,2), 'ms', d['clocks']['reasons'])" || tail -3 gpurun_out/k2s_$tag.err
}
run slab
run row SLQ_K2S=row
run kw16 SLQ_K2S_KWIN=65536
run kw18 SLQ_K2S_KWIN=262144
run lag1 SLQ_K2S_LAG=1
run lag8 SLQ_K2S_LAG=8
run nolag SLQ_K2S_LAG=100000
