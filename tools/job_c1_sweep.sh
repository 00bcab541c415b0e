#!/bin/bash
# C1 LSQR pass geometry sweep (tile rows R, stages S, CTAs per SM)
mkdir -p gpurun_out
run() {
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --m 100000 --n 100 --cond 1e3 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/c1s.jsonl 2>gpurun_out/c1s.err
  python -c "
import json; d=json.loads(open('gpurun_out/c1s.jsonl').read().strip().splitlines()[-1]); p=d['phases_s']; print('$tag', round(d['value']*1e3,3), 'ms lsqr', round(p['lsqr']*1e3,3), 'per it', round(p['lsqr_per_iteration']*1e6,1), 'us k4', round(d['roofline']['seconds_per_launch']*1e6,1))" || tail -2 gpurun_out/c1s.err
}
run default
run R24S6 SLQ_PASS_R=24 SLQ_PASS_S=6
run R16S8 SLQ_PASS_R=16 SLQ_PASS_S=8
run R32S3c2 SLQ_PASS_R=32 SLQ_PASS_S=3 SLQ_PASS_CPS=2
run R24S4c2 SLQ_PASS_R=24 SLQ_PASS_S=4 SLQ_PASS_CPS=2
run R16S4c3 SLQ_PASS_R=16 SLQ_PASS_S=4 SLQ_PASS_CPS=3
run R40S3c2 SLQ_PASS_R=40 SLQ_PASS_S=3 SLQ_PASS_CPS=2
run R8S8c2 SLQ_PASS_R=8 SLQ_PASS_S=8 SLQ_PASS_CPS=2
