#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/qrg_tests.log 2>&1; echo "tests rc $?"; tail -2 gpurun_out/qrg_tests.log
for v in graph nograph; do
  if [ $v = nograph ]; then export SLQ_NO_QR_GRAPH=1; fi
  for cfg in "" "--config c4" "--m 1048576 --n 500 --cond 1e8" "--m 100000 --n 100 --cond 1e3"; do
    timeout 300 python bench.py $cfg --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/qrg.jsonl 2>gpurun_out/qrg.err
    python -c "
import json; d=json.loads(open('gpurun_out/qrg.jsonl').read().strip().splitlines()[-1]); p=d['phases_s']; print('$v', '$cfg', round(d['value']*1e3,3), 'ms qr', round(p['qr']*1e3,3), 'inv', round(p['inverse']*1e3,3), 'launches', d['gpu_launches'], d['config'].get('lsqr_iterations'))" || tail -3 gpurun_out/qrg.err
  done
done
