#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_envelope.py tests/test_gpu_edge.py tests/test_gpu_robustness.py -x -q > gpurun_out/inv_tests.log 2>&1; echo "tests rc $?"; tail -2 gpurun_out/inv_tests.log
for cfg in "" "--config c4" "--m 1048576 --n 500 --cond 1e8"; do
  timeout 300 python bench.py $cfg --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/inv.jsonl 2>gpurun_out/inv.err
  python -c "
import json; d=json.loads(open('gpurun_out/inv.jsonl').read().strip().splitlines()[-1]); p=d['phases_s']; print('$cfg', round(d['value']*1e3,3), 'ms qr', round(p['qr']*1e3,3), 'inv', round(p['inverse']*1e3,3), d['config'].get('lsqr_iterations'), d['eta_final'])" || tail -3 gpurun_out/inv.err
done
