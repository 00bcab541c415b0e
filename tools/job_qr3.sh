#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_envelope.py -x -q > gpurun_out/qr3_tests.log 2>&1; echo "tests rc $?"; tail -2 gpurun_out/qr3_tests.log
for cfg in "--config c3" "--config c4" "--m 1048576 --n 500 --cond 1e8"; do
  timeout 300 python bench.py $cfg --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/qr3.jsonl 2>gpurun_out/qr3.err
  python -c "
import json; d=json.loads(open('gpurun_out/qr3.jsonl').read().strip().splitlines()[-1]); p=d['phases_s']; print('$cfg', round(d['value'],4), 'qr', round(p['qr']*1e3,3), 'inv', round(p['inverse']*1e3,3), 'apply', round(p['apply']*1e3,2), d['clocks']['reasons'])" || tail -3 gpurun_out/qr3.err
done
