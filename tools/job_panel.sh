#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_envelope.py tests/test_gpu_edge.py -x -q > gpurun_out/panel_tests.log 2>&1; echo "tests rc $?"; tail -1 gpurun_out/panel_tests.log
SLQ_PANEL_PROF=1 timeout 300 python tools/diag_qr.py 4000 1000 2>&1 | tail -7
SLQ_PANEL_PROF=1 timeout 300 python tools/diag_qr.py 8000 2000 2>&1 | tail -7
for cfg in "" "--config c4"; do
  timeout 300 python bench.py $cfg --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/pn.jsonl 2>gpurun_out/pn.err
  python -c "
import json; d=json.loads(open('gpurun_out/pn.jsonl').read().strip().splitlines()[-1]); p=d['phases_s']; print('$cfg', round(d['value']*1e3,3), 'ms qr', round(p['qr']*1e3,3), 'inv', round(p['inverse']*1e3,3), d['config'].get('lsqr_iterations'), d['eta_final'])" || tail -3 gpurun_out/pn.err
done
