#!/bin/bash
# K2d bank-aware grouping: parity tests, timing at m = 1e6 and C3, ncu wavefronts
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_envelope.py -x -q > gpurun_out/k2d_tests.log 2>&1; echo "tests rc $?"; tail -2 gpurun_out/k2d_tests.log
timeout 300 python tools/diag_k2d.py 1000000 1000 4000 8 2>&1 | tail -4
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/k2d_c3.jsonl 2>gpurun_out/k2d_c3.err
python -c "
import json; d=json.loads(open('gpurun_out/k2d_c3.jsonl').read().strip().splitlines()[-1]); p=d['phases_s']; print('C3', round(d['value'],4), 'apply', round(p['apply']*1e3,2), 'qr', round(p['qr']*1e3,2), 'lsqr', round(p['lsqr']*1e3,1), d['clocks']['reasons'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gather_dmma -c 1 -o gpurun_out/k2d_bank python tools/diag_k2d.py 1000000 1000 4000 8 > gpurun_out/k2d_bank.log 2>&1
ncu -i gpurun_out/k2d_bank.ncu-rep --page raw --csv > gpurun_out/k2d_bank_raw.csv 2>&1
