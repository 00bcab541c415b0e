#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sparse.py -x -q > gpurun_out/st_tests.log 2>&1; echo "tests rc $?"; tail -2 gpurun_out/st_tests.log
timeout 300 python bench.py --config c4 --steps 3 --warmup 3 > gpurun_out/bench_c4_late.jsonl 2>gpurun_out/bench_c4_late.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_c4_late.jsonl').read().strip().splitlines()[-1]); p=d['phases_s']; print(round(d['value'],4), 'apply', round(p['apply']*1e3,2), 'qr', round(p['qr']*1e3,2), 'lsqr', round(p['lsqr']*1e3,1), d['roofline']['frac'], d['clocks']['reasons'])"
