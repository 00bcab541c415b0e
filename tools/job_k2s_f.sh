#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_parity.py -x -q > gpurun_out/k2s_tests.log 2>&1; echo "tests rc $?"
tail -2 gpurun_out/k2s_tests.log
timeout 300 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu > gpurun_out/k2s_final.jsonl 2>gpurun_out/k2s_final.err
python -c "
import json; d=json.loads(open('gpurun_out/k2s_final.jsonl').read().strip().splitlines()[-1]); print(d['value'], d['phases_s'], d.get('first_solve_s'), d.get('e2e'))"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --config c4 --steps 1 --warmup 3 --no-cpu --no-e2e --iters 2 > gpurun_out/c4_launches2.csv 2> gpurun_out/c4_launches2.err
