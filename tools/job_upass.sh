#!/bin/bash
# u_hat pass ring geometries at C4 (tools/diag_spass.py), sparse tests, C4 bench line
mkdir -p gpurun_out
GEOMS=2,1,2,1 timeout 600 python tools/diag_spass.py > gpurun_out/upass_geom.log 2>&1; cat gpurun_out/upass_geom.log | tail -4
GEOMS=2,1 timeout 600 python tools/diag_spass.py 4194304 1000 20 2>&1 | tail -2
GEOMS=2,1 timeout 600 python tools/diag_spass.py 4194304 500 48 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_sparse.py -x -q > gpurun_out/upass_tests.log 2>&1; echo "tests rc $?"; tail -1 gpurun_out/upass_tests.log
timeout 300 python bench.py --config c4 --steps 3 --warmup 3 > gpurun_out/bench_c4_upass.jsonl 2> gpurun_out/bench_c4_upass.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_c4_upass.jsonl').read().strip().splitlines()[-1]); print(d['value'], d['phases_s']['apply'], d['phases_s']['lsqr'], d['roofline']['frac'], d['roofline']['seconds_per_launch'], d['clocks'])"
