#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sparse.py -x -q > gpurun_out/st_tests.log 2>&1; echo "tests rc $?"; tail -2 gpurun_out/st_tests.log
for mode in count chunk; do
  SLQ_STROWS=$mode timeout 300 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/st_$mode.jsonl 2>gpurun_out/st_$mode.err
  python -c "
import json; d=json.loads(open('gpurun_out/st_$mode.jsonl').read().strip().splitlines()[-1]); p=d['phases_s']; print('$mode', round(d['value'],4), 'apply', round(p['apply']*1e3,2), 'qr', round(p['qr']*1e3,2), 'lsqr', round(p['lsqr']*1e3,1), d['clocks']['reasons'])" || tail -3 gpurun_out/st_$mode.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"st_|gen_warp|slab|exclusive|scan" python bench.py --config c4 --steps 1 --warmup 1 --no-cpu --no-e2e --iters 2 > gpurun_out/st_launch.csv 2> gpurun_out/st_launch.err
