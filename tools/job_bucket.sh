#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_parity.py -x -q > gpurun_out/bucket_tests.log 2>&1; echo "tests rc $?"; tail -2 gpurun_out/bucket_tests.log
for mode in count bitonic; do
  if [ $mode = bitonic ]; then export SLQ_BUCKET_BITONIC=1; fi
  timeout 300 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bk_$mode.jsonl 2>gpurun_out/bk_$mode.err
  python -c "
import json; d=json.loads(open('gpurun_out/bk_$mode.jsonl').read().strip().splitlines()[-1]); p=d['phases_s']; print('$mode', round(d['value'],4), 'apply', round(p['apply']*1e3,2), 'qr', round(p['qr']*1e3,2), 'lsqr', round(p['lsqr']*1e3,1), d['config'].get('lsqr_iterations'), d['clocks']['reasons'])"
done
unset SLQ_BUCKET_BITONIC
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"bucketize|srow|gen_warp|slab" python bench.py --config c4 --steps 1 --warmup 1 --no-cpu --no-e2e --iters 2 > gpurun_out/bk_launch.csv 2> gpurun_out/bk_launch.err
SLQ_BUCKET_BITONIC=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"bucketize|srow|gen_warp|slab" python bench.py --config c4 --steps 1 --warmup 1 --no-cpu --no-e2e --iters 2 > gpurun_out/bk_launch_bitonic.csv 2> gpurun_out/bk_launch_bitonic.err
