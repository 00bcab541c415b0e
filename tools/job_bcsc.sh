#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sparse.py -x -q > gpurun_out/bcsc_tests.log 2>&1; echo "tests rc $?"; tail -1 gpurun_out/bcsc_tests.log
for g in auto 8 16 32 64 148; do
  if [ $g = auto ]; then unset SLQ_BCSC_GRID; else export SLQ_BCSC_GRID=$g; fi
  timeout 300 python bench.py --config c4 --steps 1 --warmup 1 --no-cpu --no-e2e --iters 2 > gpurun_out/bcsc_$g.jsonl 2>gpurun_out/bcsc_$g.err
  python -c "
import json; d=json.loads(open('gpurun_out/bcsc_$g.jsonl').read().strip().splitlines()[-1]); print('grid $g', 'build', round(d['transposed_copy_build_s']*1e3,1), 'ms first solve', round(d['first_solve_s']*1e3,1), 'ms')" || tail -2 gpurun_out/bcsc_$g.err
done
