#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:slq:: -c 2000 --csv --log-file gpurun_out/launches_end_c3.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --iters 30 > gpurun_out/ncu_end_c3.log 2>&1
echo "ncu rc $?"
