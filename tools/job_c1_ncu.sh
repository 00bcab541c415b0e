#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fused_pass|k5_fused" -s 20 -c 2 -o gpurun_out/c1_full python bench.py --m 100000 --n 100 --cond 1e3 --steps 1 --warmup 1 --no-cpu --no-e2e --iters 10 > gpurun_out/c1_full.log 2>&1
ncu -i gpurun_out/c1_full.ncu-rep --page raw --csv > gpurun_out/c1_full_raw.csv 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --m 100000 --n 100 --cond 1e3 --steps 1 --warmup 1 --no-cpu --no-e2e --iters 10 > gpurun_out/c1_launch.csv 2>&1
