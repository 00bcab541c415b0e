#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sparse_upass|sparse_tpass" -s 4 -c 2 -o gpurun_out/c4_2pass_r2 python bench.py --config c4 --steps 1 --warmup 3 --no-cpu --no-e2e --iters 4 > gpurun_out/ncu_c4_2pass_r2.log 2>&1
ncu -i gpurun_out/c4_2pass_r2.ncu-rep --page raw --csv > gpurun_out/c4_2pass_r2_raw.csv 2>&1
