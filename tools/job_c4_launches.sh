#!/bin/bash
# launch list (per-kernel durations) of one C4 solve: which kernels make up the sketch-apply phase
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none --csv python bench.py --config c4 --steps 1 --warmup 3 --no-cpu --no-e2e --iters 2 > gpurun_out/c4_launches.csv 2> gpurun_out/c4_launches.err
echo "ncu exit $?"
