#!/bin/bash
# full ncu capture of the sparse sketch gather (K2s) at C4 (one launch)
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sparse_gather_slab" -c 1 -o gpurun_out/k2slab_full python bench.py --config c4 --steps 1 --warmup 3 --no-cpu --no-e2e --iters 4 > gpurun_out/ncu_k2slab.log 2>&1
echo "ncu exit $?"
ncu -i gpurun_out/k2slab_full.ncu-rep --page raw --csv > gpurun_out/k2slab_raw.csv 2>&1
