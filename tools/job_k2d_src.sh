#!/bin/bash
# K2d source-level capture at m = 1e6 (which lines replay shared-memory wavefronts, which stall)
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gather_dmma -c 1 -o gpurun_out/k2d_src python tools/diag_k2d.py 1000000 1000 4000 8 > gpurun_out/k2d_src.log 2>&1
ncu -i gpurun_out/k2d_src.ncu-rep --page raw --csv > gpurun_out/k2d_src_raw.csv 2>&1
ncu -i gpurun_out/k2d_src.ncu-rep --page source --csv --print-source sass > gpurun_out/k2d_src_sass.csv 2>&1
