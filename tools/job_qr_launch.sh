#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"panel|narrow|update|merge|diag_block|maxabs|extract|trmv" python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --iters 2 > gpurun_out/qr_launch_c3.csv 2> gpurun_out/qr_launch_c3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"panel|narrow|update|merge|diag_block|maxabs|extract|trmv" python bench.py --config c4 --steps 1 --warmup 1 --no-cpu --no-e2e --iters 2 > gpurun_out/qr_launch_c4.csv 2> gpurun_out/qr_launch_c4.err
