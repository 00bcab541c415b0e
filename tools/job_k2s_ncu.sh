#!/bin/bash
# K2s at C4: bench line, then one full ncu capture of the column-slab gather and one of the row gather
mkdir -p gpurun_out
timeout 300 python bench.py --config c4 --steps 3 --warmup 3 > gpurun_out/bench_c4_slab.jsonl 2> gpurun_out/bench_c4_slab.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sparse_gather" -c 1 -o gpurun_out/k2s_slab_full python bench.py --config c4 --steps 1 --warmup 3 --no-cpu --no-e2e --iters 4 > gpurun_out/ncu_k2s_slab.log 2>&1
ncu -i gpurun_out/k2s_slab_full.ncu-rep --page raw --csv > gpurun_out/k2s_slab_raw.csv 2>&1
SLQ_K2S=row timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sparse_gather" -c 1 -o gpurun_out/k2s_row_full python bench.py --config c4 --steps 1 --warmup 3 --no-cpu --no-e2e --iters 4 > gpurun_out/ncu_k2s_row.log 2>&1
ncu -i gpurun_out/k2s_row_full.ncu-rep --page raw --csv > gpurun_out/k2s_row_raw.csv 2>&1
