# round-2 full-set ncu captures of the dominant kernels (one launch each)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fused_pass|k5_fused|gather_dmma" -s 8 -c 3 -o gpurun_out/r02_c3_full python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --iters 30 > gpurun_out/ncu_r02_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sparse_upass|sparse_tpass" -s 6 -c 2 -o gpurun_out/r02_c4_full python bench.py --config c4 --steps 1 --warmup 3 --no-cpu --no-e2e --iters 4 > gpurun_out/ncu_r02_c4.log 2>&1
