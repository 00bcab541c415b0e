# full ncu capture of the two-pass sparse LSQR operator kernels (one launch each)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sparse_upass|sparse_tpass" -s 4 -c 2 -o gpurun_out/c4_2pass_full python bench.py --config c4 --steps 1 --warmup 3 --no-cpu --no-e2e --iters 4 > gpurun_out/ncu_c4_full.log 2>&1
