ncu --set full --clock-control none --import-source on -k regex:"sparse_pass_kernel|update_apply_kernel" -s 40 -c 2 -o gpurun_out/prof_c4 \
   python bench.py --config c4 --no-cpu --no-e2e --steps 1 --warmup 3 > gpurun_out/ncu_c4.log 2>&1
echo finished
