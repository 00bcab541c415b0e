ncu --set full --clock-control none --import-source on -k regex:"slab_gather_kernel" -s 1 -c 1 -o gpurun_out/prof_slab python tools/diag_sketch.py 1000000 > gpurun_out/ncu_slab.log 2>&1
echo finished
