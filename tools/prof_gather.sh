ncu --set full --clock-control none --import-source on -k gather_kernel -s 4 -c 1 -o gpurun_out/prof_gather2 python tools/diag_sketch.py 1000000 > gpurun_out/ncu_gather2.log 2>&1
echo finished
