timeout 300 python tools/diag_sketch.py 1000000 > gpurun_out/diag_sketch_$1.log 2>&1
timeout 300 python tools/diag_sketch.py 200000 500 2000 8 >> gpurun_out/diag_sketch_$1.log 2>&1
echo finished
