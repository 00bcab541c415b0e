# sketch-apply job: GPU tests, slab vs row gather diag, launch list of the solve
tag=${1:-run}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_$tag.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests_$tag.log
timeout 300 python tools/diag_sketch.py 1000000 > gpurun_out/diag_sketch_$tag.log 2>&1
timeout 300 python tools/diag_sketch.py 200000 500 2000 8 >> gpurun_out/diag_sketch_$tag.log 2>&1
timeout 300 python tools/diag_sketch.py 100000 100 400 4 >> gpurun_out/diag_sketch_$tag.log 2>&1
timeout 300 python tools/diag_solve.py > gpurun_out/diag_solve_$tag.log 2>&1
echo finished
