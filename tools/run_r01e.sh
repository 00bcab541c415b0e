timeout 400 python -m pytest tests -m gpu -q --timeout=200 -x > gpurun_out/gpu_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/gpu_tests.log
timeout 300 python tools/diag_solve.py 4000000 > gpurun_out/diag.log 2>&1; echo "exit $?" >> gpurun_out/diag.log
CMD="python tools/diag_solve.py 1000000"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"panel|update|gather|bucketize|tri_inverse|mtz|mv_update|reduce_p|fused" --csv --log-file gpurun_out/launches_e.csv $CMD > gpurun_out/ncu_e.log 2>&1
echo finished
