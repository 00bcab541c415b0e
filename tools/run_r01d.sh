timeout 400 python -m pytest tests -m gpu -q --timeout=200 > gpurun_out/gpu_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/gpu_tests.log
timeout 300 python tools/diag_solve.py 4000000 > gpurun_out/diag.log 2>&1; echo "exit $?" >> gpurun_out/diag.log
timeout 600 python bench.py > gpurun_out/bench_full.log 2>&1; echo "exit $?" >> gpurun_out/bench_full.log
