timeout 400 python -m pytest tests -m gpu -q --timeout=200 -x > gpurun_out/gpu_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/gpu_tests.log
python tools/diag_qr.py > gpurun_out/diag_qr.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"panel|update|inverse|merge|maxabs|extract|trmv|transpose|zero_lower" --csv --log-file gpurun_out/launches_qr.csv python tools/diag_qr.py > gpurun_out/ncu_qr.log 2>&1
timeout 300 python tools/diag_solve.py 4000000 > gpurun_out/diag.log 2>&1; echo "exit $?" >> gpurun_out/diag.log
echo finished
