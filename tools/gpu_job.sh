# One gpurun job: GPU tests, QR + solve diagnostics, kernel launch list of the QR.
# usage (from the repo root, on the box): bash tools/gpu_job.sh [tag]
tag=${1:-run}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_$tag.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests_$tag.log
timeout 300 python tools/diag_qr.py > gpurun_out/diag_qr_$tag.log 2>&1
timeout 300 python tools/diag_solve.py > gpurun_out/diag_solve_$tag.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_qr_$tag.csv \
    python tools/diag_qr.py > gpurun_out/ncu_qr_$tag.log 2>&1
echo finished
