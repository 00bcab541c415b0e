# QR change check: GPU tests, QR diagnostics (C3 and C4 shapes), solve phases, QR launch list
tag=${1:-run}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_$tag.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests_$tag.log
timeout 300 python tools/diag_qr.py > gpurun_out/diag_qr_$tag.log 2>&1
timeout 300 python tools/diag_qr.py 8000 2000 >> gpurun_out/diag_qr_$tag.log 2>&1
timeout 300 python tools/diag_solve.py > gpurun_out/diag_solve_$tag.log 2>&1
echo finished
