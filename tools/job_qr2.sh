SLQ_PANEL_PROF=1 timeout 300 python tools/diag_qr.py 4000 1000 > gpurun_out/qr2_c3.log 2>&1
SLQ_PANEL_PROF=1 timeout 300 python tools/diag_qr.py 8000 2000 > gpurun_out/qr2_c4.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -k "qr or QR or precond or householder or tri" > gpurun_out/qr2_tests.log 2>&1
