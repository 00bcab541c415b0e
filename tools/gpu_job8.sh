for c in 0 8 4; do echo "cluster cap $c"; SLQ_PANEL_CLUSTER=$c timeout 300 python tools/diag_qr.py; SLQ_PANEL_CLUSTER=$c timeout 300 python tools/diag_qr.py 8000 2000; done > gpurun_out/diag_qr_cl.log 2>&1
echo finished
