python tools/diag_qr.py > gpurun_out/diag_qr.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"panel|update|tri_inverse|maxabs|extract|trmv" --csv --log-file gpurun_out/launches_qr.csv python tools/diag_qr.py > gpurun_out/ncu_qr.log 2>&1
echo finished
