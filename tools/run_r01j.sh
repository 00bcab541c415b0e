python tools/diag_qr.py > gpurun_out/diag_qr.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"panel_kernel" -s 2 -c 1 -o gpurun_out/prof_panel2 python tools/diag_qr.py > gpurun_out/ncu_panel2.log 2>&1
echo finished
