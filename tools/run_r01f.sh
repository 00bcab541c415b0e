python tools/diag_qr.py > gpurun_out/diag_qr.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"panel_kernel|mtz_kernel|mv_update" -s 4 -c 2 -o gpurun_out/prof_panel python tools/diag_qr.py > gpurun_out/ncu_panel.log 2>&1
python tools/diag_solve.py 1000000 > gpurun_out/diag_small.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"mtz_kernel|mv_update" -s 40 -c 2 -o gpurun_out/prof_small python tools/diag_solve.py 1000000 > gpurun_out/ncu_small.log 2>&1
echo finished
