# ncu --set full of the register panel (one launch of the 4000 x 1000 QR)
ncu --set full --clock-control none --import-source on -k regex:"panel_reg_kernel" -s 4 -c 1 -o gpurun_out/prof_panel3 python tools/diag_qr.py > gpurun_out/ncu_panel3.log 2>&1
echo finished
