ncu --set full --clock-control none -k regex:"gather_warp|warp_bucket|gather_dmma|tile_bucket" -c 4 -o gpurun_out/k2w_full python tools/diag_k2w.py 1000000 1000 4000 8 k2w16 > gpurun_out/k2w_ncu.log 2>&1
ncu --clock-control none -k regex:"gather_dmma|tile_bucket" -c 2 --set full -o gpurun_out/k2d_full python tools/diag_k2w.py 1000000 1000 4000 8 dmma >> gpurun_out/k2w_ncu.log 2>&1
