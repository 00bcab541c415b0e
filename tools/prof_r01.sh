set -x
CMD="python bench.py --m 1000000 --steps 1 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain_small.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fused_pass -s 3 -c 1 -o gpurun_out/prof_pass $CMD > gpurun_out/ncu_pass.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gather_kernel -c 1 -o gpurun_out/prof_gather $CMD > gpurun_out/ncu_gather.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"panel_kernel|update_kernel|bucketize|gen_warp|mtz|mv_update" -s 0 -c 8 -o gpurun_out/prof_misc $CMD > gpurun_out/ncu_misc.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py > gpurun_out/ncu_launches.log 2>&1
echo finished
