timeout 400 python -m pytest tests -m gpu -q --timeout=200 > gpurun_out/gpu_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/gpu_tests.log
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/bench_nocpu.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"panel|update|gather|bucketize|tri_inverse|gen_warp|mtz|mv_update|reduce_p|fused" --csv --log-file gpurun_out/launches_c.csv $CMD > gpurun_out/ncu_c.log 2>&1
SMALL="python bench.py --m 1000000 --steps 1 --warmup 3 --no-e2e --no-cpu"
$SMALL > gpurun_out/plain_small.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"gather_kernel|panel_kernel" -c 2 -o gpurun_out/prof_c $SMALL > gpurun_out/ncu_c2.log 2>&1
echo finished
