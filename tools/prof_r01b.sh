CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
timeout 400 python -m pytest tests -m gpu -q --timeout=200 > gpurun_out/gpu_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/gpu_tests.log
$CMD > gpurun_out/bench_nocpu.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"panel|update|gather|bucketize|tri_inverse|gen_warp|maxabs|extract|trmv|mtz|mv_update|reduce_p|fused" --csv --log-file gpurun_out/launches_b.csv $CMD > gpurun_out/ncu_b.log 2>&1
echo finished
