tag=${1:-run}
timeout 600 python -m pytest tests/test_gpu_sparse.py -x -q > gpurun_out/sparse_tests_$tag.log 2>&1; echo "rc=$?" >> gpurun_out/sparse_tests_$tag.log
timeout 900 python bench.py --config c4 --no-cpu --no-e2e > gpurun_out/bench_c4_$tag.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_$tag.csv \
    python bench.py --config c4 --no-cpu --no-e2e --steps 1 --warmup 3 > gpurun_out/ncu_launch_c4_$tag.log 2>&1
echo finished
