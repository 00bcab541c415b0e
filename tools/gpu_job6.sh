tag=${1:-run}
timeout 600 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_parity.py -x -q > gpurun_out/tests_$tag.log 2>&1; echo "rc=$?" >> gpurun_out/tests_$tag.log
timeout 900 python bench.py --config c4 --no-cpu --no-e2e > gpurun_out/bench_c4_$tag.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"sparse_pass_kernel" -s 3 -c 1 -o gpurun_out/prof_spass_$tag \
   python bench.py --config c4 --no-cpu --no-e2e --steps 1 --warmup 3 > gpurun_out/ncu_spass_$tag.log 2>&1
echo finished
