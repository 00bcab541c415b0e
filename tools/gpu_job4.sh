tag=${1:-run}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_$tag.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests_$tag.log
timeout 300 python tools/diag_qr.py > gpurun_out/diag_qr_$tag.log 2>&1
timeout 300 python tools/diag_qr.py 8000 2000 >> gpurun_out/diag_qr_$tag.log 2>&1
timeout 900 python bench.py --config c4 --no-cpu --no-e2e > gpurun_out/bench_c4_$tag.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_$tag.csv \
    python bench.py --config c4 --no-cpu --no-e2e --steps 1 --warmup 3 > gpurun_out/ncu_launch_c4_$tag.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"sparse_pass_kernel" -s 3 -c 1 -o gpurun_out/prof_spass_$tag \
   python bench.py --config c4 --no-cpu --no-e2e --steps 1 --warmup 3 > gpurun_out/ncu_spass_$tag.log 2>&1
echo finished
