# full GPU suite + C3 and C4 bench lines
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
bash tools/job_c4.sh
timeout 900 python bench.py --steps 10 --warmup 5 --no-cpu > gpurun_out/bench_c3.jsonl 2> gpurun_out/bench_c3.err
