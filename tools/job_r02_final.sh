# round-2 measurement batch: GPU suite, smoke, C1 / C2 / C3 / C4 bench lines, K4 + K2d + sparse ncu
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/box_final.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_final.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests_final.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1
timeout 600 python bench.py --m 100000 --n 100 --cond 1e3 --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_c1.jsonl 2> gpurun_out/bench_c1.err
timeout 600 python bench.py --m 1048576 --n 500 --steps 10 --warmup 5 --no-cpu > gpurun_out/bench_c2.jsonl 2> gpurun_out/bench_c2.err
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c3.jsonl 2> gpurun_out/bench_c3.err
timeout 900 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c4.jsonl 2> gpurun_out/bench_c4.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:slq:: -c 2000 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --iters 30 > gpurun_out/ncu_c3_launches.log 2>&1
