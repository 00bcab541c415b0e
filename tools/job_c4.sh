# C4 sparse: bench line + kernel launch list of one solve (two-pass K4s)
timeout 900 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c4.jsonl 2> gpurun_out/bench_c4.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"sparse_pass|sparse_upass|sparse_tpass|bcsc_build" -c 12 --csv --log-file gpurun_out/launches_c4.csv python bench.py --config c4 --steps 1 --warmup 3 --no-cpu --no-e2e --iters 4 > gpurun_out/ncu_c4.log 2>&1
