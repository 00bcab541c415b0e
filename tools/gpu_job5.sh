for i in 1 2; do timeout 900 python bench.py --config c4 --no-cpu --no-e2e > gpurun_out/bench_c4_v$i.log 2>&1; done
SLQ_NO_L2_WINDOW=1 timeout 900 python bench.py --config c4 --no-cpu --no-e2e > gpurun_out/bench_c4_nowin.log 2>&1
SLQ_NO_L2_WINDOW=1 timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/bench_c3_nowin.log 2>&1
timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/bench_c3_win.log 2>&1
echo finished
