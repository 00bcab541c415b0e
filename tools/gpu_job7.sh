for i in 1 2; do SLQ_TRACE=1 timeout 900 python bench.py --config c4 --no-cpu --no-e2e > gpurun_out/bench_c4_t$i.log 2>&1; done
SLQ_TRACE=1 timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/bench_c3_t.log 2>&1
echo finished
