# both arms at the headline config, as the driver runs them (reference first)
set -x
( time python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/bench_c3_ref.jsonl 2> gpurun_out/bench_c3_ref.err
( time python bench.py --steps 20 --warmup 5 ) > gpurun_out/bench_c3.jsonl 2> gpurun_out/bench_c3.err
