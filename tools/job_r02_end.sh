#!/bin/bash
# end-of-round measurement batch: GPU suite, smoke, the driver's two bench commands, C1/C2/C4 lines, C3 launch list
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/box_end.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputests_end.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests_end.log; tail -2 gpurun_out/gputests_end.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_end.log 2>&1; tail -1 gpurun_out/smoke_end.log
s=$(date +%s); timeout 900 python bench.py > gpurun_out/bench_end_default.jsonl 2> gpurun_out/bench_end_default.err; e=$(date +%s)
echo "default bench wall $((e - s)) s" > gpurun_out/bench_end_walltime.txt
s=$(date +%s); timeout 900 python bench.py --impl reference > gpurun_out/bench_end_reference.jsonl 2> gpurun_out/bench_end_reference.err; e=$(date +%s)
echo "reference arm wall $((e - s)) s" >> gpurun_out/bench_end_walltime.txt
timeout 600 python bench.py --m 100000 --n 100 --cond 1e3 --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_end_c1.jsonl 2> gpurun_out/bench_end_c1.err
timeout 600 python bench.py --m 1048576 --n 500 --steps 10 --warmup 5 --no-cpu > gpurun_out/bench_end_c2.jsonl 2> gpurun_out/bench_end_c2.err
timeout 900 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_end_c4.jsonl 2> gpurun_out/bench_end_c4.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:slq:: -c 2000 --csv --log-file gpurun_out/launches_end_c3.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --iters 30 > gpurun_out/ncu_end_c3.log 2>&1
for f in default reference c1 c2 c4; do python -c "
import json; d=json.loads(open('gpurun_out/bench_end_$f.jsonl').read().strip().splitlines()[-1]); print('$f', d.get('value'), d.get('e2e',{}).get('value') if isinstance(d.get('e2e'),dict) else None, d.get('roofline',{}).get('frac') if isinstance(d.get('roofline'),dict) else None, d.get('clocks'))" 2>&1 | tail -1; done
cat gpurun_out/bench_end_walltime.txt
SLQ_GUARD=1 timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputests_end_guard.log 2>&1; echo "guard suite rc=$?" >> gpurun_out/gputests_end_guard.log; tail -2 gpurun_out/gputests_end_guard.log
