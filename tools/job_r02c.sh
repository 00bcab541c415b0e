# round 2 re-entry: full GPU suite, headline bench (both arms), sanitizers on small shapes
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/box.txt
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
( time python bench.py --steps 20 --warmup 5 ) > gpurun_out/bench_c3.jsonl 2> gpurun_out/bench_c3.err
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize_workload.py > gpurun_out/sanitize_$t.log 2>&1
  echo "$t rc=$?" >> gpurun_out/sanitize_rc.txt
done
