# round 2: bench flow at a small size (both arms), sanitizer runs on the small workload
set -x
python bench.py --m 200000 --n 100 --steps 3 --warmup 3 > gpurun_out/bench_small.jsonl 2> gpurun_out/bench_small.err
python bench.py --impl reference --m 200000 --n 100 --steps 3 --warmup 3 >> gpurun_out/bench_small.jsonl 2>> gpurun_out/bench_small.err
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize_workload.py > gpurun_out/sanitize_$t.log 2>&1
  echo "$t rc=$?" >> gpurun_out/sanitize_rc.txt
done
