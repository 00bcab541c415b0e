# Round bench job: reference arm, our arm (C3 default), C4, and ncu evidence for the fused pass at C3.
tag=${1:-run}
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$tag.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c3_$tag.log 2>&1
timeout 900 python bench.py --config c4 --no-cpu > gpurun_out/bench_c4_$tag.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"fused_pass" -s 6 -c 1 -o gpurun_out/prof_pass_c3_$tag \
    python bench.py --no-e2e --no-cpu --steps 1 --warmup 3 > gpurun_out/ncu_pass_c3_$tag.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_$tag.csv \
    python bench.py --no-e2e --no-cpu --steps 1 --warmup 3 > gpurun_out/ncu_launch_c3_$tag.log 2>&1
echo finished
