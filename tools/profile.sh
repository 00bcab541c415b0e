# ncu captures used for profiles/ (run on the GPU box from the repo root, one
# GPU, never under torchrun).  Each capture runs only after the same command
# has exited 0 without ncu.
#   bash tools/profile.sh <what> [tag]
#   what: pass_c3 | launches_c3 | gather | panel | sparse_pass | launches_c4
what=${1:?what}; tag=${2:-run}
case $what in
  pass_c3)   CMD="python bench.py --no-e2e --no-cpu --steps 1 --warmup 3"; K="-k regex:fused_pass -s 6 -c 1";;
  gather)    CMD="python tools/diag_k2d.py 1000000 1000 4000 8"; K="-k regex:gather_dmma -s 1 -c 1";;
  panel)     CMD="python tools/diag_qr.py"; K="-k regex:panel_reg_kernel -s 4 -c 1";;
  sparse_pass) CMD="python bench.py --config c4 --no-cpu --no-e2e --steps 1 --warmup 3"; K="-k regex:sparse_pass_kernel -s 3 -c 1";;
  launches_c3) CMD="python bench.py --no-e2e --no-cpu --steps 1 --warmup 3";;
  launches_c4) CMD="python bench.py --config c4 --no-e2e --no-cpu --steps 1 --warmup 3";;
  *) echo "unknown: $what"; exit 2;;
esac
timeout 1200 $CMD > gpurun_out/plain_${what}_$tag.log 2>&1 || { echo "plain run failed"; exit 1; }
case $what in
  launches_*) timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
                --log-file gpurun_out/${what}_$tag.csv $CMD > gpurun_out/ncu_${what}_$tag.log 2>&1;;
  *) timeout 1800 ncu --set full --clock-control none --import-source on $K -o gpurun_out/prof_${what}_$tag \
                $CMD > gpurun_out/ncu_${what}_$tag.log 2>&1;;
esac
echo finished
