#!/bin/bash
# same-box A/B of the C3 bench: library at the start of this session (abtest/libslq_b200_old.so) vs HEAD
mkdir -p gpurun_out
cp paper_2506_03070_b200/libslq_b200.so /tmp/libnew.so
for rep in 1 2; do
  for v in new old; do
    if [ $v = old ]; then cp abtest/libslq_b200_old.so paper_2506_03070_b200/libslq_b200.so; else cp /tmp/libnew.so paper_2506_03070_b200/libslq_b200.so; fi
    timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab_$v.jsonl 2>gpurun_out/ab_$v.err
    python -c "
import json; d=json.loads(open('gpurun_out/ab_$v.jsonl').read().strip().splitlines()[-1]); p=d['phases_s']; print('$v', round(d['value'],4), 'apply', round(p['apply']*1e3,2), 'qr', round(p['qr']*1e3,2), 'lsqr', round(p['lsqr']*1e3,1), 'k4', round(d['roofline']['frac'],3), d['clocks']['reasons'])"
  done
done
cp /tmp/libnew.so paper_2506_03070_b200/libslq_b200.so
