#!/bin/bash
# Where 4-warp CTAs start to win: c2 shape (n = 4096, G = 4) at 128..512 units.
mkdir -p gpurun_out; rm -f gpurun_out/w4thr.txt
for B in 16 24 32 40 48 64; do
  for w4 in 0 1; do
    KVQ_TC_W4=$w4 timeout 300 python bench.py --config c2 --batch $B --steps 100 --warmup 10 --e2e-steps 5 --no-cpu > gpurun_out/w.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/w.json'))
print('B=$B (%d units) W4=$w4: step %.1f us decode %.1f us' % ($B * 8, d['ms_per_step']*1e3, d['roofline']['launch_us']))" >> gpurun_out/w4thr.txt
  done
done
