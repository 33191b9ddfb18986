#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/split.txt
for sp in 0 2 3 4; do
  for cfg in c2 c3b1 c5b512; do
    KVQ_TC_SPLIT=$sp timeout 300 python bench.py --config $cfg --steps 200 --warmup 10 --e2e-steps 5 --no-cpu > gpurun_out/sp.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/sp.json'))
print('split $sp $cfg: step %.1f us decode %.1f us frac %.3f' % (d['ms_per_step']*1e3, d['roofline']['launch_us'], d['roofline']['frac']))" >> gpurun_out/split.txt
  done
done
