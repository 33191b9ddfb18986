#!/bin/bash
# Cluster split S vs units: which S minimises the decode for few / many units.
mkdir -p gpurun_out; rm -f gpurun_out/split2.txt
run() {  # label, split, bench args...
  local label=$1 sp=$2; shift 2
  KVQ_TC_SPLIT=$sp timeout 300 python bench.py "$@" --steps 100 --warmup 10 --e2e-steps 5 --no-cpu > gpurun_out/s2.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/s2.json'))
print('$label S=$sp: step %.1f us decode %.1f us frac %.3f' % (d['ms_per_step']*1e3, d['roofline']['launch_us'], d['roofline']['frac']))" >> gpurun_out/split2.txt
}
for sp in 1 2 3 5 8; do run "c1 (1 unit, n=1024)" $sp --config c1; done
for sp in 1 2 3 5; do run "c5b8 (64 units, n=4096)" $sp --config c5b8; done
for sp in 1 2 3; do run "c2 B=16 (128 units, n=4096)" $sp --config c2 --batch 16; done
for sp in 1 2 3; do run "c3b1 B=16 (128 units, n=8192)" $sp --config c3b1 --batch 16; done
for sp in 1 2; do run "c2 B=24 (192 units, n=4096)" $sp --config c2 --batch 24; done
for sp in 4 5 8; do run "c4 (128 units x 2 groups, n=32768)" $sp --config c4; done
