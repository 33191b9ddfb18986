#!/bin/bash
# 4-warp CTAs (four per SM) vs 8-warp CTAs (two per SM) for the IMMA decode.
mkdir -p gpurun_out; rm -f gpurun_out/w4.txt
KVQ_TC_W4=1 timeout 600 python -m pytest tests -q -m gpu -x -k "golden or full_size or gqa or randomized or long_tail or step_api" > gpurun_out/pytest_w4.log 2>&1; echo "W4 tests: $(tail -1 gpurun_out/pytest_w4.log)" >> gpurun_out/w4.txt
for w4 in 0 1; do
  for cfg in c2 c3b1 c3b4 c4 c5b8 c5b512; do
    KVQ_TC_W4=$w4 timeout 300 python bench.py --config $cfg --steps 100 --warmup 10 --e2e-steps 5 --no-cpu > gpurun_out/w.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/w.json'))
print('W4=$w4 $cfg: step %.1f us decode %.1f us frac %.3f' % (d['ms_per_step']*1e3, d['roofline']['launch_us'], d['roofline']['frac']))" >> gpurun_out/w4.txt
  done
done
