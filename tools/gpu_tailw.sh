#!/bin/bash
# Tail pass warps per CTA for short / long tails.
mkdir -p gpurun_out; rm -f gpurun_out/tailw.txt
for w in 8 4 2; do
  touch paper_2502_14882_b200/csrc/k2_tail.cu
  KVQ_NVCC_EXTRA="-DKVQ_TAIL_WARPS=$w" python -c "from paper_2502_14882_b200 import build; build.build(False)" || continue
  for t in 64 256 1024; do
    timeout 300 python bench.py --tail $t --steps 200 --warmup 10 --e2e-steps 5 --no-cpu > gpurun_out/w.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/w.json'))
print('tail warps $w tail $t: step %.1f us decode %.1f us' % (d['ms_per_step']*1e3, d['roofline']['launch_us']))" >> gpurun_out/tailw.txt
  done
done
touch paper_2502_14882_b200/csrc/k2_tail.cu; python -c "from paper_2502_14882_b200 import build; build.build(False)"
