#!/bin/bash
# Short tails: in-kernel fp32 tail (tensor-core decode, rank 0) vs the separate tail pass.
mkdir -p gpurun_out; rm -f gpurun_out/tail_small.txt
for tm in 64 0; do
  touch paper_2502_14882_b200/csrc/kvq_capi.cu
  KVQ_NVCC_EXTRA="-DKVQ_TC_TAIL_MAX=$tm" python -c "from paper_2502_14882_b200 import build; build.build(False)"
  for t in 0 8 24; do
    timeout 300 python bench.py --tail $t --steps 300 --warmup 10 --e2e-steps 5 --no-cpu > gpurun_out/ts.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ts.json'))
print('tc_tail_max $tm tail $t: step %.1f us decode %.1f us' % (d['ms_per_step']*1e3, d['roofline']['launch_us']))" >> gpurun_out/tail_small.txt
  done
done
touch paper_2502_14882_b200/csrc/kvq_capi.cu; python -c "from paper_2502_14882_b200 import build; build.build(False)"
