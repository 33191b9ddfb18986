#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/stage.txt
for v in "2048 3" "4096 2" "1024 6"; do
  set -- $v
  touch paper_2502_14882_b200/csrc/k2_decode_tc.cu
  KVQ_NVCC_EXTRA="-DKVQ_TC_STAGE_BYTES=$1 -DKVQ_TC_STAGES=$2" python -c "from paper_2502_14882_b200 import build; build.build(False)" || continue
  for cfg in c2 c3b1 c5b512; do
    timeout 300 python bench.py --config $cfg --steps 100 --warmup 10 --e2e-steps 5 --no-cpu > gpurun_out/w.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/w.json'))
print('stage $1 w4stages $2 $cfg: step %.1f us decode %.1f us frac %.3f' % (d['ms_per_step']*1e3, d['roofline']['launch_us'], d['roofline']['frac']))" >> gpurun_out/stage.txt
  done
done
touch paper_2502_14882_b200/csrc/k2_decode_tc.cu; python -c "from paper_2502_14882_b200 import build; build.build(False)"
