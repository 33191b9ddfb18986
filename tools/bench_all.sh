#!/bin/bash
# Every BASELINE config (and the C3 ablations) through bench.py on one GPU -> gpurun_out/configs.jsonl
mkdir -p gpurun_out
cfgs=${*:-"c1 c2 c3b1 c3b2 c3b4 c4 c5b8 c5b512"}
for c in $cfgs; do
  timeout 600 python bench.py --config "$c" --no-cpu --e2e-steps 100 >> gpurun_out/configs.jsonl 2>> gpurun_out/configs.err
done
