#!/bin/bash
# Every BASELINE config through bench.py (1 GPU), one JSON line each.
mkdir -p gpurun_out
: > gpurun_out/configs.jsonl
for c in c1 c2 c3b1 c3b2 c3b4 c4 c5b8 c5b512; do
  timeout 600 python bench.py --config $c --steps 100 --warmup 10 --e2e-steps 20 --cpu-requests 4 --steps-cpu 2 >> gpurun_out/configs.jsonl 2> gpurun_out/configs_$c.err || echo "{\"config_name\": \"$c\", \"failed\": true}" >> gpurun_out/configs.jsonl
done
