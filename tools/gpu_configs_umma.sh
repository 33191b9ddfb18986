#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/configs_umma.jsonl
for c in c2 c3b1 c3b4 c4 c5b8; do
  timeout 600 python bench.py --config $c --path umma --steps 100 --warmup 10 --e2e-steps 10 --no-cpu >> gpurun_out/configs_umma.jsonl 2> gpurun_out/cu_$c.err || echo "{\"config_name\": \"$c\", \"failed\": true}" >> gpurun_out/configs_umma.jsonl
done
