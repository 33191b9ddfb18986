#!/bin/bash
# Step API timelines (KVQ_STEP_TRACE) for 1 and 2 chunks, and the bench e2e for each.
mkdir -p gpurun_out; rm -f gpurun_out/step_trace*.txt
for k in 1 2 4; do
  KVQ_STEP_CHUNKS=$k KVQ_STEP_TRACE=1 timeout 300 python bench.py --steps 20 --warmup 5 --e2e-steps 40 --no-cpu > /dev/null 2> gpurun_out/step_trace_$k.txt
  KVQ_STEP_CHUNKS=$k timeout 300 python bench.py --steps 100 --warmup 5 --e2e-steps 300 --no-cpu > gpurun_out/st2.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/st2.json')); print('chunks $k e2e', round(d['e2e']['value']), 'us/step', round(64/d['e2e']['value']*1e6,1))" >> gpurun_out/step_trace_sum.txt
done
