#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/st_*.txt
PYTHONPATH=. python tools/e2e_probe3.py > gpurun_out/st_pcie.txt 2>&1
timeout 300 python bench.py --batch 32 --steps 100 --warmup 5 --e2e-steps 5 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('B=32 decode', d['roofline']['launch_us'])" > gpurun_out/st_b32.txt
for k in 1 2; do
  KVQ_STEP_CHUNKS=$k KVQ_STEP_TRACE=1 timeout 300 python bench.py --steps 20 --warmup 5 --e2e-steps 30 --no-cpu > gpurun_out/st_$k.json 2> gpurun_out/st_trace_$k.txt
done
