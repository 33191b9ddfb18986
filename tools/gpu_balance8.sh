#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/balance8.txt
timeout 600 python -m pytest tests -q -m gpu -k "many_units or step_api or randomized" > gpurun_out/pytest_b8.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_b8.log)" >> gpurun_out/balance8.txt
run() { local label=$1 bal=$2; shift 2
  KVQ_TC_BALANCE=$bal timeout 300 python bench.py "$@" --steps 200 --warmup 10 --e2e-steps 5 --no-cpu > gpurun_out/w.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/w.json'))
print('$label balance=$bal: step %.1f us decode %.1f us' % (d['ms_per_step']*1e3, d['roofline']['launch_us']))" >> gpurun_out/balance8.txt; }
for bal in 0 1; do
  run "c3b1 (256 units, n=8192)" $bal --config c3b1
  run "c3b4 (256 units, n=8192)" $bal --config c3b4
  run "c2 B=24 (192 units)" $bal --config c2 --batch 24
  run "c2 B=32 (256 units)" $bal --config c2 --batch 32
  run "c2 (512 units)" $bal --config c2
done
