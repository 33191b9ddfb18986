#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/balance.txt
timeout 600 python -m pytest tests -q -m gpu -k "many_units or step_api or long_tail" > gpurun_out/pytest_bal.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_bal.log)" >> gpurun_out/balance.txt
for B in 40 48 54 64 72; do
  for bal in 0 1; do
    KVQ_TC_BALANCE=$bal timeout 300 python bench.py --config c2 --batch $B --steps 200 --warmup 10 --e2e-steps 5 --no-cpu > gpurun_out/w.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/w.json'))
print('B=$B (%d units) balance=$bal: step %.1f us decode %.1f us' % ($B * 8, d['ms_per_step']*1e3, d['roofline']['launch_us']))" >> gpurun_out/balance.txt
  done
done
