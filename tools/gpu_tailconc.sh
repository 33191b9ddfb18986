#!/bin/bash
# Long tails: tail pass concurrent with the decode vs chained after it.
mkdir -p gpurun_out; rm -f gpurun_out/tailconc.txt
timeout 600 python -m pytest tests -q -m gpu -k "tail or many_units or randomized or full_precision" > gpurun_out/pytest_tc.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_tc.log)" >> gpurun_out/tailconc.txt
for conc in 0 1; do
  for t in 64 256 1024; do
    KVQ_TAIL_CONCURRENT=$conc timeout 300 python bench.py --tail $t --steps 200 --warmup 10 --e2e-steps 5 --no-cpu > gpurun_out/w.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/w.json'))
print('concurrent=$conc tail $t: step %.1f us decode %.1f us frac %.3f' % (d['ms_per_step']*1e3, d['roofline']['launch_us'], d['roofline']['frac']))" >> gpurun_out/tailconc.txt
  done
done
