#!/bin/bash
# e2e (no tracing) for 1/2/4 step chunks, interleaved x2, plus the box's raw H2D rate.
mkdir -p gpurun_out; rm -f gpurun_out/e2e2.txt
PYTHONPATH=. python tools/e2e_probe3.py >> gpurun_out/e2e2.txt 2>&1
for rep in 1 2; do
  for k in 1 2 4 8; do
    for cfg in c2 c5b512; do
      KVQ_STEP_CHUNKS=$k timeout 300 python bench.py --config $cfg --steps 50 --warmup 5 --e2e-steps 200 --no-cpu > gpurun_out/e.json 2>/dev/null
      python -c "
import json; d=json.load(open('gpurun_out/e.json'))
print('rep $rep chunks $k $cfg: e2e %.0f tok/s (%.1f us/step), device %.0f' % (d['e2e']['value'], d['config']['batch_per_gpu']/d['e2e']['value']*1e6, d['value']))" >> gpurun_out/e2e2.txt
    done
  done
done
