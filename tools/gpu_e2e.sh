#!/bin/bash
# e2e step pipelining: chunks per host-buffer step vs the bench's e2e number.
mkdir -p gpurun_out; rm -f gpurun_out/e2e_chunks.txt
timeout 300 python -m pytest tests -q -m gpu -k "step_api" > gpurun_out/pytest_step.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_step.log
for k in 1 2 3 4; do
  for cfg in c2 c5b512 c3b1; do
    KVQ_STEP_CHUNKS=$k timeout 300 python bench.py --config $cfg --steps 100 --warmup 5 --e2e-steps 200 --no-cpu > gpurun_out/e.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/e.json'))
print('chunks $k $cfg: device %.0f tok/s, e2e %.0f tok/s (%.1f us/step)' % (d['value'], d['e2e']['value'], d['config']['batch_per_gpu']/d['e2e']['value']*1e6))" >> gpurun_out/e2e_chunks.txt
  done
done
