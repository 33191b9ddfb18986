#!/bin/bash
# G > 4: NT = 2 single CTA vs two head-group CTAs (NT = 1); parity tests under both.
mkdir -p gpurun_out; rm -f gpurun_out/headsplit.txt
for hs in 0 1; do
  KVQ_TC_HEADSPLIT=$hs timeout 600 python -m pytest tests -q -m gpu -k "gqa or full_size or randomized or golden_m8" > gpurun_out/pytest_hs$hs.log 2>&1; echo "hs=$hs $(tail -1 gpurun_out/pytest_hs$hs.log)" >> gpurun_out/headsplit.txt
  for cfg in c4; do
    KVQ_TC_HEADSPLIT=$hs timeout 300 python bench.py --config $cfg --steps 100 --warmup 10 --e2e-steps 5 --no-cpu > gpurun_out/hs.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/hs.json'))
print('headsplit $hs $cfg: step %.1f us decode %.1f us frac %.3f' % (d['ms_per_step']*1e3, d['roofline']['launch_us'], d['roofline']['frac']))" >> gpurun_out/headsplit.txt
  done
  for G in 6 8; do
    KVQ_TC_HEADSPLIT=$hs timeout 300 python - >> gpurun_out/headsplit.txt 2>&1 <<PY
import torch
from paper_2502_14882_b200 import kvq
B, H, G, n, d = 64, 8, $G, 4096, 128
k = torch.randn((B, H, n, d), device="cuda"); v = torch.randn((B, H, n, d), device="cuda")
c = kvq.BatchedCache.build_device(k, v, kvq.QuantizationConfig(1), kvq.CalibrationParams(1, 0), group=G)
del k, v
q = torch.randn((B, H, G, d), device="cuda"); out = torch.empty_like(q)
for _ in range(5): c.decode_device(q, out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50): c.decode_device(q, out)
e1.record(); torch.cuda.synchronize()
print("headsplit $hs B=64 G=$G n=4096: decode %.1f us" % (e0.elapsed_time(e1) / 50 * 1e3))
PY
  done
done
