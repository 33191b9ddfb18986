"""Timeline of the persistent SM-level decode (KVQ_TRACE_FILE stamps, k2_decode_ps.cu):
start, dependency released, prologue done, phase A done (params), phase B done, end.
python tools/trace_ps.py [config]"""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
raw = str(ROOT / "gpurun_out" / "trace_ps.bin")
os.environ["KVQ_TRACE_FILE"] = raw
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2502_14882_b200 import kvq  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
batch, H, G, n, bits, tau, _ = bench.CONFIGS[cfg]
dev = torch.device("cuda", 0)
k = torch.randn((batch, H, n, 128), device=dev)
v = torch.randn((batch, H, n, 128), device=dev)
c = kvq.BatchedCache.build_device(k, v, kvq.QuantizationConfig(bits), kvq.CalibrationParams(*tau), group=G)
c.set_path(7)
q = torch.randn((batch, H, G, 128), device=dev)
out = torch.empty_like(q)
for _ in range(3):
    c.decode_device(q, out, 0)
torch.cuda.synchronize()
t = np.fromfile(raw, dtype=np.uint64).reshape(-1, 256).astype(np.int64)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
us = lambda x: (x - t0) / 1e3
print(f"{cfg}: {len(t)} CTAs, span {us(t[:, 5].max()):.1f} us")
for label, col in (("start", 0), ("dependency released", 3), ("prologue done", 2), ("phase A done", 1),
                   ("phase B done", 4), ("end", 5)):
    x = us(t[:, col])
    print(f"{label:20s} mean {x.mean():6.2f}  p10 {np.percentile(x, 10):6.2f}  p90 {np.percentile(x, 90):6.2f}  max {x.max():6.2f}")
