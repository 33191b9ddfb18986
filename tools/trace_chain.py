"""Timeline of k back-to-back IMMA decodes (KVQ_TRACE_CHAIN): per decode the CTA start,
dependency release, prologue, phase A/B and end distributions on one clock, so the gap
between consecutive decodes is visible.  python tools/trace_chain.py [config] [k] [replicas] [tail rows]"""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 4
(ROOT / "gpurun_out").mkdir(exist_ok=True)
raw = str(ROOT / "gpurun_out" / "trace_chain.bin")
os.environ["KVQ_TRACE_FILE"] = raw
os.environ["KVQ_TRACE_CHAIN"] = str(K)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2502_14882_b200 import kvq  # noqa: E402

batch, H, G, n, bits, tau, _ = bench.CONFIGS[cfg]
dev = torch.device("cuda", 0)
k = torch.randn((batch, H, n, 128), device=dev)
v = torch.randn((batch, H, n, 128), device=dev)
R = int(sys.argv[3]) if len(sys.argv) > 3 else 1  # caches cycled through (R >= 3 defeats the L2)
caches = [kvq.BatchedCache.build_device(k, v, kvq.QuantizationConfig(bits), kvq.CalibrationParams(*tau), group=G)
          for _ in range(R)]
TAIL = int(sys.argv[4]) if len(sys.argv) > 4 else 0  # fp32 tail rows appended first
kn = torch.randn((batch, H, 128), device=dev)
for c in caches:
    c.set_path(2)
    c.reserve_tail(TAIL + 4)
    for _ in range(TAIL):
        c.append_device(kn, kn, 0)
q = torch.randn((batch, H, G, 128), device=dev)
out = torch.empty_like(q)
for i in range(K):  # warm-up chain (also dumped; overwritten below)
    caches[i % R].decode_device(q, out, 0)
torch.cuda.synchronize()
for i in range(K):
    caches[i % R].decode_device(q, out, 0)
torch.cuda.synchronize()
t = np.fromfile(raw, dtype=np.uint64).reshape(K, -1, 256).astype(np.int64)
t0 = t[0][t[0][:, 0] > 0, 0].min()
us = lambda x: (x - t0) / 1e3
print(f"{cfg}: {K} chained decodes, times in us from the first CTA start")
for i in range(K):
    rows = t[i][t[i][:, 0] > 0]
    pa, pb = rows[:, 8:16].max(1), rows[:, 16:24].max(1)
    line = [f"decode {i}: {len(rows)} CTAs"]
    for label, x in (("start", rows[:, 0]), ("dep", rows[:, 3]), ("prol", rows[:, 2]), ("A", pa), ("params", rows[:, 1]),
                     ("B", pb), ("end", rows[:, 5])):
        x = x[x > 0]
        if len(x):
            line.append(f"{label} {us(x.min()):6.1f}/{us(x.mean()):6.1f}/{us(x.max()):6.1f}")
    print("  ".join(line))
