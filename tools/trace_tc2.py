"""Timeline of both grids of the balanced IMMA decode (KVQ_TRACE_FILE): per grid the CTA
start / phase-A end / phase-B end / end distribution.  python tools/trace_tc2.py [config]"""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
raw = str(ROOT / "gpurun_out" / "trace_tc2.bin")
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
c.set_path(2)
q = torch.randn((batch, H, G, 128), device=dev)
out = torch.empty_like(q)
for _ in range(3):
    c.decode_device(q, out, 0)
torch.cuda.synchronize()
t = np.fromfile(raw, dtype=np.uint64).reshape(-1, 256).astype(np.int64)
used = t[:, 0] > 0
t0 = t[used, 0].min()
us = lambda x: (x - t0) / 1e3
units_split = 68 if cfg == "c2" else 0
nA = batch * H - units_split
print(f"{cfg}: {used.sum()} CTAs traced, span {us(t[used, 5].max()):.1f} us")
for name, rows in (("grid A (whole units)", t[:nA]), ("grid B (half units)", t[nA:][t[nA:, 0] > 0])):
    if not len(rows):
        continue
    pa, pb = rows[:, 8:16].max(1), rows[:, 16:24].max(1)
    for label, x in (("start", rows[:, 0]), ("prologue done", rows[:, 2]), ("phase A done", pa), ("params", rows[:, 1]),
                     ("phase B done", pb), ("end", rows[:, 5])):
        v = us(x[x > 0])
        print(f"{name:22s} {label:14s} mean {v.mean():6.2f}  p10 {np.percentile(v, 10):6.2f}  p90 {np.percentile(v, 90):6.2f}  max {v.max():6.2f}")
