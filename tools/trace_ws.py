"""Per-unit timeline of the persistent ws decode (KVQ_TRACE_FILE stamps, k2_decode_ws.cu):
score warp 0 finishing phase A of unit k (slot 8 + 2k) and value warp 0 finishing unit k
(slot 24 + k).  python tools/trace_ws.py [config]"""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
raw = str(ROOT / "gpurun_out" / "trace_ws.bin")
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
c.set_path(5)
q = torch.randn((batch, H, G, 128), device=dev)
out = torch.empty_like(q)
for _ in range(3):
    c.decode_device(q, out, 0)
torch.cuda.synchronize()
t = np.fromfile(raw, dtype=np.uint64).reshape(-1, 256).astype(np.int64)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
us = lambda x: (x - t0) / 1e3
print(f"{cfg}: {len(t)} CTAs, span {us(t[:, 5].max()):.1f} us, griddep released {np.mean(us(t[:, 3])):.2f} us")
for kk in range(8):
    a_done, b_done = t[:, 8 + 2 * kk], t[:, 24 + kk]
    m = (a_done > 0) & (b_done > 0)
    if not m.any():
        break
    print(f"unit {kk}: score warps done {np.mean(us(a_done[m])):6.2f} us (p90 {np.percentile(us(a_done[m]), 90):6.2f}) | "
          f"value warps done {np.mean(us(b_done[m])):6.2f} us (p90 {np.percentile(us(b_done[m]), 90):6.2f})  [{m.sum()} CTAs]")

print("score warp 0 per unit: prologue | freed wait | phase A   ||  value warp 0: wait ready | phase B | reduce+bar | epilogue")
for kk in range(8):
    s0, s1, s2, s3 = (t[:, 40 + 4 * kk + i] for i in range(4))
    v0, v1, v2 = (t[:, 80 + 4 * kk + i] for i in range(3))
    v3 = t[:, 24 + kk]
    m = (s0 > 0) & (s3 > 0) & (v0 > 0) & (v3 > 0)
    if not m.any():
        break
    d = lambda a, b: np.mean((b[m] - a[m]) / 1e3)
    vprev = t[:, 24 + kk - 1][m] if kk else t[:, 3][m]
    print(f"unit {kk}: {d(s0, s1):5.2f} | {d(s1, s2):5.2f} | {d(s2, s3):5.2f}  ||  "
          f"{np.mean((v0[m] - vprev) / 1e3):5.2f} | {d(v0, v1):5.2f} | {d(v1, v2):5.2f} | {d(v2, v3):5.2f}")
