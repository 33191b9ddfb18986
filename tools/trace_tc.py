"""Per-CTA timeline of one IMMA decode launch (KVQ_TRACE_FILE stamps, k2_decode_tc.cu).
python tools/trace_tc.py [config] [path id, default 2 = tc]"""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
raw = str(ROOT / "gpurun_out" / "trace_tc.bin")
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
c.set_path(int(sys.argv[2]) if len(sys.argv) > 2 else 2)
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
pa = t[:, 8:16].max(1)
pb = t[:, 16:24].max(1)
rows = [("start->griddep released", t[:, 3] - t[:, 0]), ("griddep->prologue done", t[:, 2] - t[:, 3])]
if (t[:, 24] > 0).all():
    rows += [("  q loads+reductions", t[:, 24] - t[:, 3]), ("  sync 1", t[:, 25] - t[:, 24]),
             ("  frag build", t[:, 26] - t[:, 25]), ("  sync 2 + bq", t[:, 2] - t[:, 26])]
pa_w = np.where(t[:, 8:16] > 0, t[:, 8:16], t[:, 2:3])
for name, d in rows + [
                ("prologue->phase A done", pa - t[:, 2]), ("start->phase A done (slowest warp)", pa - t[:, 0]), ("phase A warp spread", pa_w.max(1) - pa_w.min(1)),
                ("phaseA done->params", t[:, 1] - pa), ("phase B (params->slowest warp)", pb - t[:, 1]),
                ("epilogue", t[:, 5] - pb), ("CTA total", t[:, 5] - t[:, 0])]:
    d = d / 1e3
    print(f"{name:36s} mean {d.mean():6.2f} us  p10 {np.percentile(d, 10):6.2f}  p90 {np.percentile(d, 90):6.2f}")
st = us(t[:, 0])
print(f"CTA start: min {st.min():.2f} p50 {np.median(st):.2f} max {st.max():.2f} us")
grid = np.linspace(0, us(t[:, 5].max()), 40)
print("CTAs alive:", " ".join(str(int(((us(t[:, 0]) <= g) & (us(t[:, 5]) >= g)).sum())) for g in grid))
