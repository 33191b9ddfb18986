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
raw = str(ROOT / "gpurun_out" / f"trace_chain_{cfg}.bin")
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
    c.reserve_tail(TAIL + 4 + (4 * K if os.environ.get('KVQ_TRACE_STEP') == '1' else 0))
    for _ in range(TAIL):
        c.append_device(kn, kn, 0)
q = torch.randn((batch, H, G, 128), device=dev)
out = torch.empty_like(q)
STEP = os.environ.get("KVQ_TRACE_STEP", "0") == "1"  # fused decode + append steps (bench's step)


def one(c):
    if STEP:
        c.step_device(q, out, kn, kn, 0)
    else:
        c.decode_device(q, out, 0)


for i in range(K):  # warm-up chain (also dumped; overwritten below)
    one(caches[i % R])
torch.cuda.synchronize()
for i in range(K):
    one(caches[i % R])
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

# finer breakdown of the last decode (thread 0 of each CTA): slot pairs
rows = t[K - 1][t[K - 1][:, 0] > 0]
names = {0: "start", 6: "tmem alloc", 7: "stats ld", 3: "dep wait", 24: "q fold", 25: "sync1", 26: "digits",
         2: "prologue", 8: "phase A (w0)", 27: "tail scores", 30: "partials", 1: "params", 16: "phase B (w0)",
         28: "image", 29: "output sums", 5: "end"}
order = [0, 6, 7, 3, 24, 25, 26, 2, 8, 27, 30, 1, 16, 28, 29, 5]
print("last decode, mean per step (us):")
prev = None
for k in order:
    x = rows[:, k]
    if (x > 0).all():
        if prev is not None:
            print(f"  {names[prev]:>13s} -> {names[k]:<13s} {np.mean(x - rows[:, prev]) / 1e3:6.2f}")
        prev = k

# per-SM load of the last decode: CTAs per SM and the SM's last end
sm = rows[:, 31] - 1
end = (rows[:, 5] - t0) / 1e3
from collections import Counter
per = {}
for i in range(len(rows)):
    per.setdefault(int(sm[i]), []).append((i, end[i]))
ends = sorted((max(e for _, e in v), k, len(v)) for k, v in per.items())
cnt = Counter(len(v) for v in per.values())
print("CTAs per SM:", dict(cnt), " SMs used:", len(per))
print("latest SMs (end us, sm, ctas, cta ids):")
for e, k, nn in ends[-6:]:
    print(f"  {e:7.1f} sm {k:3d} ctas {nn} ids {[i for i, _ in per[k]]}")
print("earliest SMs:")
for e, k, nn in ends[:4]:
    print(f"  {e:7.1f} sm {k:3d} ctas {nn} ids {[i for i, _ in per[k]]}")

# warp imbalance inside a CTA (last decode): spread of the per-warp phase A / phase B ends
pa = rows[:, 8:16].astype(np.float64)
pb = rows[:, 16:24].astype(np.float64)
pa[pa == 0] = np.nan
pb[pb == 0] = np.nan
sa = (np.nanmax(pa, 1) - np.nanmin(pa, 1)) / 1e3
sb = (np.nanmax(pb, 1) - np.nanmin(pb, 1)) / 1e3
print(f"warp spread in a CTA (us): phase A end mean {np.nanmean(sa):.2f} p90 {np.nanpercentile(sa, 90):.2f}; "
      f"phase B end mean {np.nanmean(sb):.2f} p90 {np.nanpercentile(sb, 90):.2f}")
