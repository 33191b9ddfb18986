"""Device time of ONE decode (or step) graph launched alone (GPU idle before, events around
it) vs back-to-back launches of the same 1-step graph vs a graph of 10 steps.
    python tools/isolated_probe.py [config]     (env switches select the variant)"""
import os
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2502_14882_b200 import kvq  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
B, H, G, n, bits, tau, _ = bench.CONFIGS[cfg]
dev = torch.device("cuda", 0)
k = torch.randn((B, H, n, 128), device=dev)
v = torch.randn((B, H, n, 128), device=dev)
c = kvq.BatchedCache.build_device(k, v, kvq.QuantizationConfig(bits), kvq.CalibrationParams(*tau), group=G)
del k, v
c.reserve_tail(60)  # in-kernel tail (<= 64 rows); replays past it drop appends (overflow flag), timing unaffected
q = torch.randn((B, H, G, 128), device=dev)
kn = torch.randn((B, H, 128), device=dev)
out = torch.empty_like(q)
s = torch.cuda.Stream()
x = torch.zeros(16, device=dev)


def graph(fn, count=1):
    fn()
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(count):
            fn()
    return g


def ev_time(g, per=1, reps=40):
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            g.replay()
            e1.record(s)
        s.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / per)
    ts.sort()
    return ts[len(ts) // 2]


def b2b(g, count=10, per=1):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        g.replay()
        e0.record(s)
        for _ in range(count):
            g.replay()
        e1.record(s)
    s.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (count * per)


tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("KVQ_")) or "default"
with torch.cuda.stream(s):
    g_tiny = graph(lambda: x.add_(1.0))
    g_dec = graph(lambda: c.decode_device(q, out, s.cuda_stream))
    g_step = graph(lambda: c.step_device(q, out, kn, kn, s.cuda_stream))
    g_dec10 = graph(lambda: c.decode_device(q, out, s.cuda_stream), 10)
print(f"[{tag}] {cfg}: tiny graph alone {ev_time(g_tiny):.1f} us | decode graph alone {ev_time(g_dec):.1f} us, "
      f"b2b {b2b(g_dec):.1f} | step graph alone {ev_time(g_step):.1f}, b2b {b2b(g_step):.1f} | "
      f"10-decode graph {ev_time(g_dec10, 10):.1f} us per decode")
