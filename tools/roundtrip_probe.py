"""Why does one synchronous step cost far more than the step's device time?
    python tools/roundtrip_probe.py [config]
(a) tiny kernel + sync round trip; (b) one step graph + sync (wall); (c) the same step's
device time from events inside the replay stream (isolated, GPU idle before); (d) ten
steps back to back + one sync (per step)."""
import sys
import time
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
N = 200
c.reserve_tail(60)  # in-kernel tail (<= 64 rows)
q = torch.randn((B, H, G, 128), device=dev)
kn = torch.randn((B, H, 128), device=dev)
out = torch.empty_like(q)
s = torch.cuda.Stream()
c.step_device(q, out, kn, kn, s.cuda_stream)
s.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    c.step_device(q, out, kn, kn, s.cuda_stream)
x = torch.zeros(16, device=dev)


def wall(fn, reps=N):
    for _ in range(20):
        fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t0) / reps * 1e6


def tiny():
    with torch.cuda.stream(s):
        x.add_(1.0)
    s.synchronize()


def one():
    with torch.cuda.stream(s):
        g.replay()
    s.synchronize()


def ten():
    with torch.cuda.stream(s):
        for _ in range(10):
            g.replay()
    s.synchronize()


print(f"{cfg}: tiny kernel + sync {wall(tiny):.1f} us")
print(f"{cfg}: one step graph + sync {wall(one):.1f} us (wall)")
ev = []
for _ in range(50):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        g.replay()
        e1.record(s)
    s.synchronize()
    ev.append(e0.elapsed_time(e1) * 1e3)
ev.sort()
print(f"{cfg}: one step, device time between events (isolated) median {ev[len(ev) // 2]:.1f} us")
print(f"{cfg}: ten steps + one sync {wall(ten, N // 10) / 10:.1f} us per step")
t0 = time.perf_counter()
for _ in range(200):
    with torch.cuda.stream(s):
        g.replay()
t1 = time.perf_counter()
s.synchronize()
print(f"{cfg}: host cost of graph.replay() {(t1 - t0) / 200 * 1e6:.1f} us")

# a synchronous host-buffer step replayed by hand on one stream with events between the parts
hq = torch.randn((B, H, G, 128)).pin_memory()
hk = torch.randn((B, H, 128)).pin_memory()
hout = torch.empty((B, H, G, 128)).pin_memory()
dk = torch.empty_like(kn)
parts = []
for _ in range(60):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    with torch.cuda.stream(s):
        ev[0].record(s)
        q.copy_(hq, non_blocking=True)
        kn.copy_(hk, non_blocking=True)
        dk.copy_(hk, non_blocking=True)
        ev[1].record(s)
        c.step_device(q, out, kn, dk, s.cuda_stream)
        ev[2].record(s)
        hout.copy_(out, non_blocking=True)
        ev[3].record(s)
    s.synchronize()
    parts.append([ev[i].elapsed_time(ev[i + 1]) * 1e3 for i in range(3)])
parts.sort(key=lambda p: sum(p))
p = parts[len(parts) // 2]
print(f"{cfg}: serial host-buffer step on one stream: H2D {p[0]:.1f} us, step kernel {p[1]:.1f} us, D2H {p[2]:.1f} us")
