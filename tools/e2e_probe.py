"""Where the e2e step time goes (c2 shape): PCIe copy rates for the step's buffers, the
step API's wall time, and the host-side issue time of its calls."""
import time

import numpy as np
import torch

from paper_2502_14882_b200 import kvq


def timed_copy(nbytes, h2d, reps=50):
    host = torch.empty(nbytes // 4, dtype=torch.float32).pin_memory()
    dev = torch.empty(nbytes // 4, dtype=torch.float32, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        (dev.copy_(host, non_blocking=True) if h2d else host.copy_(dev, non_blocking=True))
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        (dev.copy_(host, non_blocking=True) if h2d else host.copy_(dev, non_blocking=True))
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / reps * 1e3
    return us, nbytes / us / 1e3


for mb in (0.25, 0.5, 1.0, 1.5):
    n = int(mb * 2**20)
    print(f"H2D {mb} MiB: %.1f us (%.1f GB/s)" % timed_copy(n, True), f" D2H: %.1f us (%.1f GB/s)" % timed_copy(n, False))

B, H, G, n, d = 64, 8, 4, 4096, 128
k = torch.randn((B, H, n, d), device="cuda")
v = torch.randn((B, H, n, d), device="cuda")
c = kvq.BatchedCache.build_device(k, v, kvq.QuantizationConfig(1), kvq.CalibrationParams(1, 0), group=G)
c.reserve_tail(2048)
del k, v
hq = torch.randn((B, H, G, d)).pin_memory().numpy()
hk = torch.randn((B, H, d)).pin_memory().numpy()
hv = torch.randn((B, H, d)).pin_memory().numpy()
ho = torch.empty((B, H, G, d)).pin_memory().numpy()
for _ in range(10):
    c.step(hq, hk, hv, ho)
ts = []
for _ in range(200):
    t0 = time.perf_counter()
    c.step(hq, hk, hv, ho)
    ts.append(time.perf_counter() - t0)
print("step wall: median %.1f us, p10 %.1f, p90 %.1f" % tuple(np.percentile(ts, [50, 10, 90]) * 1e6))
q = torch.from_numpy(hq).cuda()
out = torch.empty_like(q)
torch.cuda.synchronize()
ts = []
for _ in range(200):
    t0 = time.perf_counter()
    c.decode_device(q, out, torch.cuda.current_stream().cuda_stream)
    ts.append(time.perf_counter() - t0)
torch.cuda.synchronize()
print("decode_device host issue: median %.1f us" % (np.median(ts) * 1e6))
