"""Where does the host-buffer step (kvq_cache_step, bench.py's e2e) spend its time?
    python tools/e2e_probe4.py [config] [steps]
Prints wall microseconds per step for: the real step; the step's copies alone (same
streams/pattern through torch, no kernels); a device-only step (step_device graph, synced
per step - launch + sync overhead with no copies). KVQ_STEP_CHUNKS selects the chunking."""
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2502_14882_b200 import kvq  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40  # <= 50 host steps: the fp32 tail stays in-kernel
B, H, G, n, bits, tau, _ = bench.CONFIGS[cfg]
dev = torch.device("cuda", 0)
k = torch.randn((B, H, n, 128), device=dev)
v = torch.randn((B, H, n, 128), device=dev)
c = kvq.BatchedCache.build_device(k, v, kvq.QuantizationConfig(bits), kvq.CalibrationParams(*tau), group=G)
del k, v
c.reserve_tail(60)  # in-kernel tail; kvq_cache_step grows it (host counter) - keep N small
hq = torch.randn((B, H, G, 128)).pin_memory().numpy()
hk = torch.randn((B, H, 128)).pin_memory().numpy()
hv = torch.randn((B, H, 128)).pin_memory().numpy()
hout = torch.empty((B, H, G, 128)).pin_memory().numpy()


def wall(fn, reps=N, warm=10):
    for _ in range(warm):
        fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t0) / reps * 1e6


chunks = os.environ.get("KVQ_STEP_CHUNKS", "default")
print(f"{cfg} chunks={chunks}: step {wall(lambda: c.step(hq, hk, hv, hout)):.1f} us")

# copies alone, same volume: q + k + v up (one stream), out down (another), one sync
tq, tk, tv, to = (torch.from_numpy(x) for x in (hq, hk, hv, hout))
dq, dk, dv = tq.to(dev), tk.to(dev), tv.to(dev)
do = torch.empty_like(dq)
s_up, s_dn = torch.cuda.Stream(), torch.cuda.Stream()


def copies():
    with torch.cuda.stream(s_up):
        dq.copy_(tq, non_blocking=True)
        dk.copy_(tk, non_blocking=True)
        dv.copy_(tv, non_blocking=True)
    with torch.cuda.stream(s_dn):
        to.copy_(do, non_blocking=True)
    s_up.synchronize()
    s_dn.synchronize()


print(f"{cfg}: copies alone (up {hq.nbytes + hk.nbytes + hv.nbytes} B || down {hout.nbytes} B) {wall(copies):.1f} us")

s = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
c.step_device(dq, do, dk, dv, s.cuda_stream)
s.synchronize()
with torch.cuda.graph(g, stream=s):
    c.step_device(dq, do, dk, dv, s.cuda_stream)


def dev_step():
    g.replay()
    torch.cuda.current_stream().synchronize()


print(f"{cfg}: device step graph, synced per step {wall(dev_step):.1f} us")
