"""Device timeline of the host-buffer serving step (kvq_cache_step, bench.py's e2e) from CUPTI
activity records (torch.profiler): per step, when each H2D / D2H copy and each kernel ran.
    python tools/e2e_timeline.py [config] [steps]     (KVQ_STEP_CHUNKS selects the chunking)"""
import json
import os
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2502_14882_b200 import kvq  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
N = int(sys.argv[2]) if len(sys.argv) > 2 else 4
B, H, G, n, bits, tau, _ = bench.CONFIGS[cfg]
dev = torch.device("cuda", 0)
k = torch.randn((B, H, n, 128), device=dev)
v = torch.randn((B, H, n, 128), device=dev)
c = kvq.BatchedCache.build_device(k, v, kvq.QuantizationConfig(bits), kvq.CalibrationParams(*tau), group=G)
del k, v
c.reserve_tail(60)
hq = torch.randn((B, H, G, 128)).pin_memory().numpy()
hk = torch.randn((B, H, 128)).pin_memory().numpy()
hv = torch.randn((B, H, 128)).pin_memory().numpy()
hout = torch.empty((B, H, G, 128)).pin_memory().numpy()
for _ in range(20):
    c.step(hq, hk, hv, hout)
walls = []
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA, torch.profiler.ProfilerActivity.CPU]) as prof:
    for _ in range(N):
        t0 = time.perf_counter()
        c.step(hq, hk, hv, hout)
        walls.append((time.perf_counter() - t0) * 1e6)
out = ROOT / "gpurun_out" / f"e2e_timeline_{cfg}.json"
out.parent.mkdir(exist_ok=True)
prof.export_chrome_trace(str(out))
ev = json.loads(out.read_text())["traceEvents"]
dev_ev = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset", "cuda_runtime",
                                                                     "cuda_driver")]
dev_ev.sort(key=lambda e: e["ts"])
print(f"{cfg} chunks={os.environ.get('KVQ_STEP_CHUNKS', 'default')}: host wall per step (us):",
      " ".join(f"{w:.0f}" for w in walls))
# split into steps at each cudaGraphLaunch (host) - the step's host calls and device work
steps, cur = [], []
for e in dev_ev:
    if "GraphLaunch" in e["name"] and cur:
        steps.append(cur)
        cur = []
    cur.append(e)
steps.append(cur)
for i, st in enumerate(steps[-3:]):
    t0 = st[0]["ts"]
    span = max(e["ts"] + e["dur"] for e in st) - t0
    print(f"step {i}: device span {span:.1f} us")
    for e in st:
        name = e["name"][:60]
        print(f"   {e['ts'] - t0:7.1f} +{e['dur']:6.1f}  {e.get('cat'):10s} stream {e.get('args', {}).get('stream', '?')}  {name}")
