"""Time the K2 decode launch (prep + decode) in isolation with CUDA events, per path:
same replica repeated (L2-warm) vs rotating over replicas larger than L2 (cold)."""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2502_14882_b200 import kvq  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
batch, H, G, n, bits, tau, _ = bench.CONFIGS[cfg]
dev = torch.device("cuda", 0)
R = max(2, -(-3 * bench.L2_BYTES // (batch * H * 2 * n * 128 * bits // 8)))
k = torch.randn((batch, H, n, 128), device=dev)
v = torch.randn((batch, H, n, 128), device=dev)
caches = [kvq.BatchedCache.build_device(k, v, kvq.QuantizationConfig(bits), kvq.CalibrationParams(*tau), group=G)
          for _ in range(R)]
del k, v
q = torch.randn((batch, H, G, 128), device=dev)
out = torch.empty_like(q)
s = torch.cuda.Stream()
for path_name, path in (("tc", 2), ("umma", 3)):
    for c in caches:
        c.set_path(path)
    for mode in ("same", "rotate"):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(40)]
        for i in range(10):
            caches[i % R].decode_device(q, out, s.cuda_stream)
        for i, (a, b) in enumerate(evs):
            c = caches[0] if mode == "same" else caches[i % R]
            a.record(s)
            c.decode_device(q, out, s.cuda_stream)
            b.record(s)
        s.synchronize()
        ts = sorted(a.elapsed_time(b) * 1e3 for a, b in evs)
        print(f"{cfg} {path_name:5s} {mode:6s}: median {ts[len(ts)//2]:.1f} us  min {ts[0]:.1f} us  ({R} replicas)")
