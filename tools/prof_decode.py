"""One decode at a BASELINE config's exact geometry inside an NVTX range "profile" (for
ncu --nvtx --nvtx-include profile/): the cache built on the device as bench.py builds it,
three fp32 tail rows appended, two warm-up decodes, then the profiled one.
    python tools/prof_decode.py <config> [path]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2502_14882_b200 import kvq  # noqa: E402

cfg = sys.argv[1]
batch, H, G, n, bits, tau, _, path, _ = bench.resolve_config(cfg)
path = sys.argv[2] if len(sys.argv) > 2 else (path or "auto")
dev = torch.device("cuda", 0)
k = torch.randn((batch, H, n, bench.DIM), device=dev)
v = torch.randn((batch, H, n, bench.DIM), device=dev)
c = kvq.BatchedCache.build_device(k, v, kvq.QuantizationConfig(bits), kvq.CalibrationParams(*tau), group=G)
del k, v
c.reserve_tail(bench.TAIL_WINDOW + 8)
c.set_path(bench.PATHS[path])
for _ in range(3):
    c.append_device(torch.randn((batch, H, bench.DIM), device=dev), torch.randn((batch, H, bench.DIM), device=dev))
q = torch.randn((batch, H, G, bench.DIM), device=dev)
out = torch.empty_like(q)
for _ in range(2):
    c.decode_device(q, out)
torch.cuda.synchronize()
l0 = kvq.launch_count()
torch.cuda.nvtx.range_push("profile")
c.decode_device(q, out)
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print(f"{cfg}: {kvq.launch_count() - l0} kernel launches in the profiled decode", flush=True)
