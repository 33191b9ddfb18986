"""Quick ws-path probe: one decode at a given shape through KVQ_PATH_WS, vs the tc path."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2502_14882_b200 import kvq  # noqa: E402

B, H, G, n, bits = (int(x) for x in sys.argv[1:6])
path = int(sys.argv[6]) if len(sys.argv) > 6 else 5
dev = torch.device("cuda", 0)
k = torch.randn((B, H, n, 128), device=dev)
v = torch.randn((B, H, n, 128), device=dev)
c = kvq.BatchedCache.build_device(k, v, kvq.QuantizationConfig(bits), kvq.CalibrationParams(1.0, 0.0), group=G)
q = torch.randn((B, H, G, 128), device=dev)
o1 = torch.empty_like(q)
o2 = torch.empty_like(q)
c.set_path(2)
c.decode_device(q, o1)
torch.cuda.synchronize()
print("tc done", flush=True)
c.set_path(path)
t0 = time.time()
c.decode_device(q, o2)
torch.cuda.synchronize()
print("path", path, "done in", time.time() - t0, flush=True)
err = ((o1 - o2).norm() / o1.norm()).item()
print("rel diff vs tc", err, flush=True)
