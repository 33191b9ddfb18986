"""Tiny tensor-core decode run (debug helper): one cache, one decode, sync."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2502_14882_b200 import kvq
B, H, G, n = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (1, 1, 4, 600)))
rng = np.random.default_rng(0)
k = rng.normal(size=(B, H, n, 128)).astype(np.float32)
v = rng.normal(size=(B, H, n, 128)).astype(np.float32)
c = kvq.BatchedCache.build(k, v, kvq.QuantizationConfig(1), kvq.CalibrationParams(1, 0), group=G)
c.set_path(kvq.PATH_TC)
out, _, _ = c.decode(rng.normal(size=(B, H, G, 128)).astype(np.float32))
print("ok", float(np.abs(out).sum()))
