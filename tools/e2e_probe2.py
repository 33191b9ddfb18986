"""Step API with pinned vs pageable host buffers (KVQ_STEP_TRACE timelines on stderr)."""
import sys
import time

import numpy as np
import torch

from paper_2502_14882_b200 import kvq

B, H, G, n, d = 64, 8, 4, 4096, 128
k = torch.randn((B, H, n, d), device="cuda")
v = torch.randn((B, H, n, d), device="cuda")
c = kvq.BatchedCache.build_device(k, v, kvq.QuantizationConfig(1), kvq.CalibrationParams(1, 0), group=G)
c.reserve_tail(4096)
del k, v
kinds = {}
tq = torch.randn((B, H, G, d)).pin_memory()
tk = torch.randn((B, H, d)).pin_memory()
tv = torch.randn((B, H, d)).pin_memory()
to = torch.empty((B, H, G, d)).pin_memory()
kinds["torch_pinned"] = (tq.numpy(), tk.numpy(), tv.numpy(), to.numpy())
kinds["pageable"] = (np.random.rand(B, H, G, d).astype(np.float32), np.random.rand(B, H, d).astype(np.float32),
                     np.random.rand(B, H, d).astype(np.float32), np.empty((B, H, G, d), np.float32))
for name, (hq, hk, hv, ho) in kinds.items():
    for _ in range(5):
        c.step(hq, hk, hv, ho)
    ts = []
    print(f"--- {name}", file=sys.stderr, flush=True)
    for _ in range(30):
        t0 = time.perf_counter()
        c.step(hq, hk, hv, ho)
        ts.append(time.perf_counter() - t0)
    print(name, "step wall median %.1f us" % (np.median(ts) * 1e6), flush=True)
