"""K1 prefill (stats + codes, kvq_quantize_device) per GiB of fp32 input at a BASELINE
shape, plus a hash of codes / stats to compare variants bit for bit (KVQ_K1_CHUNK_MB: the
chunked stats / codes pipeline, read once per process).
    python tools/k1_time.py [units] [n] [bits] [mode]"""
import ctypes as C
import hashlib
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2502_14882_b200 import kvq  # noqa: E402

U = int(sys.argv[1]) if len(sys.argv) > 1 else 512
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
bits = int(sys.argv[3]) if len(sys.argv) > 3 else 1
mode = int(sys.argv[4]) if len(sys.argv) > 4 else 0
d = 128
g = torch.Generator(device="cuda")
g.manual_seed(3)
x = torch.randn((U, n, d), device="cuda", generator=g)
codes = torch.empty(U * n * 16 * bits, dtype=torch.uint8, device="cuda")
a = torch.empty((U, d), device="cuda")
b = torch.empty((U, d), device="cuda")
L = kvq.lib()
st = torch.cuda.current_stream()
call = lambda: kvq._check(L.kvq_quantize_device(x.data_ptr(), U, n, d, bits, mode, 8, codes.data_ptr(), a.data_ptr(),
                                                b.data_ptr(), st.cuda_stream))
for _ in range(3):
    call()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 10
e0.record()
for _ in range(reps):
    call()
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / reps
gib = x.numel() * 4 / 2**30
h = hashlib.sha1(codes.cpu().numpy().tobytes() + a.cpu().numpy().tobytes() + b.cpu().numpy().tobytes()).hexdigest()[:16]
print(f"chunk_mb={os.environ.get('KVQ_K1_CHUNK_MB', 'default')} U={U} n={n} b={bits} mode={mode}: {us:.1f} us "
      f"({us / gib:.1f} us/GiB, {x.numel() * 4 / us / 1e6:.2f} TB/s read-once) sha={h}")
