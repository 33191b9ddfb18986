"""H2D of a torch-pinned buffer: torch copy_ vs raw cudaMemcpyAsync, default vs
non-blocking streams (is the slow step upload a stream / engine effect?)."""
import ctypes as C

import torch

rt = C.CDLL("libcudart.so.12")
n = 1 << 20
host = torch.randn(n // 4).pin_memory()
dev = torch.empty(n // 4, device="cuda")


def t_copy(fn, stream, reps=20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        fn()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for label, stream in (("default", torch.cuda.default_stream()), ("side", torch.cuda.Stream())):
    torch_us = t_copy(lambda: dev.copy_(host, non_blocking=True), stream)
    raw = lambda: rt.cudaMemcpyAsync(C.c_void_p(dev.data_ptr()), C.c_void_p(host.data_ptr()), C.c_size_t(n), 1,
                                     C.c_void_p(stream.cuda_stream))
    raw_us = t_copy(raw, stream)
    one = []
    for _ in range(10):  # single copies, synchronised in between (the step's pattern)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        raw()
        e1.record(stream)
        torch.cuda.synchronize()
        one.append(e0.elapsed_time(e1) * 1e3)
    print(f"{label}: torch copy_ {torch_us:.1f} us, cudaMemcpyAsync {raw_us:.1f} us, single synced copies "
          f"{sorted(one)[len(one)//2]:.1f} us (median)")
