"""Host->device / device->host rates of pinned buffers: one copy vs the same bytes split
over k concurrent streams (several copy engines?), and H2D next to D2H (full duplex?).
Prints microseconds per 1.5 MiB (the C2 step's upload) and 1 MiB (its download)."""
import torch

MB = 1 << 20


def timed(fn, reps=30):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


up_h = torch.randn(3 * MB // 8).pin_memory()   # 1.5 MiB
up_d = torch.empty_like(up_h, device="cuda")
dn_d = torch.randn(MB // 4, device="cuda")     # 1 MiB
dn_h = torch.empty(MB // 4).pin_memory()
streams = [torch.cuda.Stream() for _ in range(4)]
main = torch.cuda.current_stream()


def split_copy(dst, src, k):
    ev = torch.cuda.Event()
    ev.record(main)
    n = src.numel()
    for i in range(k):
        s = streams[i]
        s.wait_event(ev)
        with torch.cuda.stream(s):
            dst[i * n // k:(i + 1) * n // k].copy_(src[i * n // k:(i + 1) * n // k], non_blocking=True)
    for i in range(k):
        main.wait_stream(streams[i])


for k in (1, 2, 4):
    us = timed(lambda: split_copy(up_d, up_h, k))
    print(f"H2D 1.5 MiB in {k} concurrent copies: {us:.1f} us = {1.5 * MB / us / 1e3:.1f} GB/s")
for k in (1, 2, 4):
    us = timed(lambda: split_copy(dn_h, dn_d, k))
    print(f"D2H 1 MiB in {k} concurrent copies: {us:.1f} us = {MB / us / 1e3:.1f} GB/s")


def duplex():
    ev = torch.cuda.Event()
    ev.record(main)
    for s in streams[:2]:
        s.wait_event(ev)
    with torch.cuda.stream(streams[0]):
        up_d.copy_(up_h, non_blocking=True)
    with torch.cuda.stream(streams[1]):
        dn_h.copy_(dn_d, non_blocking=True)
    main.wait_stream(streams[0])
    main.wait_stream(streams[1])


print(f"H2D 1.5 MiB + D2H 1 MiB concurrently: {timed(duplex):.1f} us")
