"""Does the host<->device copy rate ramp up under sustained traffic (PCIe link power
states)? Times a 1.5 MiB pinned H2D copy in consecutive 50 ms windows after an idle second,
then the same with a 1 MiB D2H copy.  python tools/pcie_ramp.py"""
import time

import torch

MB = 1 << 20
up_h = torch.randn(3 * MB // 8).pin_memory()
up_d = torch.empty_like(up_h, device="cuda")
dn_d = torch.randn(MB // 4, device="cuda")
dn_h = torch.empty(MB // 4).pin_memory()


def windows(fn, label, n=16, span=0.05):
    torch.cuda.synchronize()
    time.sleep(1.0)  # idle: let the link drop to its idle state
    out = []
    for _ in range(n):
        t0 = time.perf_counter()
        k = 0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        while time.perf_counter() - t0 < span:
            for _ in range(8):
                fn()
            k += 8
            torch.cuda.synchronize()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) * 1e3 / k)
    print(label, " ".join(f"{x:.0f}" for x in out), "us per copy (50 ms windows)")


windows(lambda: up_d.copy_(up_h, non_blocking=True), "H2D 1.5 MiB:")
windows(lambda: dn_h.copy_(dn_d, non_blocking=True), "D2H 1 MiB:  ")
