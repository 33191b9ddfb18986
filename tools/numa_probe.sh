#!/bin/bash
mkdir -p gpurun_out
{ nvidia-smi topo -m; lscpu | grep -iE "numa|socket|model name"; cat /sys/bus/pci/devices/*/numa_node 2>/dev/null | sort | uniq -c; } > gpurun_out/numa.txt 2>&1
python - >> gpurun_out/numa.txt 2>&1 <<'PY'
import os, pynvml, torch
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
mask = pynvml.nvmlDeviceGetCpuAffinity(h, 8)
cpus = [i for w, m in enumerate(mask) for i in range(64) if (m >> i) & 1 for i in [w * 64 + i]]
print("gpu-local cpus:", cpus[:8], "...", len(cpus), "of", os.cpu_count())
def h2d(label):
    n = 1 << 20
    host = torch.randn(n // 4).pin_memory(); dev = torch.empty(n // 4, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3): dev.copy_(host, non_blocking=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(20): dev.copy_(host, non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    print(label, "H2D 1 MiB %.1f us" % (e0.elapsed_time(e1) / 20 * 1e3))
h2d("default affinity")
allc = set(range(os.cpu_count()))
os.sched_setaffinity(0, set(cpus) & allc)
h2d("gpu-local affinity")
other = allc - set(cpus)
if other:
    os.sched_setaffinity(0, other)
    h2d("remote affinity")
PY
