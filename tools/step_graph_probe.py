"""c2 step time: [decode graph][append graph] replays vs one fused [decode + append] graph
per replica (programmatic dependent launch edges live inside a graph)."""
import torch

from paper_2502_14882_b200 import kvq

B, H, G, n, d, R = 64, 8, 4, 4096, 128, 12
dev = torch.device("cuda")
st = torch.cuda.Stream()
sp = st.cuda_stream
with torch.cuda.stream(st):
    k = torch.randn((B, H, n, d), device=dev)
    v = torch.randn((B, H, n, d), device=dev)
    caches = []
    for r in range(R):
        c = kvq.BatchedCache.build_device(k, v, kvq.QuantizationConfig(1), kvq.CalibrationParams(1, 0), group=G,
                                          stream=sp)
        c.reserve_tail(60)
        caches.append(c)
    del k, v
    q = torch.randn((B, H, G, d), device=dev)
    kn = torch.randn((B, H, d), device=dev)
    vn = torch.randn((B, H, d), device=dev)
    out = torch.empty_like(q)
st.synchronize()
for c in caches:
    c.decode_device(q, out, sp)
    c.append_device(kn, vn, sp)
st.synchronize()
split, fused = [], []
for c in caches:
    gd, ga, gf = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    with torch.cuda.graph(gd, stream=st):
        c.decode_device(q, out, sp)
    with torch.cuda.graph(ga, stream=st):
        c.append_device(kn, vn, sp)
    with torch.cuda.graph(gf, stream=st):
        c.decode_device(q, out, sp)
        c.append_device(kn, vn, sp)
    split.append((gd, ga))
    fused.append(gf)


def run(kind, steps=24):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    with torch.cuda.stream(st):
        torch.cuda._sleep(int(2e7))
        e0.record(st)
        for i in range(steps):
            if kind == "split":
                split[i % R][0].replay()
                split[i % R][1].replay()
            else:
                fused[i % R].replay()
        e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps * 1e3


def run_dec(steps=24):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    with torch.cuda.stream(st):
        torch.cuda._sleep(int(2e7))
        e0.record(st)
        for i in range(steps):
            split[i % R][0].replay()
        e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps * 1e3


for rep in range(2):
    print("split %.1f us/step, fused %.1f us/step, decode only %.1f us" % (run("split"), run("fused"), run_dec()))
