"""The step entry point (decode_step then append, kvq_main.cpp:313-321 order) with the append
fused into the tensor-core decode (kvq_cache_step_device):

  * bit-identical outputs and tails against the unfused sequence decode_device +
    append_device (k3_append.cu) over several steps, at every launch geometry the decode
    plans: solo CTAs, split clusters (small batches), the balanced mixed launch (4-warp CTAs
    with half-unit clusters) and the head-group split (G > 4, two CTAs per unit);
  * under CUDA-graph replay past the reserved tail, the fused append drops rows and reports
    the overflow like the append kernel (kvcache.hpp:99-109 semantics, no corruption);
  * tail_len moves on once per request: every unit of a request decodes against the same
    tail length.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GEOMETRIES = [  # (batch, kv_heads, group, n_vis, bits): what plan() picks
    (2, 2, 4, 256, 1),     # split clusters (S = ceil(128 / units))
    (1, 2, 6, 2048, 1),    # head-group split, clusters
    (40, 8, 4, 1024, 1),   # 320 units: 4-warp CTAs, balanced mixed launch (whole + half units)
    (20, 8, 4, 4096, 2),   # 160 units of 4096 tokens: 8-warp solo CTAs
    (8, 8, 6, 1024, 4),    # 64 units x 2 head groups
]


def _pair(kvq, torch, B, H, G, n, bits, reserve=12):
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev)
    gen.manual_seed(11)
    k = torch.randn((B, H, n, 128), device=dev, generator=gen)
    v = torch.randn((B, H, n, 128), device=dev, generator=gen)
    mk = lambda: kvq.BatchedCache.build_device(k, v, kvq.QuantizationConfig(bits), kvq.CalibrationParams(1.0, 0.0),
                                               group=G)
    a, b = mk(), mk()
    for c in (a, b):
        c.reserve_tail(reserve)
    return a, b, dev


@pytest.mark.parametrize("B,H,G,n,bits", GEOMETRIES)
def test_fused_step_matches_decode_then_append(kvq, B, H, G, n, bits):
    torch = pytest.importorskip("torch")
    fused, plain, dev = _pair(kvq, torch, B, H, G, n, bits)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())  # inputs come from the current stream
    gen = torch.Generator(device=dev)
    gen.manual_seed(5)
    for step in range(6):
        q = torch.randn((B, H, G, 128), device=dev, generator=gen)
        kn = torch.randn((B, H, 128), device=dev, generator=gen)
        vn = torch.randn((B, H, 128), device=dev, generator=gen)
        o1, o2 = torch.empty_like(q), torch.empty_like(q)
        s.wait_stream(torch.cuda.current_stream())
        fused.step_device(q, o1, kn, vn, s.cuda_stream)
        plain.decode_device(q, o2, s.cuda_stream)
        plain.append_device(kn, vn, s.cuda_stream)
        s.synchronize()
        assert torch.equal(o1, o2), f"step {step}: fused decode output differs"
    assert fused.tail_tokens() == plain.tail_tokens() == 6
    for u in (0, B * H // 2, B * H - 1):
        for which in (0, 1):
            assert np.array_equal(fused.tail(u, which), plain.tail(u, which)), (u, which)


def test_fused_step_graph_replay_past_capacity(kvq):
    torch = pytest.importorskip("torch")
    B, H, G = 2, 2, 4
    c, _, dev = _pair(kvq, torch, B, H, G, 256, 1, reserve=16)
    cap = c._info()[9]
    q = torch.randn((B, H, G, 128), device=dev)
    out = torch.empty_like(q)
    kn = torch.stack([torch.full((H, 128), float(b + 1), device=dev) for b in range(B)])
    vn = kn.clone()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())  # inputs come from the current stream
    c.decode_device(q, out, s.cuda_stream)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        c.step_device(q, out, kn, vn, s.cuda_stream)
    c.sync_tail()  # capture ran no kernel: host counter back to the device's
    for _ in range(cap + 5):
        graph.replay()
    torch.cuda.synchronize()
    with pytest.raises(kvq.DomainError, match="tail full"):
        c.tail_tokens()
    assert c.tail_tokens() == cap
    for u in range(B * H):
        assert np.all(c.tail(u, 0) == float(u // H + 1))
    # the decode still reads a full, consistent tail
    o2 = torch.empty_like(q)
    c.decode_device(q, o2, s.cuda_stream)
    s.synchronize()
    assert torch.isfinite(o2).all()


def test_host_step_pinned_matches_pageable(kvq):
    """kvq_cache_step (the host-buffer serving step, captured and replayed as a graph per
    buffer set) gives the same outputs and tail for pinned and pageable host buffers."""
    torch = pytest.importorskip("torch")
    B, H, G, n = 4, 8, 4, 1024
    a, b, _ = _pair(kvq, torch, B, H, G, n, 1)
    rng = np.random.default_rng(3)
    for step in range(3):
        q = rng.normal(size=(B, H, G, 128)).astype(np.float32)
        k = rng.normal(size=(B, H, 128)).astype(np.float32)
        v = rng.normal(size=(B, H, 128)).astype(np.float32)
        pq, pk, pv = (torch.from_numpy(x).pin_memory().numpy() for x in (q, k, v))
        pout = torch.empty((B, H, G, 128)).pin_memory().numpy()
        out = np.empty((B, H, G, 128), np.float32)
        a.step(pq, pk, pv, pout)
        b.step(q, k, v, out)
        assert np.array_equal(pout, out), f"step {step}"
    assert a.tail_tokens() == b.tail_tokens() == 3


def test_tail_not_grown_on_a_stale_host_count(kvq):
    """Graph captures advance the host's tail counter without appending on the device; an
    append that only *looks* past the reserved rows must reconcile with the device first
    instead of reallocating the tail (which would change the decode geometry and the
    host-step graph key)."""
    torch = pytest.importorskip("torch")
    B, H, G = 2, 2, 4
    c, _, dev = _pair(kvq, torch, B, H, G, 256, 1, reserve=16)
    cap = c._info()[9]
    q = torch.randn((B, H, G, 128), device=dev)
    out = torch.empty_like(q)
    kn = torch.randn((B, H, 128), device=dev)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())  # inputs come from the current stream
    graphs = []
    for _ in range(cap - 2):  # captures only: the host counter runs ahead by cap - 2
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            c.step_device(q, out, kn, kn, s.cuda_stream)
        graphs.append(g)
    for _ in range(4):  # real appends: host count would pass cap, the device holds 4 rows
        c.append_device(kn, kn, s.cuda_stream)
    s.synchronize()
    assert c._info()[9] == cap, "tail reallocated on a stale host count"
    assert c.tail_tokens() == 4


def test_host_step_three_chunks_long_rows(kvq):
    """Long rows (n >= 16384) take the 3-chunk host step (batch 5: chunks of 2 / 2 / 1
    requests, uneven); outputs and tails against the whole-batch device decode + append. A
    chunk plans its own CTA split, so the fp32 merge order of a unit's parts may differ."""
    torch = pytest.importorskip("torch")
    B, H, G, n = 5, 2, 6, 16384
    a, b, dev = _pair(kvq, torch, B, H, G, n, 1)
    rng = np.random.default_rng(8)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())  # inputs come from the current stream
    for step in range(3):
        q = rng.normal(size=(B, H, G, 128)).astype(np.float32)
        k = rng.normal(size=(B, H, 128)).astype(np.float32)
        v = rng.normal(size=(B, H, 128)).astype(np.float32)
        out = np.empty_like(q)
        a.step(q, k, v, out)
        qd, od = torch.from_numpy(q).to(dev), torch.empty((B, H, G, 128), device=dev)
        kd, vd = torch.from_numpy(k).to(dev), torch.from_numpy(v).to(dev)
        s.wait_stream(torch.cuda.current_stream())
        b.decode_device(qd, od, s.cuda_stream)
        b.append_device(kd, vd, s.cuda_stream)
        s.synchronize()
        want = od.cpu().numpy()
        np.testing.assert_allclose(out, want, rtol=0, atol=2e-6 * np.abs(want).max())
    b.sync_tail()
    assert a.tail_tokens() == b.tail_tokens() == 3
    for u in (0, B * H - 1):
        assert np.array_equal(a.tail(u, 0), b.tail(u, 0))
