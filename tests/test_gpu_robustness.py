"""GPU robustness of the cache around the hot path:

  * K3 under CUDA-graph replay: a captured decode + append replayed past the rows
    reserve_tail made room for must not write past the tail (kvcache.hpp:99-109 has no such
    state, but a device-resident tail does): the device drops the append and the host
    reports a domain_error at its next synchronization; replays within the capacity are
    reflected in tail_tokens() / read_tail / memory (host counters reconciled from the
    device);
  * an empty cache at d = 128 (zero-row prefill, no tail yet) decodes to zeros, like the
    reference's empty softmax row (calibrate.hpp:77-98, kernels.hpp:415-426);
  * the multi-GPU shard path with the real GPU backend (two ranks on this GPU, gloo) equals
    one whole-batch cache;
  * BatchedCache.step rejects buffers it would read / write out of bounds.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _cache(kvq, torch, B=2, H=2, G=4, n=256, bits=1, reserve=16):
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    k = torch.randn((B, H, n, 128), device=dev, generator=g)
    v = torch.randn((B, H, n, 128), device=dev, generator=g)
    c = kvq.BatchedCache.build_device(k, v, kvq.QuantizationConfig(bits), kvq.CalibrationParams(1.0, 0.0), group=G)
    c.reserve_tail(reserve)
    return c, dev


def test_graph_replay_within_capacity_reconciles_host_counters(kvq):
    torch = pytest.importorskip("torch")
    c, dev = _cache(kvq, torch)
    B, H, G = 2, 2, 4
    q = torch.randn((B, H, G, 128), device=dev)
    out = torch.empty_like(q)
    kn = torch.randn((B, H, 128), device=dev)
    vn = torch.randn((B, H, 128), device=dev)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())  # inputs come from the current stream
    c.decode_device(q, out, s.cuda_stream)
    c.append_device(kn, vn, s.cuda_stream)  # 1 row
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        c.decode_device(q, out, s.cuda_stream)
        c.append_device(kn, vn, s.cuda_stream)
    for _ in range(5):
        graph.replay()
    torch.cuda.synchronize()
    assert c.tail_tokens() == 6  # the device's count, not the host's (capture ran no kernel)
    tail = c.tail(3, 0)
    assert tail.shape == (6, 128)
    want = kn.view(B * H, 128)[3].cpu().numpy()
    assert np.array_equal(tail, np.broadcast_to(want, tail.shape))
    assert c.memory().tail_bytes == B * H * 2 * 6 * 128 * 4


def test_graph_replay_past_capacity_is_an_error_not_corruption(kvq):
    torch = pytest.importorskip("torch")
    c, dev = _cache(kvq, torch, reserve=16)
    cap = c._info()[9]
    B, H, G = 2, 2, 4
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
        c.decode_device(q, out, s.cuda_stream)
        c.append_device(kn, vn, s.cuda_stream)
    for _ in range(cap + 5):
        graph.replay()
    torch.cuda.synchronize()
    with pytest.raises(kvq.DomainError, match="tail full"):
        c.tail_tokens()
    assert c.tail_tokens() == cap  # reported once; the tail holds exactly its capacity
    for u in range(B * H):  # no unit's rows were overwritten by its neighbour's appends
        assert np.all(c.tail(u, 0) == float(u // H + 1))


def test_empty_cache_d128_decodes_to_zeros(kvq):
    torch = pytest.importorskip("torch")
    B, H, G = 2, 2, 4
    k = np.zeros((B, H, 0, 128), np.float32)
    cache = kvq.BatchedCache.build(k, k, kvq.QuantizationConfig(1), kvq.CalibrationParams(1.0, 0.0), group=G)
    q = np.random.default_rng(1).normal(size=(B, H, G, 128)).astype(np.float32)
    for path in (kvq.PATH_AUTO, kvq.PATH_GENERIC):
        cache.set_path(path)
        out, _, _ = cache.decode(q)
        assert np.array_equal(out, np.zeros_like(out)), path
    full = kvq.BatchedCache.build(k, k, kvq.QuantizationConfig(kvq.FULL_PRECISION_BITS), kvq.CalibrationParams(), group=G)
    out, _, _ = full.decode(q)
    assert np.array_equal(out, np.zeros_like(out))


def test_step_rejects_bad_buffers(kvq):
    B, H, G, n = 1, 2, 4, 64
    rng = np.random.default_rng(3)
    k = rng.normal(size=(B, H, n, 128)).astype(np.float32)
    c = kvq.BatchedCache.build(k, k, kvq.QuantizationConfig(1), kvq.CalibrationParams(1.0, 0.0), group=G)
    q = np.zeros((B, H, G, 128), np.float32)
    kv = np.zeros((B, H, 128), np.float32)
    out = np.zeros_like(q)
    c.step(q, kv, kv, out)
    for bad in (q.astype(np.float64), q[..., :64], np.zeros((B, H, G, 256), np.float32)[..., ::2]):
        with pytest.raises(kvq.DomainError):
            c.step(bad, kv, kv, out)
    with pytest.raises(kvq.DomainError):
        c.step(q, kv, kv, np.zeros((B, H, G, 64), np.float32))


def _shard_worker(rank, world, port, result_path):
    import torch.distributed as dist

    from paper_2502_14882_b200 import kvq
    from paper_2502_14882_b200.shard import ShardSpec, ShardedCache
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), LOCAL_RANK="0")  # one GPU, two ranks
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(11)
    B, H, G, n = int(os.environ["KVQ_SHARD_B"]), 8, 4, 700
    k = rng.normal(size=(B, H, n, 128)).astype(np.float32)
    v = rng.normal(size=(B, H, n, 128)).astype(np.float32)
    spec = ShardSpec(B, H, G, n, 128, rank, world)
    sc = ShardedCache(spec, k, v, kvq.QuantizationConfig(1), kvq.CalibrationParams(1.0, 0.0))
    outs = []
    for _ in range(2):
        q = rng.normal(size=(B, H, G, 128)).astype(np.float32)
        kn = rng.normal(size=(B, H, 128)).astype(np.float32)
        full = sc.gather(sc.step(q, kn, kn))
        if rank == 0:
            outs.append(full)
    if rank == 0:
        np.save(result_path, np.stack(outs))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("batch", [3, 1])
def test_sharded_gpu_backend_matches_whole_batch(kvq, tmp_path, monkeypatch, batch):
    """Two ranks (request slices for batch 3; the 8 units of batch 1 round-robin) with the
    GPU BatchedCache backend, gathered as tensors, equal one whole-batch cache (to 2e-6: a
    shard's unit count picks its own CTA split, i.e. the fp32 merge order of a unit's parts)."""
    import torch.multiprocessing as mp
    monkeypatch.setenv("KVQ_SHARD_B", str(batch))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    res = tmp_path / "out.npy"
    mp.spawn(_shard_worker, args=(2, port, str(res)), nprocs=2, join=True)
    got = np.load(res)
    rng = np.random.default_rng(11)
    B, H, G, n = batch, 8, 4, 700
    k = rng.normal(size=(B, H, n, 128)).astype(np.float32)
    v = rng.normal(size=(B, H, n, 128)).astype(np.float32)
    whole = kvq.BatchedCache.build(k, v, kvq.QuantizationConfig(1), kvq.CalibrationParams(1.0, 0.0), group=G)
    for t in range(2):
        q = rng.normal(size=(B, H, G, 128)).astype(np.float32)
        kn = rng.normal(size=(B, H, 128)).astype(np.float32)
        want, _, _ = whole.decode(q)
        whole.append(kn, kn)
        np.testing.assert_allclose(got[t], want, rtol=0, atol=2e-6)


@pytest.mark.parametrize("batch,heads,world", [(7, 8, 3), (1, 8, 3), (2, 3, 8), (64, 8, 8)])
def test_shard_place_matches_host_placement(kvq, batch, heads, world):
    """kvq_shard_place (the NCCL gather's last hop: one placement kernel + one D2H copy)
    against ShardSpec.place on the same gathered rows, request slices and round-robin,
    host and device destinations."""
    torch = pytest.importorskip("torch")
    from paper_2502_14882_b200.shard import ShardSpec, assign_units
    G, d = 4, 128
    row = G * d
    shares = assign_units(batch, heads, world)
    width = max(len(s) for s in shares) * row + 5  # odd padding: the scalar copy path too
    rng = np.random.default_rng(batch * 100 + world)
    parts = rng.normal(size=(world, width)).astype(np.float32)
    want = np.zeros((batch, heads, G, d), np.float32)
    for r in range(world):
        spec = ShardSpec(batch, heads, G, 16, d, r, world)
        n = len(shares[r])
        if n:
            lb, lh = spec.local_shape
            spec.place(want, parts[r, :n * row].reshape(lb, lh, G, d), r)
    dev = torch.from_numpy(parts).cuda()
    got = np.full(want.shape, np.nan, np.float32)
    kvq.shard_place(dev.data_ptr(), world, width, batch, heads, row, got)
    assert np.array_equal(got, want)
    got_dev = torch.full(want.shape, float("nan"), device="cuda")
    kvq.shard_place(dev.data_ptr(), world, width, batch, heads, row, got_dev.data_ptr())
    assert np.array_equal(got_dev.cpu().numpy(), want)
