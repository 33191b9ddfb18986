"""Multi-GPU shard logic on CPU (gloo, world_size 2): request partitioning, per-rank
decode + append in the reference order, and the rank-0 gather reproduce a single-process
run exactly. The per-rank compute backend here is the C restatement (oracle/) — the
stand-in for the GPU BatchedCache, which the B200 tests cover."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2502_14882_b200.shard import ShardSpec, ShardedCache, assign_units, partition


def test_partition_covers_batch_contiguously():
    for batch in (1, 2, 7, 8, 64, 513):
        for world in (1, 2, 4, 8):
            parts = partition(batch, world)
            assert parts[0][0] == 0 and parts[-1][1] == batch
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            sizes = [e - s for s, e in parts]
            assert max(sizes) - min(sizes) <= 1


def test_assign_units_requests_then_round_robin():
    # batch >= world: contiguous request slices with all KV heads
    shares = assign_units(5, 2, 2)
    assert shares[0] == [(0, 0), (0, 1), (1, 0), (1, 1), (2, 0), (2, 1)] and shares[1][0] == (3, 0)
    # batch < world: (request, KV head) units dealt round-robin - no idle rank while units remain
    for batch, heads, world in ((1, 8, 8), (1, 2, 4), (3, 8, 4), (2, 3, 8)):
        shares = assign_units(batch, heads, world)
        flat = sorted(u for s in shares for u in s)
        assert flat == [(b, h) for b in range(batch) for h in range(heads)]
        sizes = [len(s) for s in shares]
        assert max(sizes) - min(sizes) <= 1
        assert min(sizes) > 0 or batch * heads < world


class OracleCache:
    """Oracle-backed stand-in with the BatchedCache decode/append interface."""

    def __init__(self, k, v, bits, tau, group):
        from oracle.oracle import C_Oracle
        self.o, self.bits, self.tau, self.group = C_Oracle(), bits, tau, group
        self.k, self.v = k, v
        B, H, n, d = k.shape
        self.segs = {}
        for b in range(B):
            for h in range(H):
                ka, kb = self.o.compute_stats(k[b, h])
                va, vb = self.o.compute_stats(v[b, h])
                self.segs[b, h] = (self.o.quantize(k[b, h], ka, kb, bits), ka, kb, self.o.quantize(v[b, h], va, vb, bits),
                                   va, vb)
        self.tk = [[[] for _ in range(H)] for _ in range(B)]
        self.tv = [[[] for _ in range(H)] for _ in range(B)]

    def decode(self, q):
        B, H, G, d = q.shape
        out = np.zeros_like(q)
        n = self.k.shape[2]
        for b in range(B):
            for h in range(H):
                kc, ka, kb, vc, va, vb = self.segs[b, h]
                for g in range(G):
                    out[b, h, g] = self.o.decode_head(q[b, h, g], n, self.bits, 8, kc, ka, kb, vc, va, vb,
                                                      np.array(self.tk[b][h]), np.array(self.tv[b][h]), *self.tau)[0]
        return out

    def append(self, kn, vn):
        for b in range(kn.shape[0]):
            for h in range(kn.shape[1]):
                self.tk[b][h].append(kn[b, h])
                self.tv[b][h].append(vn[b, h])


def make_problem(seed=5, B=5, H=2, G=2, n=40, d=16, steps=2):
    B = int(os.environ.get("KVQ_TEST_SHARD_B", B))
    rng = np.random.default_rng(seed)
    k = rng.normal(size=(B, H, n, d)).astype(np.float32)
    v = rng.normal(size=(B, H, n, d)).astype(np.float32)
    qs = [rng.normal(size=(B, H, G, d)).astype(np.float32) for _ in range(steps)]
    kn = [rng.normal(size=(B, H, d)).astype(np.float32) for _ in range(steps)]
    vn = [rng.normal(size=(B, H, d)).astype(np.float32) for _ in range(steps)]
    return k, v, qs, kn, vn


def _worker(rank, world, port, result_path):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    k, v, qs, kn, vn = make_problem()
    B, H, n, d = k.shape
    G = qs[0].shape[2]
    spec = ShardSpec(B, H, G, n, d, rank, world)
    backend = lambda kk, vv, cfg, cal, group: OracleCache(kk, vv, 2, (1.0, 0.5), group)  # noqa: E731
    sc = ShardedCache(spec, k, v, None, None, backend=backend)
    outs = []
    for t in range(len(qs)):
        full = sc.gather(sc.step(qs[t], kn[t], vn[t]))
        if rank == 0:
            outs.append(full)
    if rank == 0:
        np.save(result_path, np.stack(outs))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.timeout(300)
@pytest.mark.parametrize("batch", [5, 1])
def test_two_rank_gloo_matches_single_process(tmp_path, monkeypatch, batch):
    """batch 5 on 2 ranks: request slices; batch 1: the 2 units round-robin, one per rank."""
    monkeypatch.setenv("KVQ_TEST_SHARD_B", str(batch))
    result = tmp_path / "out.npy"
    mp.spawn(_worker, args=(2, _free_port(), str(result)), nprocs=2, join=True)
    sharded = np.load(result)
    k, v, qs, kn, vn = make_problem()
    single = OracleCache(k, v, 2, (1.0, 0.5), qs[0].shape[2])
    for t in range(len(qs)):
        want = single.decode(qs[t])
        single.append(kn[t], vn[t])
        assert np.array_equal(sharded[t], want)


def test_native_assignment_matches_the_spec_and_validates(kvq_host):
    """kvq_shard_assign (the library's assignment, used by assign_units and the native
    gather) against §8(e) written out in Python; bad ranks are domain errors."""
    for batch, heads, world in ((5, 2, 2), (64, 8, 8), (3, 8, 4), (1, 8, 8), (2, 3, 8), (0, 8, 2)):
        for r in range(world):
            if batch >= world:
                s, e = partition(batch, world)[r]
                spec = [b * heads + h for b in range(s, e) for h in range(heads)]
            else:
                spec = list(range(r, batch * heads, world))
            assert kvq_host.shard_assign(batch, heads, world, r).tolist() == spec
    with pytest.raises(kvq_host.DomainError):
        kvq_host.shard_assign(4, 8, 2, 2)
