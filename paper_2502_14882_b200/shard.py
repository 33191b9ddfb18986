"""Multi-GPU sharding of the decode hot path.

Units (request, KV head) are independent in quantize (K1), decode (K2) and append (K3),
so the path shards with no collective on the data path: rank r owns a contiguous slice
of the requests (all their KV heads, so a request's q/out rows stay contiguous), runs
its own device-resident BatchedCache, and the per-rank outputs are gathered to rank 0
off the timed path (host-side gather; torch.distributed over NCCL on B200s, gloo in the
CPU tests).

One process per GPU, launched by torchrun; RANK / WORLD_SIZE / LOCAL_RANK from the env.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np


def partition(batch: int, world: int) -> list[tuple[int, int]]:
    """Contiguous request slices [start, stop) per rank; the first batch % world ranks
    take one extra request. Ranks beyond the batch get empty slices."""
    base, extra = divmod(batch, world)
    out, start = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        out.append((start, start + n))
        start += n
    return out


@dataclass
class ShardSpec:
    batch: int
    kv_heads: int
    group: int
    n_vis: int
    dim: int
    rank: int
    world: int

    @property
    def slice(self) -> tuple[int, int]:
        return partition(self.batch, self.world)[self.rank]

    @property
    def local_batch(self) -> int:
        s, e = self.slice
        return e - s


# A backend builds a per-rank cache from host prefill [b][H][n][d] and returns an object
# with .decode(q[b][H][G][d]) -> out and .append(k[b][H][d], v[b][H][d]).
Backend = Callable[..., object]


def gpu_backend(k_vis, v_vis, cfg, cal, group):
    """The product backend: a device-resident BatchedCache on this rank's GPU."""
    from .kvq import BatchedCache
    return BatchedCache.build(k_vis, v_vis, cfg, cal, group=group)


class ShardedCache:
    """This rank's share of a batched hybrid cache plus the rank-0 gather."""

    def __init__(self, spec: ShardSpec, k_vis: np.ndarray, v_vis: np.ndarray, cfg, cal,
                 backend: Optional[Backend] = None):
        self.spec = spec
        s, e = spec.slice
        self.local = None
        if e > s:
            self.local = (backend or gpu_backend)(np.ascontiguousarray(k_vis[s:e]), np.ascontiguousarray(v_vis[s:e]),
                                                  cfg, cal, spec.group)

    def step(self, q_all: np.ndarray, k_new_all: np.ndarray, v_new_all: np.ndarray) -> np.ndarray:
        """Decode this rank's requests (reference bench order: decode, then append) and
        return the local output rows [local_batch][H][G][d]."""
        s, e = self.spec.slice
        if self.local is None:
            return np.zeros((0, self.spec.kv_heads, self.spec.group, self.spec.dim), np.float32)
        out = self.local.decode(np.ascontiguousarray(q_all[s:e]))
        out = out[0] if isinstance(out, tuple) else out
        self.local.append(np.ascontiguousarray(k_new_all[s:e]), np.ascontiguousarray(v_new_all[s:e]))
        return np.asarray(out, np.float32)

    def gather(self, out_local: np.ndarray, dst: int = 0) -> Optional[np.ndarray]:
        """Concatenate every rank's rows on `dst` in rank order (None elsewhere)."""
        import torch
        import torch.distributed as dist
        if not dist.is_initialized() or self.spec.world == 1:
            return out_local
        parts = [None] * self.spec.world if self.spec.rank == dst else None
        dist.gather_object(out_local, parts, dst=dst)
        if self.spec.rank != dst:
            return None
        del torch
        return np.concatenate([p for p in parts if p is not None and p.size], axis=0)
