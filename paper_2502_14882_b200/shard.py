"""Multi-GPU sharding of the decode hot path.

Units (request, KV head) are independent in quantize (K1), decode (K2) and append (K3),
so the path shards with no collective on the data path:

  * batch >= world: rank r owns a contiguous slice of the requests with all their KV
    heads (a request's q / out rows stay contiguous; the local cache is [b_r][H]);
  * batch < world: the (request, KV head) units are dealt round-robin, so no GPU idles while
    units remain (the local cache is [u_r][1]: every unit its own one-head "request").

Each rank builds its own device-resident BatchedCache from its share of the prefill (the
packed KV never crosses GPUs), decodes and appends its units, and the outputs are gathered
to one rank off the timed path: every rank's rows come off the device through the C-ABI
(kvq_cache_decode's device-to-host copy) and travel as tensors (torch.distributed gather,
NCCL between B200s, gloo in the CPU tests) - no pickling; under NCCL the destination places
them in the global order with one kernel and one device-to-host copy (kvq_shard_place).
The unit assignment itself is native (kvq_shard_assign). One process per GPU (torchrun);
the rank binds its device from LOCAL_RANK before any CUDA work.
"""
from __future__ import annotations

import os
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


def assign_units(batch: int, kv_heads: int, world: int) -> list[list[tuple[int, int]]]:
    """(request, KV head) units per rank per §8(e): contiguous request slices when every
    rank gets at least one request, else units dealt round-robin (u = b * H + h). The
    assignment is the library's (kvq_shard_assign, csrc/kvq_shard.cu), so the Python driver
    and the native gather (kvq_shard_place) agree by construction."""
    from . import kvq
    return [[divmod(int(u), kv_heads) for u in kvq.shard_assign(batch, kv_heads, world, r)] for r in range(world)]


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
    def by_request(self) -> bool:
        return self.batch >= self.world

    @property
    def units(self) -> list[tuple[int, int]]:
        return assign_units(self.batch, self.kv_heads, self.world)[self.rank]

    @property
    def slice(self) -> tuple[int, int]:
        """This rank's request range (request mode)."""
        return partition(self.batch, self.world)[self.rank]

    @property
    def local_shape(self) -> tuple[int, int]:
        """(requests, KV heads) of this rank's cache."""
        if self.by_request:
            s, e = self.slice
            return e - s, self.kv_heads
        return len(self.units), 1

    def take(self, x: np.ndarray) -> np.ndarray:
        """This rank's rows of a [B][H][...] array, in its cache's [b][h][...] layout."""
        if self.by_request:
            s, e = self.slice
            return np.ascontiguousarray(x[s:e])
        u = self.units
        if not u:
            return np.zeros((0, 1) + x.shape[2:], x.dtype)
        return np.ascontiguousarray(np.stack([x[b, h] for b, h in u])[:, None])

    def place(self, out: np.ndarray, local: np.ndarray, rank: int) -> None:
        """Write rank `rank`'s local rows into the global [B][H][...] output."""
        if self.by_request:
            s, e = partition(self.batch, self.world)[rank]
            out[s:e] = local.reshape((e - s,) + out.shape[1:])
        else:
            for i, (b, h) in enumerate(assign_units(self.batch, self.kv_heads, self.world)[rank]):
                out[b, h] = local[i, 0]


def bind_device() -> int:
    """Bind this process to GPU LOCAL_RANK: the CUDA runtime the kernel library calls
    (kvq_set_device) and torch. Returns the device index."""
    local = int(os.environ.get("LOCAL_RANK", "0"))
    from . import kvq
    kvq.set_device(local)
    try:
        import torch
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
    except ImportError:
        pass
    return local


# A backend builds a per-rank cache from host prefill [b][H][n][d] and returns an object
# with .decode(q[b][H][G][d]) -> out and .append(k[b][H][d], v[b][H][d]).
Backend = Callable[..., object]


def gpu_backend(k_vis, v_vis, cfg, cal, group):
    """The product backend: a device-resident BatchedCache on this rank's GPU."""
    from .kvq import BatchedCache
    bind_device()
    return BatchedCache.build(k_vis, v_vis, cfg, cal, group=group)


class ShardedCache:
    """This rank's share of a batched hybrid cache plus the gather."""

    def __init__(self, spec: ShardSpec, k_vis: np.ndarray, v_vis: np.ndarray, cfg, cal,
                 backend: Optional[Backend] = None):
        self.spec = spec
        self.local = None
        if spec.local_shape[0] > 0:
            self.local = (backend or gpu_backend)(spec.take(k_vis), spec.take(v_vis), cfg, cal, spec.group)

    def step(self, q_all: np.ndarray, k_new_all: np.ndarray, v_new_all: np.ndarray) -> np.ndarray:
        """Decode this rank's units (reference bench order: decode, then append) and
        return the local output rows [b_r][H_r][G][d]."""
        b, h = self.spec.local_shape
        if self.local is None:
            return np.zeros((0, h, self.spec.group, self.spec.dim), np.float32)
        out = self.local.decode(self.spec.take(q_all))
        out = out[0] if isinstance(out, tuple) else out
        self.local.append(self.spec.take(k_new_all), self.spec.take(v_new_all))
        return np.asarray(out, np.float32)

    def gather(self, out_local: np.ndarray, dst: int = 0) -> Optional[np.ndarray]:
        """Every rank's rows assembled into the global [B][H][G][d] output on `dst` (None
        elsewhere). Rows travel as equal-size tensors (padded to the largest share)."""
        spec = self.spec
        full_shape = (spec.batch, spec.kv_heads, spec.group, spec.dim)
        try:
            import torch
            import torch.distributed as dist
            distributed = dist.is_initialized() and spec.world > 1
        except ImportError:
            distributed = False
        if not distributed:
            out = np.zeros(full_shape, np.float32)
            spec.place(out, out_local, spec.rank)
            return out
        shares = assign_units(spec.batch, spec.kv_heads, spec.world)
        row = spec.group * spec.dim
        width = max(len(s) for s in shares) * row
        dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")
        buf = torch.zeros(width, dtype=torch.float32, device=dev)
        flat = torch.from_numpy(np.ascontiguousarray(out_local, np.float32).reshape(-1))
        buf[:flat.numel()] = flat.to(dev)
        parts = [torch.empty_like(buf) for _ in range(spec.world)] if spec.rank == dst else None
        dist.gather(buf, parts, dst=dst)
        if spec.rank != dst:
            return None
        out = np.zeros(full_shape, np.float32)
        if dev.type == "cuda":  # NCCL: the rows are on this GPU - one placement kernel, one D2H copy
            from . import kvq
            stacked = torch.stack(parts)
            kvq.shard_place(stacked.data_ptr(), spec.world, width, spec.batch, spec.kv_heads, row, out,
                            torch.cuda.current_stream().cuda_stream)
            return out
        for r, p in enumerate(parts):
            n = len(shares[r])
            if not n:
                continue
            lb, lh = (n // spec.kv_heads, spec.kv_heads) if spec.by_request else (n, 1)
            spec.place(out, p[:n * row].cpu().numpy().reshape(lb, lh, spec.group, spec.dim), r)
        return out
