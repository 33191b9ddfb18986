"""Benchmark: CalibQuant quantized decode attention on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

One STEP = one decode step of one attention layer for a batch of requests, in the
reference's bench order (kvq_main.cpp:313-321): K2 fused calibrated decode over the
packed visual cache + fp32 tail for every (request, KV head, query head), then K3 append
of the step's new K/V row. Default workload = BASELINE config 2 (InternVL2.5-8B shape:
32 q / 8 KV heads, d = 128, 4096 visual tokens, batch 64 per GPU, 1-bit, calibration).

Timing: W warm-up steps, then exactly K steps between barrier + synchronize, CUDA events
on the launching stream, max over ranks. Each timed step is one CUDA-graph replay of
[K2 decode + K3 append]; a second pass replays one graph chaining every replica's decode
back to back (no events between launches, PDL overlap intact) for the roofline's kernel
time. After timing, a parity spot check decodes replica 0 and compares three units with the
float64 reference math on the cache's own codes. The packed caches are device-resident; the
step rotates over R cache replicas whose total size exceeds the 126 MB L2 (so no step
reads a cache another step left in L2) and which also bounds every replica's fp32 tail
to <= tail_window generated tokens. `e2e` repeats the step through the public C-ABI
(kvq_cache_step) with pinned host buffers: queries/new K,V copied in and outputs copied
out every step.

Multi-GPU (torchrun, one rank per GPU): a global batch (config batch x GPUs by default =
weak scaling; --global-batch B = strong scaling) is sharded per SURVEY §8e by
paper_2502_14882_b200.shard (request slices, or (request, KV head) units round-robin when
B < GPUs); no collective on the data path, NCCL only for the barrier and the max-over-ranks
timing. `value` is the whole job's tokens/s; `per_gpu` divides by the GPU count.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "quantized decode-attn tokens/s/GPU and HBM GB/s (% of peak), 1/2/4/8 B200 vs CPU ref"

CONFIGS = {
    # name: (batch, kv_heads, group, n_vis, bits, tau, description)
    "c1": (1, 1, 1, 1024, 1, (1.0, 0.0), "BASELINE c1: 1 request, 1 KV head, d=128, 1024 visual tokens, 1-bit"),
    "c2": (64, 8, 4, 4096, 1, (1.0, 0.0),
           "BASELINE c2: InternVL2.5-8B decode, 32 q / 8 KV heads, d=128, 4096 visual tokens, batch 64, "
           "1-bit, calibration tau=(1,0)"),
    "c3b1": (32, 8, 4, 8192, 1, (1.0, 0.0), "BASELINE c3: 32q/8kv, 8192 visual tokens, batch 32, 1-bit"),
    "c3b2": (32, 8, 4, 8192, 2, (1.0, 0.0), "BASELINE c3: 32q/8kv, 8192 visual tokens, batch 32, 2-bit"),
    "c3b4": (32, 8, 4, 8192, 4, (1.0, 0.0), "BASELINE c3: 32q/8kv, 8192 visual tokens, batch 32, 4-bit"),
    "c4": (16, 8, 6, 32768, 1, (1.0, 0.0),
           "BASELINE c4: InternVL2.5-26B long video, 48 q / 8 KV heads, 32k visual tokens, batch 16, 1-bit"),
    "c5b8": (8, 8, 4, 4096, 1, (1.0, 0.0), "BASELINE c5: batch 8, 4096 visual tokens, 1-bit"),
    "c5b512": (512, 8, 4, 4096, 1, (1.0, 0.0), "BASELINE c5: batch 512, 4096 visual tokens, 1-bit"),
}
# BASELINE config 3 "with and without post-scaling and calibration": name -> (base config,
# tau, decode path, CPU arm). "nocal" = tau (0, 0) (the identity g, calibrate.hpp:62-67);
# "deq" = dequantize-then-dot (every code dequantized in-register, then dotted: the
# reference's naive_qk(q, dequantize(seg)) / naive_wv, kernels.hpp:401-426 on
# quantize.hpp:129-146) on the generic decode, next to the same kernel post-scaled ("gen").
ABLATIONS = {}
for _b in ("c3b1", "c3b2", "c3b4"):
    ABLATIONS[_b + "_nocal"] = (_b, (0.0, 0.0), None, "post")
    ABLATIONS[_b + "_gen"] = (_b, None, "generic", "post")
    ABLATIONS[_b + "_gen_nocal"] = (_b, (0.0, 0.0), "generic", "post")
    ABLATIONS[_b + "_deq"] = (_b, None, "dequant", "dequant")
    ABLATIONS[_b + "_deq_nocal"] = (_b, (0.0, 0.0), "dequant", "dequant")


# Opt-in token-wise V (north_star "token-wise min/max for V"; KVQ_MODE_V_TOKEN_WISE) on a
# BASELINE shape: name -> base config. The CPU arm runs the reference's own (channel-wise V)
# decode of the same shape - the reference has no token-wise mode.
VTOKEN = {"c2_vtok": "c2", "c3b1_vtok": "c3b1", "c3b4_vtok": "c3b4"}


def resolve_config(name: str):
    """(batch, kv_heads, group, n, bits, tau, description, path override, CPU arm)."""
    if name in CONFIGS:
        return (*CONFIGS[name], None, "post")
    if name in VTOKEN:
        batch, H, G, n, bits, tau, desc = CONFIGS[VTOKEN[name]]
        desc += "; opt-in token-wise V quantization (K channel-wise); CPU arm: the reference's channel-wise V"
        return batch, H, G, n, bits, tau, desc, None, "post"
    base, tau, path, cpu = ABLATIONS[name]
    batch, H, G, n, bits, tau0, desc = CONFIGS[base]
    tau = tau0 if tau is None else tau
    desc += f"; ablation: tau={tuple(tau)}, " + ("dequantize-then-dot (no post-scaling)" if cpu == "dequant" else
                                                   "post-scaled") + (f", {path} decode path" if path else "")
    return batch, H, G, n, bits, tau, desc, path, cpu


DIM = 128
PATHS = {"auto": 0, "generic": 1, "tc": 2, "umma": 3, "dequant": 4}  # KVQ_PATH_* (include/kvq_capi.h)
TAIL_WINDOW = 32
L2_BYTES = 126 * 1024 * 1024


def alg_bytes_unit(n_vis: int, bits: int, group: int, n_tail: int, dim: int = DIM, v_token_wise: bool = False) -> int:
    """Algorithmic HBM bytes of one decode step for one unit:
    packed K+V codes + alpha/beta for K and V (token-wise V: per token) + q in/out + fp32 tail K+V."""
    v_stats = 2 * n_vis * 4 if v_token_wise else 2 * dim * 4
    return 2 * n_vis * dim * bits // 8 + 2 * dim * 4 + v_stats + 2 * group * dim * 4 + 2 * n_tail * dim * 4


def workload_config(args, world: int) -> dict:
    """The workload the line measures - identical in both arms (the driver compares them):
    BASELINE config name, shape, quantization and the global batch; no implementation keys."""
    batch, H, G, n, bits, tau, desc, _, _ = resolve_config(args.config)
    if args.batch:
        batch = args.batch
    if args.tail:
        desc += f", {args.tail} generated tokens in the fp32 tail"
    global_batch = args.global_batch or batch * world
    return {"workload": desc, "name": args.config, "global_batch": global_batch, "q_heads": H * G, "kv_heads": H,
            "head_dim": DIM, "n_vis": n, "bits": bits, "tau": list(tau), "tail_prefill": args.tail,
            "parallelism": (f"{'request slices' if global_batch >= world else '(request, KV head) units round-robin'}"
                            f" x{world} GPUs, no collective")}


def decode_f64(codes_k, codes_v, ka, kb, va, vb, q, kt, vt, bits, tau, v_token_wise: bool = False) -> np.ndarray:
    """The reference decode (kvcache.hpp:263-311: post-scaled scores, calibrated softmax
    over [g(vis) | tail], w.V) in float64 on the cache's own integer codes - the spot
    check's ground truth (SURVEY.md §8c rule 4)."""
    f = np.float64
    L = float((1 << bits) - 1)
    ka, kb, va, vb, q = (np.asarray(x, f) for x in (ka, kb, va, vb, q))
    sk = np.where(kb > ka, (kb - ka) / L, 0.0)
    sv = np.where(vb > va, (vb - va) / L, 0.0)
    isd = 1.0 / np.sqrt(f(q.size))
    vis = (codes_k.astype(f) @ (q * sk) + q @ ka) * isd
    tail = (np.asarray(kt, f) @ q) * isd
    gamma, delta = vis.min(), vis.max()
    if delta > gamma:
        t = (vis - gamma) / (delta - gamma)
        vis = vis - (tau[0] * (1 - t) + tau[1] * t)
    else:
        vis = vis - tau[0]
    row = np.concatenate([vis, tail])
    p = np.exp(row - row.max())
    p /= p.sum()
    if v_token_wise:  # va / vb per token: alpha_j + code_jc (beta_j - alpha_j) / L
        return p[:vis.size] @ (va[:, None] + codes_v.astype(f) * sv[:, None]) + p[vis.size:] @ np.asarray(vt, f)
    return p[:vis.size] @ (va + codes_v.astype(f) * sv) + p[vis.size:] @ np.asarray(vt, f)


def unpack_rows(raw: np.ndarray, n: int, bits: int) -> np.ndarray:
    """Codes [n][128] of a reference M = 8 segment (MSB-first within bytes, bitpack.hpp:85)."""
    b = np.asarray(raw, np.uint8).reshape(n, 16 * bits)
    shifts = 8 - bits * (np.arange(8 // bits) + 1)
    return ((b[..., None] >> shifts) & ((1 << bits) - 1)).reshape(n, DIM)


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def peak_hbm() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """Samples SM clock + throttle reasons via NVML while the timed region runs."""

    REASONS = {
        "hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4,
        "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self._stop = [], set(), threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv, self.h = pynvml, self._handle(pynvml, index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
            self.max_mhz = None

    @staticmethod
    def _handle(pynvml, index: int):
        """NVML handle of CUDA device `index`: by PCI address (CUDA and NVML may enumerate
        differently, e.g. under CUDA_VISIBLE_DEVICES), else by index."""
        try:
            import torch
            pr = torch.cuda.get_device_properties(index)
            bus = "%08x:%02x:%02x.0" % (pr.pci_domain_id, pr.pci_bus_id, pr.pci_device_id)
            return pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
        except Exception:
            return pynvml.nvmlDeviceGetHandleByIndex(index)

    def _sample(self):
        self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
        r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        for name, bit in self.REASONS.items():
            if r & bit:
                self.reasons.add(name)

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            time.sleep(0.005)

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        if self.nv:
            self._stop.set()
            self._t.join()
            self._sample()

    def summary(self):
        if not self.nv or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        backend = "nccl" if args.impl == "ours" else "gloo"
        if backend == "nccl":
            import torch
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    return world, rank, local


def cpu_reference(cfg_name: str, requests: int, steps: int, threads: int, warmup: int = 1, budget_s: float = 0.0,
                  tail: int = 0):
    """The reference's own HybridKVCache::decode_step (oracle/_ref/libkvq_ref.so, compiled
    unmodified from /root/reference) on a bounded sample of the workload: `requests` of the
    config's requests, all KV heads, G decode_step calls per request (GQA emulated), outer
    thread pool over requests; `warmup` untimed steps, median of `steps` timed steps (capped
    so the timed steps take about `budget_s` seconds when budget_s > 0). Returns
    (tokens/s, detail)."""
    from oracle.oracle import Ref
    batch, H, G, n, bits, tau, _, _, cpu_arm = resolve_config(cfg_name)
    requests = min(requests, batch)
    rng = np.random.default_rng(7)
    k = rng.standard_normal((requests, H, n, DIM), dtype=np.float32)
    v = rng.standard_normal((requests, H, n, DIM), dtype=np.float32)
    q = rng.standard_normal((requests, H, G, DIM), dtype=np.float32)
    kn = rng.standard_normal((requests, H, DIM), dtype=np.float32)
    vn = rng.standard_normal((requests, H, DIM), dtype=np.float32)
    # b >= 2 needs the reference's M = 32 path for correct output at n >= 512
    # (kernels.hpp:220 defect); b = 1 runs as shipped (M = 8).
    word_bits = 8 if bits == 1 else 32
    ref = Ref()
    if budget_s > 0:  # size the run: one probe step
        probe, _ = ref.bench_decode(k, v, requests, H, G, n, DIM, bits, word_bits, tau[0], tau[1], q, kn, vn,
                                    threads, 2, tail, dequant=cpu_arm == "dequant")
        steps = max(1, min(steps, int(budget_s / max(min(probe), 1e-6))))
    secs, _ = ref.bench_decode(k, v, requests, H, G, n, DIM, bits, word_bits, tau[0], tau[1], q, kn, vn, threads,
                               steps + warmup, tail, dequant=cpu_arm == "dequant")
    step_s = statistics.median(secs[warmup:])
    return requests / step_s, {
        "sample": f"{requests} of {batch} requests x {H} KV heads x G={G}, n_vis={n}, b={bits}, M={word_bits}, "
                  f"fp32 tail {tail}+; "
                  f"median of {steps} steps after {warmup} warm-up; reference "
                  + ("dequantize + naive_qk/naive_wv (no post-scaling)" if cpu_arm == "dequant"
                     else "HybridKVCache::decode_step") + " + append",
        "step_seconds": step_s,
        "steps": steps,
    }


def run_reference(args, world, rank):
    """Reference arm: the reference's CPU path on this host's cores (rank 0 only), same
    config / metric / unit as our arm, `--steps K --warmup W` honoured (K capped so the
    timed part stays around a minute)."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    batch, H, G, n, bits, tau, desc, _, _ = resolve_config(args.config)
    if args.tail:
        desc += f", {args.tail} generated tokens in the fp32 tail"
    t0 = time.time()
    warm = max(1, args.warmup)
    value, det = cpu_reference(args.config, args.cpu_requests, args.steps, threads, warmup=warm, budget_s=60.0,
                               tail=args.tail)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": det["steps"], "warmup": warm, "ms_per_step": det["step_seconds"] * 1e3, "higher_is_better": True,
        "scaling": "strong" if args.global_batch else "weak", "vs_baseline": None, "dtype": f"u{bits}",
        "data": "synthetic (gaussian)", "config": workload_config(args, world),
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "reference",
                         "cpu_model": cpu_model(), "sample": det["sample"]},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": time.time() - t0,
    }
    print(json.dumps(line), flush=True)


def run_ours(args, world, rank, local):
    import torch
    from paper_2502_14882_b200 import kvq

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    batch, H, G, n, bits, tau, desc, path_override, _ = resolve_config(args.config)
    if path_override:
        args.path = path_override
    if args.tail:
        desc += f", {args.tail} generated tokens in the fp32 tail"
    if args.batch:
        batch = args.batch
    # §8(e) sharding: a global batch over the ranks (contiguous request slices, or
    # (request, KV head) units round-robin when the batch is smaller than the GPU count);
    # weak scaling by default (config batch per GPU), strong with --global-batch.
    from paper_2502_14882_b200.shard import ShardSpec
    global_batch = args.global_batch or batch * world
    spec = ShardSpec(global_batch, H, G, n, DIM, rank, world)
    batch, H = spec.local_shape  # this rank's cache: [batch][H] units
    if batch == 0:
        raise SystemExit(f"rank {rank}: no units (global batch {global_batch} x {spec.kv_heads} KV heads < {world} GPUs)")
    units = batch * H
    stream = torch.cuda.Stream(device=dev)
    sptr = stream.cuda_stream
    W, K = args.warmup, args.steps

    # Replicas: total packed bytes > L2 and <= TAIL_WINDOW appends per replica.
    cache_bytes = units * (2 * n * DIM * bits // 8 + 16 * DIM)
    K2 = min(K, 200)  # second timed pass (decode chain): about this many decode launches
    total_steps = W + K + args.e2e_steps
    R = max(2, -(-total_steps // TAIL_WINDOW), -(-(3 * L2_BYTES) // cache_bytes))
    tail_cap = -(-(total_steps + 2 * R) // R) + 3  # per replica: warm-up + timed + e2e appends
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    kv_chunk = max(1, min(batch, (1 << 31) // (H * n * DIM * 4)))  # bound the fp32 staging to ~2 GiB
    caches = []
    with torch.cuda.stream(stream):
        k = torch.randn((batch, H, n, DIM), device=dev, dtype=torch.float32, generator=gen)
        v = torch.randn((batch, H, n, DIM), device=dev, dtype=torch.float32, generator=gen)
        for r in range(R):
            qmode = kvq.QuantMode.v_token_wise if args.config in VTOKEN else kvq.QuantMode.channel_wise
            c = kvq.BatchedCache.build_device(k, v, kvq.QuantizationConfig(bits, qmode), kvq.CalibrationParams(*tau),
                                              group=G, stream=sptr)
            c.reserve_tail(tail_cap + args.tail)
            c.set_path(PATHS[args.path])
            caches.append(c)
        del k, v
        q = [torch.randn((batch, H, G, DIM), device=dev, generator=gen) for _ in range(4)]
        kn = [torch.randn((batch, H, DIM), device=dev, generator=gen) for _ in range(4)]
        vn = [torch.randn((batch, H, DIM), device=dev, generator=gen) for _ in range(4)]
        out = torch.empty((batch, H, G, DIM), device=dev)
    stream.synchronize()
    torch.cuda.empty_cache()
    del kv_chunk

    tails = [0] * R
    # --tail N: every request already generated N tokens (fp32 tail rows) before the timed
    # steps - the long-generation regime where the dense tail is a second bandwidth term.
    for r in range(R):
        for i in range(args.tail):
            caches[r].append_device(kn[i % 4], vn[i % 4], sptr)
        tails[r] += args.tail
    stream.synchronize()

    # Eager warm-up (allocates the decode scratch), then CUDA graphs of whole steps [K2 decode
    # + K3 append] through kvq_cache_step_device (one kernel per step when the decode owns
    # the fp32 tail in-kernel: the append is fused into it). A serving engine captures a
    # decode iteration as one graph, so consecutive kernels keep their programmatic
    # dependent launch edges: the timed steps replay graphs of consecutive steps (one per
    # round over the R replicas, plus one of the first K % R steps) - no host launch and no
    # graph boundary between steps. A second graph chains the R replicas' decodes alone (the
    # roofline's kernel time, no events between launches).
    for t in range(R):
        caches[t].step_device(q[t % 4], out, kn[t % 4], vn[t % 4], sptr)
        tails[t] += 1
    stream.synchronize()

    def capture_steps(count):
        g = torch.cuda.CUDAGraph()
        l0 = kvq.launch_count()
        with torch.cuda.graph(g, stream=stream):
            for r in range(count):
                caches[r].step_device(q[r % 4], out, kn[r % 4], vn[r % 4], sptr)
        return g, (kvq.launch_count() - l0) // count

    g_round, launches_step = capture_steps(R)
    g_part = capture_steps(K % R)[0] if K % R else None
    g_chain = torch.cuda.CUDAGraph()
    l0 = kvq.launch_count()
    with torch.cuda.graph(g_chain, stream=stream):
        for r in range(R):
            caches[r].decode_device(q[r % 4], out, sptr)
    launches_dec = (kvq.launch_count() - l0) // R

    def run_steps(count):  # `count` steps from replica 0: whole rounds, then the first count % R
        with torch.cuda.stream(stream):
            for _ in range(count // R):
                g_round.replay()
            if count % R:
                assert count % R == K % R
                g_part.replay()
        for t in range(count):
            tails[t % R] += 1

    W_run = -(-W // R) * R  # warm-up in whole rounds (>= the requested W steps)
    run_steps(W_run)
    stream.synchronize()
    if world > 1:
        torch.distributed.barrier()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c_start, c_stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    chain_reps = max(2, -(-K2 // R))
    bytes_alg = 0
    sampler = ClockSampler(local)
    with sampler:
        torch.cuda.synchronize()
        # Let the host run ahead: a ~20 ms spin on the stream (before the timed region)
        # while all K steps are enqueued, so no launch gap lands inside an event interval.
        with torch.cuda.stream(stream):
            torch.cuda._sleep(int(4e7))
        for i in range(K):  # the timed steps' tail lengths (replica i % R, before its append)
            bytes_alg += units * alg_bytes_unit(n, bits, G, tails[i % R] + i // R, v_token_wise=args.config in VTOKEN)
        start.record(stream)
        run_steps(K)
        stop.record(stream)
        stream.synchronize()
        # second pass: the decode chain (roofline timing of the dominant kernel)
        with torch.cuda.stream(stream):
            torch.cuda._sleep(int(2e7))
            c_start.record(stream)
            for _ in range(chain_reps):
                g_chain.replay()
            c_stop.record(stream)
        stream.synchronize()
    bytes_alg2 = sum(units * alg_bytes_unit(n, bits, G, tails[r], v_token_wise=args.config in VTOKEN) for r in range(R)) / R  # per decode launch
    launches = K * launches_step
    # Parity spot check at the measured geometry (outside the timed region): one decode of
    # replica 0, the first / last / a middle unit against the float64 reference math on the
    # cache's own codes, stats and tail rows.
    spot = None
    if rank == 0 and args.path != "generic":
        with torch.cuda.stream(stream):
            caches[0].decode_device(q[0], out, sptr)
        stream.synchronize()
        got, qh = out.cpu().numpy(), q[0].cpu().numpy()
        worst = 0.0
        checked = sorted({0, units // 2, units - 1})
        for u in checked:
            bq, hq_ = divmod(u, H)
            ks, vs = caches[0].segment(u, 0), caches[0].segment(u, 1)
            ck, cv = unpack_rows(ks.codes.bytes, n, bits), unpack_rows(vs.codes.bytes, n, bits)
            kt, vt = caches[0].tail(u, 0), caches[0].tail(u, 1)
            vtok = args.config in VTOKEN
            va, vb = caches[0].value_token_stats(u) if vtok else (vs.stats.alpha, vs.stats.beta)
            for g in range(G):
                want = decode_f64(ck, cv, ks.stats.alpha, ks.stats.beta, va, vb, qh[bq, hq_, g], kt, vt, bits, tau,
                                  v_token_wise=vtok)
                worst = max(worst, float(np.linalg.norm(got[bq, hq_, g] - want) / np.linalg.norm(want)))
        spot = {"units": checked, "heads": G, "max_rel_l2_vs_float64": worst, "tail_rows": int(kt.shape[0])}
    assert max(tails) <= tail_cap + args.tail, "bench tail accounting exceeded the reserved capacity"
    elapsed_ms = start.elapsed_time(stop)
    dec_mean_s = c_start.elapsed_time(c_stop) * 1e-3 / (chain_reps * R)
    if world > 1:
        tt = torch.tensor([elapsed_ms], device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        elapsed_ms = float(tt.item())
        torch.distributed.barrier()
    ms_per_step = elapsed_ms / K
    value = global_batch * K / (elapsed_ms * 1e-3)  # every request of the global batch: one token per step

    # Roofline of the dominant kernel. When the step is ONE kernel (the append fused into the
    # decode, launches_step == 1) that kernel's time per launch IS the step time: K launches
    # back to back between the events, PDL overlap intact. Otherwise (the tail pass, or the
    # append kernel) the K2 decode's time comes from the decode-only chain.
    one_kernel = launches_step == 1
    kernel_s = ms_per_step * 1e-3 if one_kernel else dec_mean_s
    bytes_launch = bytes_alg / K if one_kernel else bytes_alg2
    achieved = bytes_launch / kernel_s / 1e9
    peak, peak_kind = peak_hbm()
    prof = ROOT / "profiles" / "decode_ncu_summary.json"
    traffic = None
    if prof.exists():
        try:
            key = args.config + (f"+tail{args.tail}" if args.tail else "")
            traffic = json.loads(prof.read_text()).get(key, {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    # e2e through the public C-ABI with host (pinned) buffers.
    E = args.e2e_steps
    hq = torch.randn((batch, H, G, DIM)).pin_memory().numpy()
    hk = torch.randn((batch, H, DIM)).pin_memory().numpy()
    hv = torch.randn((batch, H, DIM)).pin_memory().numpy()
    hout = torch.empty((batch, H, G, DIM)).pin_memory().numpy()
    for t in range(R):  # every replica once: per-cache streams / events are created lazily
        caches[t].step(hq, hk, hv, hout)
    if world > 1:
        torch.distributed.barrier()
    # Collect and freeze the interpreter's garbage before the timed host loop, as a serving
    # process would after start-up: without it, 2 of 3 C2 runs showed two ~4 ms stalls in 100
    # steps (e2e 0.37 M vs 0.67 M tok/s; per-step median unchanged, `step_us_p10_p50_p90`).
    gc.collect()
    gc.freeze()
    t0 = time.perf_counter()
    marks = []  # per-step host timestamps (the spread shows host / PCIe jitter)
    for t in range(E):
        caches[t % R].step(hq, hk, hv, hout)
        marks.append(time.perf_counter())
    e2e_s = time.perf_counter() - t0
    step_us = np.diff(np.array([t0] + marks)) * 1e6
    if world > 1:
        tt = torch.tensor([e2e_s], device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(tt.item())
    e2e_value = global_batch * E / e2e_s

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cv, det = cpu_reference(args.config, args.cpu_requests, args.steps_cpu, os.cpu_count() or 1,
                                    tail=args.tail)
            cpu = {"value": cv, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "reference",
                   "cpu_model": cpu_model(), "sample": det["sample"]}
        except Exception as e:  # keep the GPU line even if the checker is missing
            cpu = {"value": None, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if args.global_batch else "weak", "vs_baseline": None,
            "dtype": f"u{bits}", "data": "synthetic (gaussian K/V/q, torch.randn on device)",
            "config": workload_config(args, world),
            "per_gpu": {"value": value / world, "unit": "tokens/s/GPU", "rank0_units": units},
            "impl_details": {"tail_window": TAIL_WINDOW, "warmup_steps_run": W_run,
                             "graph": f"steps replayed as CUDA graphs of {R} consecutive steps (one round over the "
                                      "replicas; PDL edges between steps kept)",
                             "l2": f"inputs larger than L2: {R} rotating cache replicas x {cache_bytes / 2**20:.1f} MiB",
                             "step": "K2 decode (all q heads) + K3 append", "decode_path": args.path},
            "hbm_gbs": bytes_alg / K / (ms_per_step * 1e-3) / 1e9,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                         "kernel": ("K2 decode + K3 append, one fused kernel per step" if one_kernel else
                                    "K2 decode" + (" + fp32 tail pass" if args.tail + tail_cap > 64 else "")),
                         "alg_bytes_per_launch": bytes_launch,
                         "launch_us": kernel_s * 1e6,
                         "launches_per_step": launches_step,
                         "decode_only_chain_us": dec_mean_s * 1e6,
                         "launches_per_decode": launches_dec,
                         "timing": ("the timed steps themselves: CUDA events around K back-to-back launches of the "
                                    "fused kernel (multi-step graphs, PDL overlap kept)" if one_kernel else
                                    f"CUDA events around {chain_reps} replays of one graph chaining the {R} replicas' "
                                    "decodes back to back (PDL overlap between launches kept, no events in between)")},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "tokens/s", "h2d_bytes_per_step": int(hq.nbytes + hk.nbytes + hv.nbytes),
                    "d2h_bytes_per_step": int(hout.nbytes), "steps": E,
                    "step_us_p10_p50_p90": [round(float(np.percentile(step_us, x)), 1) for x in (10, 50, 90)],
                    "slowest_steps_us": sorted(((round(float(u), 1), int(i)) for i, u in enumerate(step_us)),
                                               reverse=True)[:5]},
            "gpu_launches": int(launches),
            "spot_check": spot,
            "clocks": sampler.summary(),
        }
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS) + sorted(ABLATIONS) + sorted(VTOKEN))
    ap.add_argument("--batch", type=int, default=0, help="override the config's per-GPU batch")
    ap.add_argument("--global-batch", type=int, default=0,
                    help="fixed global batch sharded over the GPUs (strong scaling); default: config batch per GPU")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=100)
    ap.add_argument("--tail", type=int, default=0,
                    help="generated tokens already in every request's fp32 tail (SURVEY §8 f2 long-tail runs)")
    ap.add_argument("--cpu-requests", type=int, default=16)
    ap.add_argument("--steps-cpu", type=int, default=3)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--path", default=os.environ.get("KVQ_PATH", "auto"), choices=sorted(PATHS),
                    help="K2 decode kernel: auto, tc (mma.sync IMMA), umma (tcgen05), generic")
    args = ap.parse_args()
    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
