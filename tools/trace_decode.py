"""Debug timeline of one tcgen05 decode launch (KVQ_TRACE_FILE stamps, k2_decode_umma.cu).

    python tools/trace_decode.py [--config c2] [--out gpurun_out/trace.txt]

Builds the bench workload on cuda:0, runs a few decodes, and summarises the per-CTA
globaltimer stamps of the last one: CTA start spread, phase durations, and the
per-block intervals of phase A / phase B.
"""
import argparse
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "trace.txt"))
    args = ap.parse_args()
    raw = str(ROOT / "gpurun_out" / "trace.bin")
    os.environ["KVQ_TRACE_FILE"] = raw
    import torch

    import bench
    from paper_2502_14882_b200 import kvq

    batch, H, G, n, bits, tau, _ = bench.CONFIGS[args.config]
    if args.batch:
        batch = args.batch
    dev = torch.device("cuda", 0)
    k = torch.randn((batch, H, n, 128), device=dev)
    v = torch.randn((batch, H, n, 128), device=dev)
    c = kvq.BatchedCache.build_device(k, v, kvq.QuantizationConfig(bits), kvq.CalibrationParams(*tau), group=G)
    q = torch.randn((batch, H, G, 128), device=dev)
    out = torch.empty_like(q)
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        c.decode_device(q, out, s)
    torch.cuda.synchronize()
    t = np.fromfile(raw, dtype=np.uint64).reshape(-1, 256).astype(np.int64)
    t = t[t[:, 0] > 0]
    t0 = t[:, 0].min()
    lines = []
    rel = lambda x: (x - t0) / 1e3  # us
    ctas = len(t)
    lines.append(f"config {args.config} batch {batch}: {ctas} CTAs traced, kernel span {rel(t[:, 5].max()):.1f} us")
    for name, a_, b_ in [("start->first K block", 0, 1), ("issuer prologue->griddep", 6, 7), ("phase A", 1, 2),
                         ("reduce+calibration", 2, 3), ("phase B", 3, 4), ("epilogue", 4, 5), ("CTA total", 0, 5)]:
        d = (t[:, b_] - t[:, a_]) / 1e3
        lines.append(f"{name:28s} mean {d.mean():7.2f} us  p10 {np.percentile(d, 10):7.2f}  p90 {np.percentile(d, 90):7.2f}")
    st = rel(t[:, 0])
    lines.append(f"CTA start: min {st.min():.2f} p50 {np.median(st):.2f} max {st.max():.2f} us")
    blk = t[:, 64:128].reshape(-1, 16, 4)
    ok = np.all(blk[:, :, 0] > 0, axis=1)
    if ok.any():
        b = blk[ok]
        iss = t[ok, 128:192].reshape(-1, 16, 4)
        prod = t[ok, 192:256]
        base = b[:, :1, 0]
        f = lambda x: " ".join(f"{v:6.2f}" for v in x)
        lines.append("phase A, per block (us from block-0 full; mean over CTAs):")
        lines.append("  full ok     " + f(((b[:, :, 0] - base) / 1e3).mean(0)))
        lines.append("  afull sent  " + f(((b[:, :, 1] - base) / 1e3).mean(0)))
        lines.append("  issuer afull" + f(((iss[:, :, 0] - base) / 1e3).mean(0)))
        lines.append("  issuer dempt" + f(((iss[:, :, 1] - base) / 1e3).mean(0)))
        lines.append("  MMA issued  " + f(((iss[:, :, 2] - base) / 1e3).mean(0)))
        lines.append("  dfull seen  " + f(((b[:, :, 2] - base) / 1e3).mean(0)))
        lines.append("  TMA issued  " + f(((prod[:, :16] - base) / 1e3).mean(0)))
    # concurrency histogram: CTAs alive over time
    grid = np.linspace(0, rel(t[:, 5].max()), 40)
    alive = [int(((rel(t[:, 0]) <= g) & (rel(t[:, 5]) >= g)).sum()) for g in grid]
    lines.append("CTAs alive over time: " + " ".join(str(a) for a in alive))
    txt = "\n".join(lines)
    print(txt)
    Path(args.out).write_text(txt + "\n")


if __name__ == "__main__":
    main()
