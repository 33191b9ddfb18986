"""Per-SM load vs finish time of one traced decode (the bin tools/trace_chain.py writes).

    python tools/trace_sm.py gpurun_out/trace_chain_c2.bin <decodes in the bin> <solo CTAs> [decode index]

Groups the CTAs of one decode by the SM they ran on (slot 31 = smid + 1), counts solo
(whole-unit) and split (half-unit) CTAs per SM, and prints the finish-time distribution per
SM load: a placement imbalance (SMs holding more units than the mean) shows up as the
latest SMs.
"""
import sys
from collections import defaultdict

import numpy as np

path, K, whole = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
idx = int(sys.argv[4]) if len(sys.argv) > 4 else K - 1
t = np.fromfile(path, dtype=np.uint64).reshape(K, -1, 256).astype(np.int64)
rows = t[idx]
live = np.nonzero(rows[:, 0] > 0)[0]
t0 = rows[live, 0].min()
per = defaultdict(lambda: [0, 0, 0.0, 1e18])
for i in live:
    sm = int(rows[i, 31]) - 1
    e = per[sm]
    if i < whole:
        e[0] += 1
    else:
        e[1] += 1
    e[2] = max(e[2], (rows[i, 5] - t0) / 1e3)
    e[3] = min(e[3], (rows[i, 0] - t0) / 1e3)
by = defaultdict(list)
for sm, (s, h, end, start) in per.items():
    by[(s, h)].append(end)
print(f"decode {idx}: {len(live)} CTAs on {len(per)} SMs, span {max(v[2] for v in per.values()):.1f} us")
print(" solo half  load  SMs   end min / mean / max (us)")
for (s, h), ends in sorted(by.items()):
    print(f" {s:4d} {h:4d} {s + h / 2:5.1f} {len(ends):4d}   {min(ends):6.1f} / {np.mean(ends):6.1f} / {max(ends):6.1f}")
