"""Summarise an ncu source page (cuda,sass) by CUDA source line: instructions executed
and warp-stall samples. Usage: ncu -i rep --page source --csv --print-source cuda,sass
> x.csv; python tools/ncu_lines.py x.csv [topN]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = next(r for r in rows if "Instructions Executed" in r)
ie, st = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
agg, cur = {}, None
for r in rows[rows.index(hdr) + 1:]:
    if r and r[0].isdigit():
        cur = (int(r[0]), r[1][:100])
        agg.setdefault(cur, [0, 0])
        continue
    if cur and len(r) > ie and r[ie].isdigit():
        agg[cur][0] += int(r[ie])
        agg[cur][1] += int(r[st] or 0)
tot = sum(v[0] for v in agg.values()) or 1
tots = sum(v[1] for v in agg.values()) or 1
print(f"total instructions {tot}, stall samples {tots}")
for (ln, src), (n, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * n / tot:5.1f}%  stall {100 * s / tots:5.1f}%  L{ln:<4} {src}")
