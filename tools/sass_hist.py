"""Per-opcode instruction / stall histogram of one kernel from an ncu report's SASS page.

    python tools/sass_hist.py gpurun_out/prof_x.ncu-rep [addr_lo addr_hi]

Groups `Instructions Executed` and warp-stall samples by opcode (optionally inside an
address window), and prints the hottest basic regions (runs of instructions with the same
execution count) so loop bodies can be costed per iteration.
"""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
hdr = rows[0]
ia, isrc, iex, ist = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index(
    "Warp Stall Sampling (All Samples)")
ins = []
for r in rows[1:]:
    try:
        ins.append((int(r[ia], 16), r[isrc].strip(), int(r[iex] or 0), int(r[ist] or 0)))
    except (ValueError, IndexError):
        pass
base = ins[0][0]
lo = int(sys.argv[2], 16) if len(sys.argv) > 2 else 0
hi = int(sys.argv[3], 16) if len(sys.argv) > 3 else 1 << 62
cnt, stall = defaultdict(int), defaultdict(int)
tot = tots = 0
for a, s, e, st in ins:
    if not lo <= a - base < hi:
        continue
    op = s.split()[0] if not s.startswith("@") else s.split()[1]
    op = op.split(".")[0]
    cnt[op] += e
    stall[op] += st
    tot += e
    tots += st
print(f"total executed {tot}  stall samples {tots}")
for op, c in sorted(cnt.items(), key=lambda x: -x[1])[:30]:
    print(f"{op:12s} {c:10d} {100*c/tot:5.1f}%   stalls {stall[op]:7d} {100*stall[op]/max(tots,1):5.1f}%")
# regions: consecutive instructions with equal exec count
print("\nhot regions (offset range, count per instr, #instr, stall samples):")
regs = []
cur = None
for a, s, e, st in ins:
    if cur and cur[2] == e:
        cur[1] = a - base
        cur[3] += 1
        cur[4] += st
    else:
        if cur:
            regs.append(cur)
        cur = [a - base, a - base, e, 1, st]
regs.append(cur)
for r in sorted(regs, key=lambda r: -r[2] * r[3])[:25]:
    print(f"  {r[0]:#07x}-{r[1]:#07x}  x{r[2]:8d}  n={r[3]:4d}  stalls={r[4]}")
