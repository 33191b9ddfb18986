"""Opcode mix of address windows of one kernel in an ncu report's SASS page.

    python tools/sass_regions.py rep.ncu-rep lo:hi [lo:hi ...]   (offsets from the kernel start, hex)
"""
import csv
import subprocess
import sys
from collections import Counter

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
hdr = rows[0]
ia, isrc, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
ins = []
for r in rows[1:]:
    try:
        ins.append((int(r[ia], 16), r[isrc].strip(), int(r[iex] or 0)))
    except (ValueError, IndexError):
        pass
base = ins[0][0]
for win in sys.argv[2:]:
    lo, hi = (int(x, 16) for x in win.split(":"))
    c = Counter()
    n = 0
    for a, s, e in ins:
        if lo <= a - base < hi:
            tok = s.split()
            c[tok[1] if tok[0].startswith("@") else tok[0]] += 1
            n += 1
    print(f"{win}: {n} instr  " + ", ".join(f"{k} {v}" for k, v in c.most_common()))
