"""Warp-stall reasons summed over address windows of one kernel (ncu SASS page).

    python tools/sass_stalls.py rep.ncu-rep lo:hi [lo:hi ...]   (hex offsets from the kernel start)
"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
hdr = rows[0]
ia = hdr.index("Address")
cols = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
ins = []
for r in rows[1:]:
    try:
        ins.append((int(r[ia], 16), [int(r[i] or 0) for i, _ in cols]))
    except (ValueError, IndexError):
        pass
base = ins[0][0]
for win in sys.argv[2:]:
    lo, hi = (int(x, 16) for x in win.split(":"))
    tot = [0] * len(cols)
    for a, v in ins:
        if lo <= a - base < hi:
            tot = [x + y for x, y in zip(tot, v)]
    s = sum(tot) or 1
    print(f"{win}: {s} samples  " + ", ".join(f"{cols[i][1][6:]} {100 * x / s:.0f}%"
                                               for i, x in sorted(enumerate(tot), key=lambda z: -z[1]) if x))
