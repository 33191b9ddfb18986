"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel:
launches, mean/min/max device time and share of the total.

    python tools/launch_summary.py gpurun_out/launches.csv [--skip-prefix at::] > profiles/…md

ncu launch times are cold-cache and serialised: compare SHARES, not absolutes.
"""
import csv
import sys
from collections import OrderedDict


def load(path):
    lines = [l for l in open(path) if not l.startswith("==")]
    out = []
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "nsecond")
        ns = v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(unit, 1)
        name = r["Kernel Name"].split("(")[0].replace("void ", "").strip()
        out.append((name, r.get("Grid Size", ""), r.get("Block Size", ""), ns))
    return out


def main():
    path = sys.argv[1]
    skip = [a.split("=", 1)[1] for a in sys.argv[2:] if a.startswith("--skip-prefix=")]
    rows = [r for r in load(path) if not any(r[0].startswith(s) for s in skip)]
    agg = OrderedDict()
    for name, grid, block, ns in rows:
        a = agg.setdefault(name, {"n": 0, "sum": 0.0, "min": 1e30, "max": 0.0, "grid": grid, "block": block})
        a["n"] += 1
        a["sum"] += ns
        a["min"] = min(a["min"], ns)
        a["max"] = max(a["max"], ns)
    tot = sum(a["sum"] for a in agg.values()) or 1.0
    print(f"| kernel | grid | block | launches | mean us | min us | max us | share |")
    print(f"|---|---|---|---|---|---|---|---|")
    for name, a in agg.items():
        print(f"| `{name}` | {a['grid']} | {a['block']} | {a['n']} | {a['sum'] / a['n'] / 1e3:.2f} | "
              f"{a['min'] / 1e3:.2f} | {a['max'] / 1e3:.2f} | {100 * a['sum'] / tot:.1f}% |")


if __name__ == "__main__":
    main()
