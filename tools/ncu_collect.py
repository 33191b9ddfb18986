"""Fold the ncu evidence of tools/ncu_all.sh into profiles/ (run here, after the gpurun call):

    python tools/ncu_collect.py [cfg ...]

Per config: profiles/r02_ncu_<cfg>.json (tools/ncu_summary.py of the --set full capture) and
the decode kernel's mean duration and DRAM bytes per launch over the launch list, merged into
profiles/decode_ncu_summary.json (bench.py reads `dram_bytes_per_launch` from it for
roofline.traffic) and printed as a markdown table.
"""
import csv
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
NCU = ROOT / "gpurun_out" / "ncu"
SUMMARY = ROOT / "profiles" / "decode_ncu_summary.json"
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1, "nsecond": 1e-3, "msecond": 1e3,
         "ns": 1e-3, "us": 1, "ms": 1e3}


def launches(cfg):
    rows = [r for r in csv.reader(open(NCU / f"{cfg}_launches.csv")) if r]
    hdr = next(r for r in rows if "Kernel Name" in r and "Metric Name" in r)
    ik, im, iu, iv, iid = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "ID"))
    per = {}
    for r in rows[rows.index(hdr) + 1:]:
        if len(r) <= iv:
            continue
        v = float(r[iv].replace(",", "")) * SCALE.get(r[iu], 1)
        per.setdefault((r[iid], r[ik]), {})[r[im]] = v
    ids = sorted(int(i) for (i, k) in per if "spin_kernel" in k)
    lo, hi = (ids[0], ids[1]) if len(ids) > 1 else (ids[0] if ids else -1, 1 << 30)
    dec = [m for (i, k), m in per.items() if "decode" in k and lo < int(i) < hi]  # the timed steps' launches
    return per, dec


def main():
    cfgs = sys.argv[1:] or sorted(p.stem for p in NCU.glob("*.ncu-rep"))
    summary = json.loads(SUMMARY.read_text()) if SUMMARY.exists() else {}
    print("| config | decode launches | us per launch (ncu, serialised) | DRAM bytes per launch | share of kernel time |")
    print("|---|---|---|---|---|")
    for cfg in cfgs:
        rep = NCU / f"{cfg}.ncu-rep"
        if rep.exists():
            out = subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_summary.py"), str(rep), "decode"],
                                 capture_output=True, text=True).stdout
            (ROOT / "profiles" / f"r02_ncu_{cfg}.json").write_text(out)
        per, dec = launches(cfg) if (NCU / f"{cfg}_launches.csv").exists() else ({}, [])
        if not dec:  # the launch list ended before the timed steps (many replicas to build):
            full = ROOT / "profiles" / f"r02_ncu_{cfg}.json"  # the --set full capture's launch
            if full.exists() and full.stat().st_size > 0:
                pl = json.loads(full.read_text())["per_launch"][0]
                summary[cfg] = {"kernel": pl["kernel"], "dram_bytes_per_launch": round(pl["dram_bytes"]),
                                "us_per_launch_ncu": pl["us"], "launches_averaged": 1,
                                "source": f"ncu --set full of one decode launch of bench.py --config {cfg} "
                                          "(tools/ncu_all.sh), round 2"}
                print(f"| {cfg} | 1 (--set full) | {pl['us']:.1f} | {pl['dram_bytes'] / 1e6:.2f} MB | - |")
            continue
        us = sum(m.get("gpu__time_duration.sum", 0) for m in dec) / len(dec)
        byts = sum(m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0) for m in dec) / len(dec)
        # the decode's share of the timed region's kernel time: bench.py brackets the timed
        # steps with host-run-ahead spins (the first spin_kernel before, the second after)
        ids = sorted(((int(i), k, m) for (i, k), m in per.items()), key=lambda x: x[0])
        spins = [i for i, k, m in ids if "spin_kernel" in k]
        lo, hi = (spins[0], spins[1]) if len(spins) > 1 else (spins[0] if spins else -1, 1 << 30)
        path = [(k, m) for i, k, m in ids if lo < i < hi]
        tot = sum(m.get("gpu__time_duration.sum", 0) for k, m in path)
        share = sum(m.get("gpu__time_duration.sum", 0) for k, m in path if "decode" in k) / tot
        summary[cfg] = {"kernel": "decode_tc_kernel (fused decode + append step)",
                        "dram_bytes_per_launch": round(byts), "us_per_launch_ncu": round(us, 2),
                        "launches_averaged": len(dec),
                        "source": f"ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                                  f"--clock-control none of bench.py --config {cfg} (tools/ncu_all.sh), round 2"}
        print(f"| {cfg} | {len(dec)} | {us:.1f} | {byts / 1e6:.2f} MB | {share:.2f} |")
    SUMMARY.write_text(json.dumps(summary, indent=1) + "\n")


if __name__ == "__main__":
    main()
