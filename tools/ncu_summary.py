"""Condense one kernel of an `ncu --set full` report into the JSON kept under profiles/.

    python tools/ncu_summary.py gpurun_out/prof_decode.ncu-rep [kernel-regex] > profiles/r01_ncu_x.json

Reads `ncu -i <rep> --page raw --csv` (first matching launch) and the SASS source page
(warp-stall samples per instruction, top 12). Metrics: duration, DRAM bytes, throughput
fractions, issue activity, pipe utilisation, occupancy and the stall breakdown.
"""
import csv
import io
import json
import re
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_imma.avg.pct_of_peak_sustained_active",
]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True, check=True).stdout


def main():
    rep = sys.argv[1]
    pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    hdr, units = rows[0], rows[1]
    matching = [r for r in rows[2:] if not pat or pat.search(r[hdr.index("Kernel Name")])]
    launch = matching[0]
    col = dict(zip(hdr, launch))
    unit = dict(zip(hdr, units))
    out = {"kernel": col["Kernel Name"][:160], "launches_in_report": len(matching)}
    # every launch of the report (a balanced decode is two grids): durations and DRAM bytes
    def num(r, k):
        try:
            return float(r[hdr.index(k)].replace(",", ""))
        except (ValueError, IndexError):
            return 0.0
    out["per_launch"] = [{"kernel": r[hdr.index("Kernel Name")][:80], "grid": r[hdr.index("Grid Size")] if "Grid Size" in hdr else None,
                          "us": num(r, "gpu__time_duration.sum"),
                          "dram_bytes": num(r, "dram__bytes_read.sum") * (1e6 if unit.get("dram__bytes_read.sum") == "Mbyte" else 1)
                          + num(r, "dram__bytes_write.sum") * (1e6 if unit.get("dram__bytes_write.sum") == "Mbyte" else
                                                                1e3 if unit.get("dram__bytes_write.sum") == "Kbyte" else 1)}
                         for r in matching]
    for k in KEYS:
        if k in col:
            v = col[k].replace(",", "")
            try:
                v = float(v)
            except ValueError:
                pass
            out[k] = v if not unit.get(k) else {"value": v, "unit": unit[k]}
    stalls = {k.split("issue_stalled_")[1].split("_per_issue")[0]: float(col[k])
              for k in hdr if "average_warps_issue_stalled" in k and k.endswith("per_issue_active.ratio")
              and col.get(k, "").replace(".", "", 1).isdigit() and float(col[k]) >= 0.05}
    out["stall_cycles_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass"))))
    h = next(r for r in src if "Warp Stall Sampling (All Samples)" in r)
    i_s, i_e = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    body = [r for r in src[src.index(h) + 1:] if len(r) > i_s and r[i_s].replace(".", "", 1).isdigit()]
    tot = sum(float(r[i_s]) for r in body) or 1.0
    top = sorted(body, key=lambda r: -float(r[i_s]))[:12]
    out["stall_samples_top"] = [{"sass": r[1].strip()[:60], "share": round(float(r[i_s]) / tot, 4),
                                 "executed": r[i_e]} for r in top]
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
