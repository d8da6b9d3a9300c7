"""Summarise an ncu report (details page + per-source-line stall samples) as JSON/text.
    python scripts/ncu_summary.py gpurun_out/prof_c1.ncu-rep [--top 25] [--json out.json]
"""
import argparse
import csv
import io
import json
import subprocess

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread", "Theoretical Occupancy",
        "Achieved Occupancy", "Achieved Active Warps Per SM", "Waves Per SM", "Block Limit Registers",
        "Block Limit Shared Mem", "Dynamic Shared Memory Per Block", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "Grid Size", "Block Size"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__inst_executed.sum", "smsp__inst_executed.sum"]


def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=25)
    ap.add_argument("--json")
    a = ap.parse_args()
    out = {"report": a.rep, "details": {}, "raw": {}, "hot_lines": []}
    rows = list(csv.reader(io.StringIO(run([a.rep, "--page", "details", "--csv"]))))
    h = rows[0]
    out["kernel"] = rows[1][h.index("Kernel Name")]
    for r in rows[1:]:
        name = r[h.index("Metric Name")]
        if name in KEYS:
            out["details"][name] = f"{r[h.index('Metric Value')]} {r[h.index('Metric Unit')]}".strip()
    raw = list(csv.reader(io.StringIO(run([a.rep, "--page", "raw", "--csv"]))))
    for i, name in enumerate(raw[0]):
        if name in RAW:
            out["raw"][name] = f"{raw[2][i]} {raw[1][i]}".strip()
    src = list(csv.reader(io.StringIO(run([a.rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]))))
    agg, f = [], None
    for r in src:
        if not r:
            continue
        if r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name", "Line No") or len(r) < 8 or r[2] != "-":
            continue
        try:
            agg.append((f, int(r[0]), r[1].strip()[:100], float(r[4] or 0), float(r[7] or 0)))
        except ValueError:
            pass
    ts = sum(x[3] for x in agg) or 1.0
    ti = sum(x[4] for x in agg) or 1.0
    for x in sorted(agg, key=lambda x: -x[3])[:a.top]:
        out["hot_lines"].append({"file": x[0], "line": x[1], "stall_pct": round(100 * x[3] / ts, 2),
                                 "inst_pct": round(100 * x[4] / ti, 2), "src": x[2]})
    out["inst_executed_warp"] = ti
    if a.json:
        with open(a.json, "w") as fh:
            json.dump(out, fh, indent=1)
    print(out["kernel"])
    for k, v in out["details"].items():
        print(f"  {k}: {v}")
    for k, v in out["raw"].items():
        print(f"  {k}: {v}")
    for x in out["hot_lines"]:
        print(f"  {x['file']:18s}{x['line']:5d} stall {x['stall_pct']:5.1f}% inst {x['inst_pct']:5.1f}%  {x['src']}")


if __name__ == "__main__":
    main()
