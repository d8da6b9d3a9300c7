"""Writes profiles/ncu_counters.json (the per-launch counters bench.py's roofline reads) from ncu
--set full captures of this build:
    python scripts/counters_from_ncu.py --c1 gpurun_out/prof_r02_c1.ncu-rep [--c2 prof_c2.ncu-rep]
        [--c3 c3_metrics.csv]   (a --metrics launch list of k_step_warp over whole C3 runs)
        [--c4 c4_metrics.csv]   (a --metrics launch list of the k_det_* kernels of C4 runs)"""
import argparse
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    d = {}
    for i, name in enumerate(rows[0]):
        d[name] = (rows[2][i], rows[1][i])
    return d


def num(v, unit):
    x = float(v)
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c1")
    ap.add_argument("--c2")
    ap.add_argument("--c3")
    ap.add_argument("--c4")
    a = ap.parse_args()
    path = os.path.join(ROOT, "profiles", "ncu_counters.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    if a.c1:
        r = raw(a.c1)
        out["k_step_warp:1024x128x128x200"] = {
            "inst_executed_per_launch": num(*r["smsp__inst_executed.sum"]),
            "dram_bytes_per_launch": num(*r["dram__bytes_read.sum"]) + num(*r["dram__bytes_write.sum"]),
            "duration_us_cold": num(*r["gpu__time_duration.sum"]),
            "source": os.path.basename(a.c1)}
    if a.c2:
        r = raw(a.c2)
        out["k_rl_tanker_warp:16384x64x64x256"] = {
            "dram_bytes_per_launch": num(*r["dram__bytes_read.sum"]) + num(*r["dram__bytes_write.sum"]),
            "inst_executed_per_launch": num(*r["smsp__inst_executed.sum"]),
            "source": os.path.basename(a.c2)}
    if a.c3:
        # per-launch rows of one metric each; one C3 run = ceil(500 / 16) = 32 step launches
        launches = {}
        for r in csv.DictReader(l for l in open(a.c3) if l.startswith('"')):
            if "k_step_warp" not in r["Kernel Name"]:
                continue
            launches.setdefault(int(r["ID"]), {})[r["Metric Name"]] = num(r["Metric Value"].replace(",", ""), r["Metric Unit"])
        ids = sorted(launches)[:32]  # the first run
        tot = lambda k: sum(launches[i].get(k, 0.0) for i in ids)
        out["k_step_warp:c3:16384x16384x500"] = {
            "inst_executed_per_run": tot("smsp__inst_executed.sum"),
            "dram_bytes_per_run": tot("dram__bytes_read.sum") + tot("dram__bytes_write.sum"),
            "duration_us_cold_per_run": tot("gpu__time_duration.sum") / 1e3,
            "launches": len(ids), "source": os.path.basename(a.c3)}
    if a.c4:
        # one C4 run (256 x 128^2 x 100): the forward launches, the p_bd pass, the loss, the backward launches and
        # the gradient reduction, up to the 100th backward launch and the reduction after it
        launches = {}
        for r in csv.DictReader(l for l in open(a.c4) if l.startswith('"')):
            if "k_det_" not in r["Kernel Name"]:
                continue
            d = launches.setdefault(int(r["ID"]), {"name": r["Kernel Name"]})
            d[r["Metric Name"]] = num(r["Metric Value"].replace(",", ""), r["Metric Unit"])
        ids, n_back = [], 0
        order = sorted(launches)
        fwd = ["k_det_forward" in launches[i]["name"] for i in order]
        start = next(j for j in range(len(order)) if all(fwd[j:j + 100]) and len(fwd[j:j + 100]) == 100)
        for i in order[start:]:  # (the bench's short preparation calls before the run are skipped)
            nm = launches[i]["name"]
            if n_back == 100 and "reduce" not in nm:
                break
            ids.append(i)
            n_back += "k_det_back" in nm
            if n_back == 100 and "reduce" in nm:
                break
        tot = lambda k, f="": sum(launches[i].get(k, 0.0) for i in ids if f in launches[i]["name"])
        dram = lambda f="": tot("dram__bytes_read.sum", f) + tot("dram__bytes_write.sum", f)
        out["c4:256x128x128x100"] = {
            "dram_bytes_per_run": dram(),
            "dram_bytes_forward_per_run": dram("k_det_forward"),
            "dram_bytes_backward_per_run": dram("k_det_back"),
            "duration_us_cold_per_run": tot("gpu__time_duration.sum") / 1e3,
            "launches": len(ids), "backward_launches": n_back, "source": os.path.basename(a.c4)}
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
