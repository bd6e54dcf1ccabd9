"""Summaries under profiles/ from the raw outputs of tools/round_profile.sh
(gpurun_out/): the bench lines, the ncu launch list (per kernel: count, mean,
share of the listed time) and the key metrics of the --set full capture of
the fused kernel; also refreshes profiles/traffic.json, which bench.py reads.

    python tools/summarize_profiles.py [round-tag]     (default: round1)
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RAW = os.path.join(ROOT, "gpurun_out")
OUT = os.path.join(ROOT, "profiles")
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
           "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
           "launch__registers_per_thread"]


def last_json(path):
    with open(path) as f:
        lines = [x for x in f.read().splitlines() if x.startswith("{")]
    return json.loads(lines[-1])


def launches(path):
    txt = open(path).read()
    rows = list(csv.reader(io.StringIO(txt[txt.find('"ID"'):])))
    h = {k: j for j, k in enumerate(rows[0])}
    agg = defaultdict(list)
    for r in rows[1:]:
        if r[h["Metric Name"]] == "gpu__time_duration.sum":
            agg[r[h["Kernel Name"]]].append(float(r[h["Metric Value"]]) / 1e3)   # ns -> us
    total = sum(sum(v) for v in agg.values())
    return [{"kernel": k, "launches": len(v), "mean_us": round(sum(v) / len(v), 3),
             "share_of_listed_time": round(sum(v) / total, 4)} for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))]


def ncu_full(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    for r in rows[2:]:
        d = dict(zip(h, r))
        if "occ_v2" in d.get("Kernel Name", ""):
            out = {"kernel": d["Kernel Name"]}
            for k in METRICS:
                v = d.get(k)
                out[k] = float(v.replace(",", "")) if v not in (None, "") else None
            return out
    return None


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "round1"
    os.makedirs(OUT, exist_ok=True)
    b1 = last_json(os.path.join(RAW, "bench_n1.json"))
    json.dump(b1, open(os.path.join(OUT, f"{tag}_bench_n1.json"), "w"), indent=1)
    ref = os.path.join(RAW, "bench_ref.json")
    if os.path.exists(ref):
        json.dump(last_json(ref), open(os.path.join(OUT, f"{tag}_bench_reference.json"), "w"), indent=1)
    ll = launches(os.path.join(RAW, "launches_n1.csv"))
    with open(os.path.join(OUT, f"{tag}_launches_n1.csv"), "w") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "launches", "mean_us", "share_of_listed_time"])
        for x in ll:
            w.writerow([x["kernel"], x["launches"], x["mean_us"], x["share_of_listed_time"]])
    full = ncu_full(os.path.join(RAW, "prof_bench_n1.ncu-rep"))
    if full:
        full["source"] = ("ncu --set full --clock-control none --import-source on -k regex:occ_v2 --launch-skip 3 -c 1 "
                          "python bench.py --steps 5 --warmup 3 (tools/round_profile.sh)")
        json.dump(full, open(os.path.join(OUT, f"{tag}_ncu_full_v2_n1.json"), "w"), indent=1)
        cfg = b1["config"]
        key = f"{cfg['n']}x{cfg['m']}x{cfg['rank']}"
        traffic = {key: int((full["dram__bytes_read.sum"] + full["dram__bytes_write.sum"]) * 1e6),
                   "_note": ("dram__bytes_read.sum + dram__bytes_write.sum (MB in the ncu report) of the fused "
                             f"kernel from profiles/{tag}_ncu_full_v2_n1.json. Writes of e_new/M' still resident in L2 "
                             "at kernel end are written back after the kernel and are not counted.")}
        json.dump(traffic, open(os.path.join(OUT, "traffic.json"), "w"), indent=1)
    print(json.dumps({"bench": b1["ms_per_step"], "launches": ll[:3], "ncu": full}, indent=1))


if __name__ == "__main__":
    main()
