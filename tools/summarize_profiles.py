"""Summaries under profiles/ from the raw outputs of tools/round_profile.sh
(gpurun_out/): the bench lines, the ncu launch list (per kernel: count, mean,
share of the listed time) and the key metrics of the --set full capture of
the fused kernel; also refreshes profiles/traffic.json, which bench.py reads.

    python tools/summarize_profiles.py [round-tag] [raw-prefix]   (default: round2b r2g,
    the outputs of tools/round2b_profile.sh)
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


def ncu_kernels(rep, match):
    """Key metrics of every captured kernel whose name contains `match` (from the
    report, or from its raw-page CSV exported on the GPU box)."""
    csvp = rep[:-len(".ncu-rep")] + ".raw.csv"
    if os.path.exists(csvp):
        raw = open(csvp).read()
    elif os.path.exists(rep):
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    else:
        return []
    rows = list(csv.reader(io.StringIO(raw)))
    if not rows:
        return []
    h = rows[0]
    out = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        if match in d.get("Kernel Name", ""):
            x = {"kernel": d["Kernel Name"]}
            for k in METRICS + ["sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
                                "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
                                "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
                                "dram__throughput.avg.pct_of_peak_sustained_elapsed",
                                "smsp__average_warp_latency_per_inst_issued.ratio"]:
                v = d.get(k)
                try:
                    x[k] = float(v.replace(",", "")) if v not in (None, "") else None
                except ValueError:
                    x[k] = v
            out.append(x)
    return out


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "round2b"
    pre = os.path.join(RAW, sys.argv[2] if len(sys.argv) > 2 else "r2g")
    os.makedirs(OUT, exist_ok=True)
    res = {}
    for name in ("bench_n1", "bench_C3", "bench_C4", "bench_ref"):
        f = f"{pre}_{name}.json"
        if os.path.exists(f):
            try:
                d = last_json(f)
            except Exception:
                continue
            json.dump(d, open(os.path.join(OUT, f"{tag}_{name.replace('bench_ref', 'bench_reference')}.json"), "w"),
                      indent=1)
            res[name] = d.get("ms_per_step")
    for lname in ("n1", "C3", "C4"):
        f = f"{pre}_launches_{lname}.csv"
        if not os.path.exists(f):
            continue
        ll = launches(f)
        with open(os.path.join(OUT, f"{tag}_launches_{lname}.csv"), "w") as fo:
            w = csv.writer(fo)
            w.writerow(["kernel", "launches", "mean_us", "share_of_listed_time"])
            for x in ll:
                w.writerow([x["kernel"], x["launches"], x["mean_us"], x["share_of_listed_time"]])
        res["launches_" + lname] = ll[:6]
    f = f"{pre}_pytest_gpu.log"
    if os.path.exists(f):
        with open(os.path.join(OUT, f"{tag}_pytest_gpu.log"), "w") as fo:
            fo.write(open(f).read())
    caps = {"v2_C2": ("occ_v2_kernel", "bench.py --config C2"), "v2_T": ("occ_v2_kernel", "bench.py --config T"),
            "phaseA_C3": ("occ_step_kernel", "big_phase_times multi, launch 0"),
            "phaseD_C3": ("occ_step_kernel", "big_phase_times multi, launch 5"),
            "decompress_C3": ("occ_v2_decompress_band", "big_phase_times multi, EF + plain"),
            "phaseF_C4": ("occ_step_kernel", "big_phase_times multi, launch 30 (DP reconstruction, MLP)"),
            "sweep1_C4": ("umma_sweep_kernel", "tools/dp_driver.py: tcgen05 sweep 1, 3072x12288 r64"),
            "sweep2_C4": ("umma_sweep_kernel", "tools/dp_driver.py: tcgen05 sweep 2 (MN-major A), 3072x12288 r64"),
            "recon_C4": ("umma_recon_kernel", "tools/dp_driver.py: tcgen05 DP reconstruction, 3072x12288 r64"),
            "orth_C4": ("occ_step_kernel", "tools/dp_driver.py: Gram + one-CTA factorisation + apply, 3072x12288 r64")}
    ncu = {}
    for key, (match, how) in caps.items():
        rep = f"{pre}_{key}.ncu-rep"
        if os.path.exists(rep) or os.path.exists(f"{pre}_{key}.raw.csv"):
            ncu[key] = {"source": f"ncu --set full --clock-control none --import-source on ({how}); tools/round2b_profile.sh",
                        "kernels": ncu_kernels(rep, match)}
    json.dump(ncu, open(os.path.join(OUT, f"{tag}_ncu_full.json"), "w"), indent=1)
    if "v2_C2" in ncu and ncu["v2_C2"]["kernels"]:
        k = ncu["v2_C2"]["kernels"][0]
        traffic = {"C2": int((k["dram__bytes_read.sum"] + k["dram__bytes_write.sum"]) * 1e6),
                   "_note": ("dram__bytes_read.sum + dram__bytes_write.sum (MB in the ncu report) of the fused "
                             f"kernel on C2 from profiles/{tag}_ncu_full.json (ncu flushes caches before the "
                             "replayed kernel; writes still in L2 at kernel end are not counted).")}
        if "v2_T" in ncu and ncu["v2_T"]["kernels"]:
            kt = ncu["v2_T"]["kernels"][0]
            traffic["T"] = int((kt["dram__bytes_read.sum"] + kt["dram__bytes_write.sum"]) * 1e6)
        json.dump(traffic, open(os.path.join(OUT, "traffic.json"), "w"), indent=1)
    f = f"{pre}_rank_sweep.jsonl"
    if os.path.exists(f):
        with open(os.path.join(OUT, f"{tag}_rank_sweep.jsonl"), "w") as fo:
            fo.write("".join(x for x in open(f) if x.startswith("{")))
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
