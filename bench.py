#!/usr/bin/env python
"""Benchmark of the Optimus-CC compression hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N = 1: the 1-GPU compress+decompress step (occ_compress: a1-a9) on
BASELINE.json configs[1], the GPT-2.5B-shaped inter-stage tensor
(1024 tokens x micro-batch 4) x 1920 hidden = 4096 x 1920 fp32 at rank 16.
N > 1 (torchrun, one rank per GPU): weak scaling of the pipeline backward link
in its 1F1B steady state (concurrent sender -> receiver
pairs), as a ring: every rank compresses its own 4096 x 1920 gradient and
sends the factors to rank - 1 while receiving rank + 1's factors and
decompressing them (occ_sendrecv_factors, one NCCL group over NVLink).
--mode dp instead runs the data-parallel step (occ_allreduce_factors:
ncclAllReduce of P then of Q).
--impl reference: the fp64 CPU oracle (oracle/) timed on the host cores on the
same workload (the reference arm of this paper-only tier; rank 0 only).

One JSON line on rank 0.  L2 is flushed (a clean read of 2x the L2 size)
before every timed step; each step is timed with CUDA events on the launching
stream; the reported time is the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "compress+decompress GB/s per B200 (% of HBM peak); factor comm µs at 1/2/4/8 GPUs"
N_ROWS, N_COLS, RANK = 4096, 1920, 16            # BASELINE.json configs[1] (reading C6: 1024*4 x 1920)
T_ROWS, T_COLS = 1024, 3072                      # north-star target T (1024 x 3072, r = 16)
WORKLOAD = ("GPT-2.5B-shaped inter-stage backprop tensor (1024 tokens x micro-batch 4 = 4096 rows x "
            "1920 hidden, fp32), rank 16, error feedback, 1 step = P=(M+e)Q, orth, Q=(M+e)^T P, M', e_new")


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def alg_bytes(n, m, m_bytes=4, dp=False):
    """Algorithmic HBM bytes of one step: read M, read e, write e_new,
    write M' (+ the r(n+m) fp32 factors, read Q_prev / write P, Q)."""
    return n * m * (2 * m_bytes + 8) + RANK * (n + 2 * m) * 4


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x1: "gpu_idle", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, dev_index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(s)}


def cpu_threads():
    try:
        from threadpoolctl import threadpool_info
        return max(x["num_threads"] for x in threadpool_info())
    except Exception:
        return os.cpu_count()


def make_inputs(n, m, seed=1000 * 2):
    from workloads import synth
    M = synth.d2_gradlike(n, m, seed)
    e = synth.e0(n, m, seed + 1, like=M)
    Q0 = synth.q0(m, RANK, 7)   # same on every rank (reading C5)
    return M, e, Q0


def run_oracle(n, m, steps, budget_s):
    """Oracle (oracle/, as it stands) on this workload; returns (s/step, steps run)."""
    import oracle
    M, e, Q0 = make_inputs(n, m)
    done, t0 = 0, time.perf_counter()
    while done < steps:
        o = oracle.compress_step(M, e, Q0)
        e, Q0 = o["err"], o["Q"]
        done += 1
        if time.perf_counter() - t0 > budget_s:
            break
    return (time.perf_counter() - t0) / done, done


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    n, m = N_ROWS, N_COLS
    # torchrun exports OMP_NUM_THREADS=1; rank 0 alone runs the oracle, so give it
    # every host core it may use, as at N=1.
    import numpy  # noqa: F401  (load its BLAS before the limit is raised)
    from threadpoolctl import threadpool_limits
    with threadpool_limits(limits=len(os.sched_getaffinity(0))):
        run_oracle(n, m, args.warmup, 60.0)
        dt, done = run_oracle(n, m, args.steps, 240.0)
        cores = cpu_threads()
    gbs = n * m * 4 / dt / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": args.gpus,
            "steps": done, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "n": n, "m": m, "rank": RANK, "parallelism": "cpu"},
            "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": cores, "kind": "oracle",
                             "sample": f"{done} full oracle steps (NumPy fp64) of the {n}x{m} r={RANK} workload"},
            "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-target", action="store_true", help="skip the 1024x3072 north-star line")
    ap.add_argument("--mode", default="pp", choices=["pp", "dp"],
                    help="N > 1: pipeline ring (occ_sendrecv_factors, default) or data-parallel allreduce")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        return reference_arm(args)

    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2301_09830_b200 import build as occ_build
    from paper_2301_09830_b200 import occ

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"warning: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    if rank == 0:
        occ_build.build()
    if world > 1:
        dist.barrier()
    occ.lib()
    stream = torch.cuda.current_stream()
    hbm_peak, peak_kind = peaks()
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(2 * l2 // 4, dtype=torch.float32, device=dev).uniform_()
    sink = torch.empty(1, device=dev)

    def flush_l2():
        torch.sum(flush, dim=0, out=sink[0])   # clean read of 2x L2: no dirty lines left behind

    comm = occ.Comm.from_process_group() if world > 1 else None

    mode = "1gpu" if world == 1 else args.mode
    dp = mode == "dp"
    snd_peer, rcv_peer = (rank - 1) % world, (rank + 1) % world   # pp ring

    def bench_shape(n, m, steps, warmup, mode):
        dp = mode == "dp"
        M, e, Q0 = make_inputs(n, m, seed=2000 + 10 * rank)
        Md = torch.from_numpy(M).to(dev)
        Ed = torch.from_numpy(e).to(dev)
        Qd = torch.from_numpy(Q0).to(dev)
        Pd = torch.empty(n, RANK, device=dev)
        Rd = torch.empty_like(Md)            # M' (1gpu) / the received stage's M' (pp)
        Pr = torch.empty(n, RANK, device=dev)
        Qr = torch.empty(m, RANK, device=dev)
        ws = occ.alloc_workspace(n, m, RANK, device=dev)
        Mkeep = Md.clone()

        def step():
            if dp:
                Md.copy_(Mkeep)   # G is overwritten in place by M'; restored outside the timing
                return lambda: occ.occ_allreduce_factors([Md], [Ed], [Qd], [Pd], RANK, 1.0 / world,
                                                         comm=comm, ws=ws)
            if mode == "pp":
                return lambda: occ.occ_sendrecv_factors(Md, Ed, Qd, Pd, RANK, snd_peer, Rd, Pr, Qr, rcv_peer,
                                                        comm, ws=ws)
            return lambda: occ.occ_compress(Md, Ed, Qd, Pd, Rd, r=RANK, ws=ws)

        for _ in range(warmup):
            flush_l2()
            step()()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        sampler = ClockSampler(local)
        with sampler:
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            for i in range(steps):
                call = step()
                flush_l2()
                ev[i][0].record(stream)
                call()
                ev[i][1].record(stream)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
        times = [a.elapsed_time(b) for a, b in ev]   # ms
        tot = torch.tensor([sum(times)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tot, op=dist.ReduceOp.MAX)
        ms = tot.item() / steps
        stats = occ.occ_read_stats(ws)
        return {"ms": ms, "times": times, "clocks": sampler.summary(), "stats": stats,
                "bufs": (Md, Ed, Qd, Pd, Rd, ws, Mkeep, Pr, Qr)}

    n, m = N_ROWS, N_COLS
    res = bench_shape(n, m, args.steps, args.warmup, mode)
    ms = res["ms"]
    value = world * n * m * 4 / (ms * 1e-3) / 1e9               # GB/s uncompressed, whole job
    ab = alg_bytes(n, m)
    achieved = ab / (ms * 1e-3) / 1e9
    launches_per_step = 1 if res["stats"]["path"] in (1, 3) else 9
    if dp:
        launches_per_step = 3
    elif mode == "pp":
        launches_per_step = 2   # fused compress + decompress (NCCL's send/recv kernels are not ours)

    # e2e through the public API with HOST buffers: every step copies its M in
    # (pinned host -> device), runs the step and copies its M' out.  The copies
    # run on their own streams with M and M' double-buffered on the device, so
    # step k's D2H overlaps step k+1's H2D (PCIe is full duplex); the events
    # order H2D -> step -> D2H per step and stop a buffer being overwritten
    # before the step / copy that reads it has finished.
    Md, Ed, Qd, Pd, Rd, ws, Mkeep, Pr, Qr = res["bufs"]
    Mh = torch.from_numpy(make_inputs(n, m, seed=2000 + 10 * rank)[0]).pin_memory()
    Rh = torch.empty(n, m, dtype=torch.float32).pin_memory()
    nbuf = int(os.environ.get("OCC_E2E_NBUF", "2"))
    Mb = [Md] + [torch.empty_like(Md) for _ in range(nbuf - 1)]
    Rb = [Rd] + [torch.empty_like(Rd) for _ in range(nbuf - 1)]
    h2d_s, d2h_s = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    e2e_steps = max(3, min(args.steps, 20))

    def e2e_run(k_steps):
        ev = [[torch.cuda.Event() for _ in range(3)] for _ in range(k_steps)]   # H2D done, step done, D2H done
        h2d_s.wait_stream(stream)   # the first copy starts after the caller's start event
        for k in range(k_steps):
            b = k % nbuf
            if k >= nbuf:   # buffer b was last read by step k-nbuf (and, for DP, by its D2H)
                h2d_s.wait_event(ev[k - nbuf][2] if dp else ev[k - nbuf][1])
            with torch.cuda.stream(h2d_s):
                Mb[b].copy_(Mh, non_blocking=True)
            ev[k][0].record(h2d_s)
            stream.wait_event(ev[k][0])
            if k >= nbuf:
                stream.wait_event(ev[k - nbuf][2])   # M'[b] of step k-nbuf copied out
            if dp:
                occ.occ_allreduce_factors([Mb[b]], [Ed], [Qd], [Pd], RANK, 1.0 / world, comm=comm, ws=ws)
                out = Mb[b]
            elif mode == "pp":
                occ.occ_sendrecv_factors(Mb[b], Ed, Qd, Pd, RANK, snd_peer, Rb[b], Pr, Qr, rcv_peer, comm, ws=ws)
                out = Rb[b]
            else:
                occ.occ_compress(Mb[b], Ed, Qd, Pd, Rb[b], r=RANK, ws=ws)
                out = Rb[b]
            ev[k][1].record(stream)
            d2h_s.wait_event(ev[k][1])
            with torch.cuda.stream(d2h_s):
                Rh.copy_(out, non_blocking=True)
            ev[k][2].record(d2h_s)
        stream.wait_stream(d2h_s)
        stream.wait_stream(h2d_s)

    e2e_run(2)   # warm-up
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    e2e_run(e2e_steps)
    t1.record(stream)
    torch.cuda.synchronize()
    e_tot = torch.tensor([t0.elapsed_time(t1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e_tot, op=dist.ReduceOp.MAX)
    e_ms = e_tot.item() / e2e_steps
    e2e = {"value": world * n * m * 4 / (e_ms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": e_ms,
           "h2d_bytes_per_step": n * m * 4, "d2h_bytes_per_step": n * m * 4}

    # factor communication alone (a3 + a6 message sizes), NCCL over NVLink
    comm_us = 0.0
    if dp:
        pbuf = torch.zeros(n * RANK, device=dev)
        qbuf = torch.zeros(m * RANK, device=dev)
        for _ in range(5):
            dist.all_reduce(pbuf)
            dist.all_reduce(qbuf)
        torch.cuda.synchronize()
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 50
        c0.record()
        for _ in range(reps):
            dist.all_reduce(pbuf)
            dist.all_reduce(qbuf)
        c1.record()
        torch.cuda.synchronize()
        ct = torch.tensor([c0.elapsed_time(c1) / reps * 1e3], dtype=torch.float64, device=dev)
        dist.all_reduce(ct, op=dist.ReduceOp.MAX)
        comm_us = ct.item()
    elif mode == "pp":   # the grouped factor send/recv alone (P n x r + Q m x r each way)
        bufs = [torch.zeros(n * RANK, device=dev), torch.zeros(m * RANK, device=dev),
                torch.zeros(n * RANK, device=dev), torch.zeros(m * RANK, device=dev)]

        def xchg():
            ops = [dist.P2POp(dist.isend, bufs[0], snd_peer), dist.P2POp(dist.isend, bufs[1], snd_peer),
                   dist.P2POp(dist.irecv, bufs[2], rcv_peer), dist.P2POp(dist.irecv, bufs[3], rcv_peer)]
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        for _ in range(5):
            xchg()
        torch.cuda.synchronize()
        dist.barrier()
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 50
        c0.record()
        for _ in range(reps):
            xchg()
        c1.record()
        torch.cuda.synchronize()
        ct = torch.tensor([c0.elapsed_time(c1) / reps * 1e3], dtype=torch.float64, device=dev)
        dist.all_reduce(ct, op=dist.ReduceOp.MAX)
        comm_us = ct.item()

    # north-star target T on one GPU (reported beside the headline)
    target = None
    if not args.no_target and world == 1:
        t = bench_shape(T_ROWS, T_COLS, args.steps, args.warmup, "1gpu")
        tab = alg_bytes(T_ROWS, T_COLS)
        target = {"workload": "north-star T: 1024 x 3072 fp32, rank 16, 1 GPU", "ms_per_step": t["ms"],
                  "value": T_ROWS * T_COLS * 4 / (t["ms"] * 1e-3) / 1e9, "unit": "GB/s",
                  "roofline_frac": tab / (t["ms"] * 1e-3) / 1e9 / hbm_peak}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        dt, done = run_oracle(n, m, 1000, 12.0)
        cpu = {"value": n * m * 4 / dt / 1e9, "unit": "GB/s", "cores": cpu_threads(), "kind": "oracle",
               "sample": f"{done} oracle steps (NumPy fp64, ~12 s budget) of the same {n}x{m} r={RANK} workload"}

    traffic = None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(f"{n}x{m}x{RANK}" + ("" if mode == "1gpu" else "_" + mode))
        except Exception:
            traffic = None

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": WORKLOAD + {"1gpu": "",
                                                "pp": f"; pipeline backward link, ring of {world} stages: compress + send factors to rank-1, receive rank+1's factors + decompress (1F1B steady state)",
                                                "dp": f"; data-parallel allreduce of P and Q over {world} ranks"}[mode],
                       "n": n, "m": m, "rank": RANK, "M_dtype": "f32",
                       "parallelism": {"1gpu": "1gpu", "pp": f"pp-ring{world}", "dp": f"dp{world}"}[mode],
                       "l2": "flushed before every step",
                       "path": {1: "v1 fused persistent kernel", 3: "fused TMEM-resident persistent kernel"}.get(res["stats"]["path"], "per-phase launches")},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "traffic": traffic, "peak_kind": peak_kind,
                         "alg_bytes_per_launch": ab,
                         "kernel": {"1gpu": "occ_v2_kernel (fused step)", "pp": "step (fused compress + NCCL send/recv + decompress)",
                                    "dp": "step (3 launches + 2 NCCL allreduces)"}[mode]},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": res["clocks"],
            "factor_comm_us": comm_us,
            "orth": {"second_pass": res["stats"]["second_pass"], "kappa_est": res["stats"]["kappa_est"],
                     "fallback_columns": res["stats"]["fallback_columns"]},
        }
        if target:
            line["north_star_target"] = target
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.destroy()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
