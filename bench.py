#!/usr/bin/env python
"""Benchmark of the Optimus-CC compression hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

A "step" is one pass of the hot path (a1-a9) over one matrix
(or one DP bucket) of synthetic input, through the C-ABI (libocc.so):

  C1  128 x 256 fp32 r4                 occ_compress (+ M')        BASELINE configs[0]
  C2  4096 x 1920 fp32 r16 (default)    occ_compress (+ M')        configs[1], the metric's workload
  T   1024 x 3072 fp32 r16              occ_compress (+ M')        north-star target
  C3  8192 x 3072 fp32 r32              sender occ_compress + receiver occ_decompress   configs[2]
  C4  {3072 x 12288, 3072 x 9216} r64   occ_allreduce_factors (one DP bucket)           configs[3]

N = 1: the step on one GPU.  N > 1 (torchrun, one rank per GPU, NCCL): weak
scaling.  C1/C2/T/C3 run the pipeline backward link in its 1F1B steady state
as a ring (occ_sendrecv_factors: compress + send the factors to rank - 1,
receive rank + 1's and decompress them); C4 runs the data-parallel step over
all ranks (allreduce of P, then of Q).

Timing (all on the device, CUDA events on the launching stream, max over ranks):
  * value / ms_per_step: K steps back to back over rotating input sets whose
    total size exceeds 3x L2 (every step reads cold inputs from HBM, and pays
    for the write-back of earlier steps' dirty lines, as in steady state);
  * per_step: the same step timed alone K times after an L2 flush (a write
    of 2x L2), median / p10 / p90;
  * factor_comm_us (N > 1): the exchange alone through the library
    (occ_sendrecv_factors with M = NULL / out = NULL, or the two DP allreduces
    of occ_allreduce_factors' message sizes), beside the NVLink bandwidth
    measured in the same run (1 GiB all-reduce and 1 GiB ring send/recv);
  * e2e: the same step through the public API with pinned HOST buffers,
    H2D of M and D2H of M' inside the timed region.
--impl reference: the fp64 CPU oracle (oracle/) on the same config on the host
cores (the reference arm of this paper-only tier; rank 0 only).
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

CONFIGS = {
    "C1": {"shapes": [(128, 256)], "r": 4, "kind": "1gpu",
           "desc": "BASELINE configs[0]: single activation-gradient matrix 128x256 fp32, rank 4"},
    "C2": {"shapes": [(4096, 1920)], "r": 16, "kind": "1gpu",
           "desc": "BASELINE configs[1]: GPT-2.5B-shaped inter-stage backprop tensor (1024 tokens x micro-batch 4 "
                   "= 4096 rows x 1920 hidden, fp32), rank 16"},
    "T": {"shapes": [(1024, 3072)], "r": 16, "kind": "1gpu",
          "desc": "north-star T: 1024 x 3072 activation-gradient tensor fp32, rank 16"},
    "C3": {"shapes": [(8192, 3072)], "r": 32, "kind": "pp",
           "desc": "BASELINE configs[2]: GPT-8.3B-shaped inter-stage tensor (1024 tokens x micro-batch 8 = 8192 x 3072 "
                   "fp32), rank 32, sender compress + receiver decompress"},
    "C4": {"shapes": [(3072, 12288), (3072, 9216)], "r": 64, "kind": "dp",
           "desc": "BASELINE configs[3]: data-parallel compression of the 8.3B-shaped MLP (3072x12288) and QKV "
                   "(3072x9216) weight gradients as one bucket, fp32, rank 64, allreduce(P) then allreduce(Q)"},
}
STEP_DESC = "1 step = A=M+e, P=AQ, orth(P), Q=A^T P, exchange, M'=P Q^T, e_new=A-M' (a1-a9)"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def alg_bytes(cfg, world):
    """Algorithmic HBM bytes of one step per GPU:
    read M and e, write e_new and M' (fp32: 16 B/elt; the PP sender 12 B/elt and the
    receiver 4 B/elt, 16 together on a ring rank or the N = 1 sender+receiver pair;
    the DP rank 16 B/elt, G overwritten by M'), plus the factors r(n + m) x 4 B
    read (Q_prev) and written (P_hat, Q) once each."""
    r = cfg["r"]
    tot = 0
    for n, m in cfg["shapes"]:
        tot += n * m * 16 + r * (n + 2 * m) * 4
    return tot


def elems(cfg):
    return sum(n * m for n, m in cfg["shapes"])


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
            time.sleep(0.001)

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


def make_inputs(n, m, r, seed):
    from workloads import synth
    M = synth.d2_gradlike(n, m, seed)
    e = synth.e0(n, m, seed + 1, like=M)
    Q0 = synth.q0(m, r, 7)   # same on every rank (reading C5)
    return M, e, Q0


def run_oracle(cfg, steps, budget_s, world=1):
    """The oracle (oracle/, as it stands) on this config: returns (s/step, steps run).
    C4 simulates the DP group of `world` ranks in-process (oracle.dp_step)."""
    import oracle
    r = cfg["r"]
    ins = [make_inputs(n, m, r, 2000 + 17 * i) for i, (n, m) in enumerate(cfg["shapes"])]
    done, t0 = 0, time.perf_counter()
    while done < steps:
        for i, (M, e, Q0) in enumerate(ins):
            if cfg["kind"] == "dp":
                o = oracle.dp_step([M] * world, [e] * world, Q0, scale=1.0 / world)
                ins[i] = (M, o["err"][0], o["Q"])
            else:
                o = oracle.compress_step(M, e, Q0)
                if cfg["kind"] == "pp":
                    oracle.decompress(o["P_hat"], o["Q"])   # the receiver's M'
                ins[i] = (M, o["err"], o["Q"])
        done += 1
        if time.perf_counter() - t0 > budget_s:
            break
    return (time.perf_counter() - t0) / done, done


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = CONFIGS[args.config]
    import numpy  # noqa: F401  (load its BLAS before the limit is raised)
    from threadpoolctl import threadpool_limits
    # torchrun exports OMP_NUM_THREADS=1; rank 0 alone runs the oracle: give it every core
    with threadpool_limits(limits=len(os.sched_getaffinity(0))):
        run_oracle(cfg, args.warmup, 60.0)
        dt, done = run_oracle(cfg, args.steps, 240.0)
        cores = cpu_threads()
    gbs = elems(cfg) * 4 / dt / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": args.gpus,
            "steps": done, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(args.config, 1, "cpu"),
            "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": cores, "kind": "oracle",
                             "sample": f"{done} full oracle steps (NumPy fp64) of the {args.config} workload"},
            "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def config_dict(name, world, parallelism):
    cfg = CONFIGS[name]
    return {"workload": cfg["desc"] + "; " + STEP_DESC, "config": name,
            "shapes": [list(s) for s in cfg["shapes"]], "rank": cfg["r"], "M_dtype": "f32",
            "parallelism": parallelism}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-target", action="store_true", help="skip the north-star T line (C2 only)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="N = 1: time the back-to-back steps eagerly only (default: CUDA-graph replay, eager beside it)")
    ap.add_argument("--exchange", default="link", choices=["link", "nccl"],
                    help="N > 1 pipeline ring: in-kernel NVLink exchange (occ_link, default) or NCCL send/recv")
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
    flush = torch.empty(2 * l2 // 4, dtype=torch.float32, device=dev)
    comm = occ.Comm.from_process_group() if world > 1 else None
    snd_peer, rcv_peer = (rank - 1) % world, (rank + 1) % world   # pp ring
    links = []   # occ_link per input set (N > 1 ring with --exchange link)
    use_link = world > 1 and args.exchange == "link" and CONFIGS[args.config]["kind"] != "dp"
    # DP (C4) with --exchange link: the factor sums in-kernel over NVLink (occ_dplink) at N = 2,
    # where it measured faster than NCCL (47 vs 56 us for the two sums); its one-shot push
    # moves (N - 1) buckets per rank, so N > 2 stays on ncclAllReduce (95 vs 63 us at N = 4)
    dplink = None
    if world == 2 and args.exchange == "link" and CONFIGS[args.config]["kind"] == "dp":
        c4 = CONFIGS[args.config]
        dplink = occ.DpLink.open(comm, max(sum(n for n, _ in c4["shapes"]), sum(m for _, m in c4["shapes"])) * c4["r"])

    def flush_l2():
        flush.fill_(1.0)   # write 2x L2: evicts (and writes back) everything before the timed step

    def max_over_ranks(x):
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def make_step(name, seed_base):
        """Device buffers of one input set and a closure running one step on them."""
        cfg = CONFIGS[name]
        r = cfg["r"]
        mats = []
        for i, (n, m) in enumerate(cfg["shapes"]):
            M, e, Q0 = make_inputs(n, m, r, seed_base + 10 * rank + 17 * i)
            b = {"M": torch.from_numpy(M).to(dev), "E": torch.from_numpy(e).to(dev),
                 "Q": torch.from_numpy(Q0).to(dev), "P": torch.empty(n, r, device=dev),
                 "R": torch.empty(n, m, device=dev), "Pr": torch.empty(n, r, device=dev),
                 "Qr": torch.empty(m, r, device=dev)}
            mats.append(b)
        nmax = max(n for n, _ in cfg["shapes"])
        mmax = max(m for _, m in cfg["shapes"])
        ws = occ.alloc_workspace(nmax, mmax, r, nmat=len(mats), device=dev)
        kind = cfg["kind"]
        link = occ.Link.open(comm, snd_peer, rcv_peer, nmax, mmax, r) if use_link else None
        if link is not None:
            links.append(link)

        def step(Min=None, Rout=None):
            b = mats[0]
            M = b["M"] if Min is None else Min
            R = b["R"] if Rout is None else Rout
            if kind == "dp":
                Gs = [x["M"] for x in mats] if Min is None else [M] + [x["M"] for x in mats[1:]]
                if dplink is not None:
                    occ.occ_allreduce_factors_link(Gs, [x["E"] for x in mats], [x["Q"] for x in mats],
                                                   [x["P"] for x in mats], r, 1.0 / world, dplink, ws=ws)
                else:
                    occ.occ_allreduce_factors(Gs, [x["E"] for x in mats], [x["Q"] for x in mats],
                                              [x["P"] for x in mats], r, 1.0 / world, comm=comm, ws=ws)
                return M
            if world > 1 and link is not None:
                occ.occ_sendrecv_factors_link(M, b["E"], b["Q"], b["P"], r, R, b["Pr"], b["Qr"], link, ws=ws)
                return R
            if world > 1:
                occ.occ_sendrecv_factors(M, b["E"], b["Q"], b["P"], r, snd_peer, R, b["Pr"], b["Qr"], rcv_peer,
                                         comm, ws=ws)
                return R
            if kind == "pp":   # N = 1: the sender's compress, then the receiver's decompress of its factors
                occ.occ_compress(M, b["E"], b["Q"], b["P"], None, r=r, ws=ws)
                occ.occ_decompress(b["P"], b["Q"], R)
                return R
            occ.occ_compress(M, b["E"], b["Q"], b["P"], R, r=r, ws=ws)
            return R
        step.mats, step.ws, step.cfg, step.link = mats, ws, cfg, link
        return step

    def bench_config(name, steps, warmup):
        cfg = CONFIGS[name]
        per_set = elems(cfg) * 12   # M, e, M' (fp32)
        nsets = max(2, int(np.ceil(3 * l2 / per_set)))
        sets = [make_step(name, 2000 + 1000 * k) for k in range(nsets)]
        for k in range(warmup):
            sets[k % nsets]()
        barrier()
        # (1) back to back over the rotating sets: the headline per-step time.  At
        # N = 1 the steps' API calls are captured once per rotation into a CUDA
        # graph and replayed (the same kernels with the same arguments: outputs
        # bit-identical, tools/graph_probe.py); the eager loop is timed beside it.
        # N > 1 stays eager (the link protocols number their calls on the host).
        graph = None
        if world == 1 and not args.no_graph:
            try:
                cs = torch.cuda.Stream(device=dev)
                cs.wait_stream(torch.cuda.current_stream())
                torch.cuda.synchronize()
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph, stream=cs):
                    for k in range(nsets):
                        sets[k]()
                torch.cuda.synchronize()
                graph.replay()
                torch.cuda.synchronize()
            except Exception as exc:   # noqa: BLE001
                print(f"bench: graph capture unavailable ({exc}); eager only", file=sys.stderr)
                graph = None

        def timed_loop(use_graph):
            barrier()
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record(stream)
            if use_graph:
                for _ in range(steps // nsets):
                    graph.replay()
                for k in range(steps % nsets):
                    sets[k]()
            else:
                for k in range(steps):
                    sets[k % nsets]()
            t1.record(stream)
            barrier()
            return max_over_ranks(t0.elapsed_time(t1) / steps)

        sampler = ClockSampler(local)
        with sampler:
            eager_ms = timed_loop(False)
            ms = timed_loop(True) if graph is not None else eager_ms
        # (2) each step alone after a 2x-L2 write flush, events around it
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        barrier()
        for k in range(steps):
            flush_l2()
            ev[k][0].record(stream)
            sets[0]()
            ev[k][1].record(stream)
        barrier()
        t = np.array([a.elapsed_time(b) for a, b in ev])
        per = {"median_ms": max_over_ranks(float(np.median(t))), "p10_ms": max_over_ranks(float(np.percentile(t, 10))),
               "p90_ms": max_over_ranks(float(np.percentile(t, 90))), "mean_ms": max_over_ranks(float(t.mean()))}
        stats = occ.occ_read_stats(sets[0].ws)
        return {"ms": ms, "eager_ms": eager_ms, "graph": graph is not None, "per_step": per,
                "clocks": sampler.summary(), "stats": stats, "sets": sets, "nsets": nsets}

    def count_launches(step):
        """Kernels of OURS launched by one step (torch profiler, untimed)."""
        try:
            from torch.profiler import ProfilerActivity, profile
            barrier()
            with profile(activities=[ProfilerActivity.CUDA]) as prof:
                step()
                torch.cuda.synchronize()
            names = [e.name for e in prof.events() if e.device_type.name == "CUDA"]
            ours = [x for x in names if "occ" in x]
            return len(ours), sorted(set(ours))
        except Exception as exc:   # noqa: BLE001
            return None, [f"profiler unavailable: {exc}"[:120]]

    name = args.config
    cfg = CONFIGS[name]
    res = bench_config(name, args.steps, args.warmup)
    ms = res["ms"]
    value = world * elems(cfg) * 4 / (ms * 1e-3) / 1e9   # GB/s of uncompressed fp32 tensor, whole job
    ab = alg_bytes(cfg, world)
    achieved = ab / (ms * 1e-3) / 1e9
    launches, kernel_names = count_launches(res["sets"][0])
    kind = cfg["kind"]
    parallelism = "1gpu" if world == 1 else (f"dp{world}" if kind == "dp" else f"pp-ring{world}" + ("-link" if use_link else "-nccl"))

    # ---------------------------------------------------------------- e2e
    e2e = None
    if not args.no_e2e:
        step = res["sets"][0]
        b = step.mats[0]
        n, m = cfg["shapes"][0]
        Mh = b["M"].cpu().pin_memory()
        Rh = torch.empty(n, m, dtype=torch.float32).pin_memory()
        nbuf = 2
        Mb = [torch.empty_like(b["M"]) for _ in range(nbuf)]
        Rb = [torch.empty_like(b["R"]) for _ in range(nbuf)]
        h2d_s, d2h_s = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
        e2e_steps = max(3, min(args.steps, 20))

        def e2e_run(k_steps):
            # H2D of M and D2H of the step's M' on their own streams, M / M' double
            # buffered on the device so step k's D2H overlaps step k+1's H2D
            ev = [[torch.cuda.Event() for _ in range(3)] for _ in range(k_steps)]   # H2D, step, D2H done
            h2d_s.wait_stream(stream)
            for k in range(k_steps):
                j = k % nbuf
                if k >= nbuf:
                    h2d_s.wait_event(ev[k - nbuf][2] if kind == "dp" else ev[k - nbuf][1])
                with torch.cuda.stream(h2d_s):
                    Mb[j].copy_(Mh, non_blocking=True)
                ev[k][0].record(h2d_s)
                stream.wait_event(ev[k][0])
                if k >= nbuf:
                    stream.wait_event(ev[k - nbuf][2])
                out = step(Mb[j], Rb[j])
                ev[k][1].record(stream)
                d2h_s.wait_event(ev[k][1])
                with torch.cuda.stream(d2h_s):
                    Rh.copy_(out, non_blocking=True)
                ev[k][2].record(d2h_s)
            stream.wait_stream(d2h_s)
            stream.wait_stream(h2d_s)

        e2e_run(2)
        barrier()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        e2e_run(e2e_steps)
        t1.record(stream)
        barrier()
        e_ms = max_over_ranks(t0.elapsed_time(t1) / e2e_steps)
        e2e = {"value": world * elems(cfg) * 4 / (e_ms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": e_ms,
               "h2d_bytes_per_step": n * m * 4, "d2h_bytes_per_step": n * m * 4,
               "note": "first matrix of the config through H2D/D2H; the step itself is the full config"}

    # ---------------------------------------------------------------- factor comm + NVLink (N > 1)
    comm_line = None
    if world > 1:
        r = cfg["r"]
        fbytes = sum((n + m) * r * 4 for n, m in cfg["shapes"])   # P_hat + Q per matrix, fp32
        reps = 50
        if kind == "dp":
            pb = torch.zeros(sum(n for n, _ in cfg["shapes"]) * r, device=dev)
            qb = torch.zeros(sum(m for _, m in cfg["shapes"]) * r, device=dev)

            def xchg():   # the two factor sums of occ_allreduce_factors(_link), on its bucket sizes
                if dplink is not None:
                    dplink.allreduce(pb, pb)
                    dplink.allreduce(qb, qb)
                else:
                    dist.all_reduce(pb)
                    dist.all_reduce(qb)
        else:
            b = res["sets"][0].mats[0]
            lk = res["sets"][0].link

            def xchg_nccl():   # the library's NCCL exchange: occ_sendrecv_factors with M = NULL, out = NULL
                occ.occ_sendrecv_factors(None, None, b["Q"], b["P"], r, snd_peer, None, b["Pr"], b["Qr"], rcv_peer,
                                         comm)

            def xchg_link():   # the in-kernel NVLink exchange alone: occ_sendrecv_factors_link, M = NULL, out = NULL
                occ.occ_sendrecv_factors_link(None, None, b["Q"], b["P"], r, None, b["Pr"], b["Qr"], lk)
            xchg = xchg_link if lk is not None else xchg_nccl
            nccl_reps = 20
            for _ in range(3):
                xchg_nccl()
            barrier()
            n0, n1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            n0.record(stream)
            for _ in range(nccl_reps):
                xchg_nccl()
            n1.record(stream)
            barrier()
            nccl_us = max_over_ranks(n0.elapsed_time(n1) / nccl_reps * 1e3)
        for _ in range(5):
            xchg()
        barrier()
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record(stream)
        for _ in range(reps):
            xchg()
        c1.record(stream)
        barrier()
        comm_us = max_over_ranks(c0.elapsed_time(c1) / reps * 1e3)
        # NVLink bandwidth in the same run: 1 GiB all-reduce (bus bandwidth) and 1 GiB ring send/recv
        big = torch.ones(256 * 1024 * 1024, device=dev)
        big2 = torch.empty_like(big)
        nb = big.numel() * 4

        def ring():
            ops = [dist.P2POp(dist.isend, big, snd_peer), dist.P2POp(dist.irecv, big2, rcv_peer)]
            for q in dist.batch_isend_irecv(ops):
                q.wait()
        bw = {}
        for nm, fn in (("allreduce", lambda: dist.all_reduce(big)), ("sendrecv", ring)):
            fn()
            barrier()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            for _ in range(5):
                fn()
            a1.record(stream)
            barrier()
            t = max_over_ranks(a0.elapsed_time(a1) / 5 * 1e-3)
            bw[nm] = (2 * (world - 1) / world * nb / t / 1e9) if nm == "allreduce" else nb / t / 1e9
        del big, big2
        if kind == "dp":   # ring model 2V(R-1)/R per allreduce, both allreduces
            model_us = 2 * fbytes * (world - 1) / world / (bw["allreduce"] * 1e9) * 1e6
        else:              # one P2P message of V bytes per link
            model_us = fbytes / (bw["sendrecv"] * 1e9) * 1e6
        # the same step without the exchange (compress, then decompress the own
        # factors locally): ring step - this = the exchange's cost inside the step
        local_us = None
        if kind != "dp":
            sets = res["sets"]

            def local_step(k):
                b = sets[k % len(sets)].mats[0]
                occ.occ_compress(b["M"], b["E"], b["Q"], b["P"], None, r=r, ws=sets[k % len(sets)].ws)
                occ.occ_decompress(b["P"], b["Q"], b["R"])
            for k in range(3):
                local_step(k)
            barrier()
            l0, l1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            l0.record(stream)
            for k in range(args.steps):
                local_step(k)
            l1.record(stream)
            barrier()
            local_us = max_over_ranks(l0.elapsed_time(l1) / args.steps * 1e3)
        comm_line = {"factor_comm_us": comm_us,
                     "exchange": ("dp-link" if dplink is not None else "dp-nccl") if kind == "dp" else args.exchange,
                     "step_without_exchange_us": local_us,
                     "exchange_cost_in_step_us": None if local_us is None else ms * 1e3 - local_us,
                     "nccl_sendrecv_us": None if kind == "dp" else nccl_us,
                     "factor_bytes": fbytes, "nvlink_busbw_allreduce_GBs": bw["allreduce"],
                     "nvlink_sendrecv_GBs": bw["sendrecv"], "model_us": model_us, "frac_of_nvlink_roofline": model_us / comm_us,
                     "how": "DP: the two factor sums of the step on its bucket sizes (occ_dplink_allreduce in-kernel over "
                            "NVLink peer memory with --exchange link, else ncclAllReduce); PP: the "
                            "library's exchange of (P_hat, Q) alone -- occ_sendrecv_factors_link(M=NULL, out=NULL) "
                            "(in-kernel NVLink stores + flag, --exchange link) or occ_sendrecv_factors(M=NULL, "
                            "out=NULL) (grouped NCCL send/recv, also reported as nccl_sendrecv_us); model = "
                            "PAPER.md:607 ring cost (DP) or V / measured P2P bandwidth (PP)"}

    # ---------------------------------------------------------------- north-star T beside C2
    target = None
    if name == "C2" and world == 1 and not args.no_target:
        t = bench_config("T", args.steps, args.warmup)
        tab = alg_bytes(CONFIGS["T"], 1)
        target = {"workload": CONFIGS["T"]["desc"], "ms_per_step": t["ms"], "eager_ms_per_step": t["eager_ms"],
                  "per_step_flushed": t["per_step"],
                  "value": 1024 * 3072 * 4 / (t["ms"] * 1e-3) / 1e9, "unit": "GB/s",
                  "roofline_frac": tab / (t["ms"] * 1e-3) / 1e9 / hbm_peak,
                  "roofline_frac_flushed_median": tab / (t["per_step"]["median_ms"] * 1e-3) / 1e9 / hbm_peak}
        del t

    # ---------------------------------------------------------------- oracle on the host
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from threadpoolctl import threadpool_limits
        dt, done = run_oracle(cfg, 1000, 12.0)
        cores = cpu_threads()
        with threadpool_limits(limits=1):
            dt1, done1 = run_oracle(cfg, 1000, 6.0)
        cpu = {"value": elems(cfg) * 4 / dt / 1e9, "unit": "GB/s", "cores": cores, "kind": "oracle",
               "sample": f"{done} oracle steps (NumPy fp64, ~12 s budget) of the same {name} workload",
               "one_thread": {"value": elems(cfg) * 4 / dt1 / 1e9, "unit": "GB/s", "cores": 1,
                              "sample": f"{done1} oracle steps, BLAS limited to 1 thread, ~6 s budget"}}

    traffic = None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(name if world == 1 else f"{name}_{parallelism}")
        except Exception:
            traffic = None

    if rank == 0:
        kern = {"1gpu": "occ_v2_kernel (fused step)" if res["stats"]["path"] == 3 else "per-phase kernels",
                "pp": "sender compress + receiver decompress kernels" + ("" if world == 1 else (" + in-kernel NVLink exchange" if use_link else " + NCCL send/recv")),
                "dp": "DP step kernels + 2 factor sums" + (" (in-kernel NVLink, occ_dplink)" if dplink is not None else " (NCCL allreduce)")}[kind]
        cd = config_dict(name, world, parallelism)
        cd["l2"] = (f"inputs larger than L2: {res['nsets']} rotating input sets of {elems(cfg) * 12 / 1e6:.0f} MB "
                    f"(M, e, M') back to back; per_step: each step alone after a 2x-L2 write flush")
        cd["timing"] = ("back to back: one rotation of the steps' API calls captured in a CUDA graph and replayed "
                        "(eager_ms_per_step: the same loop issued eagerly)" if res["graph"] else
                        "back to back, eager")
        cd["path"] = {1: "v1 fused persistent kernel", 2: "per-phase launches",
                      3: "fused TMEM-resident persistent kernel"}.get(res["stats"]["path"], "per-phase launches")
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "eager_ms_per_step": res["eager_ms"],
            "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded, DESIGN.md §4 D2 gradient-like)",
            "config": cd,
            "per_step_flushed": res["per_step"],
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "traffic": traffic, "peak_kind": peak_kind,
                         "alg_bytes_per_step": ab, "kernel": kern,
                         "frac_flushed_median": ab / (res["per_step"]["median_ms"] * 1e-3) / 1e9 / hbm_peak},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches * args.steps if launches is not None else None,
            "launches_per_step": launches, "kernels": kernel_names,
            "clocks": res["clocks"],
            "factor_comm": comm_line,
            "orth": {"second_pass": res["stats"]["second_pass"], "kappa_est": res["stats"]["kappa_est"],
                     "fallback_columns": res["stats"]["fallback_columns"]},
        }
        if target:
            line["north_star_target"] = target
        print(json.dumps(line), flush=True)
    barrier()
    for lk in links:
        lk.close()
    if dplink is not None:
        dplink.close()
    if comm is not None:
        comm.destroy()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
