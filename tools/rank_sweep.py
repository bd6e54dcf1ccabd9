"""Throughput versus rank ("the
throughput decreases as the rank increases" because orthogonalisation
dominates).  occ_compress with M' on T (1024 x 3072) and configs[1]
(4096 x 1920) at r = 4 .. 64, back to back over rotating input sets larger
than L2 (as bench.py), plus the per-sample matricisation alternative of
reading C6: configs[1] as 4 separate 1024 x 1920 micro-batch matrices (each
with its own error and warm start) instead of one 4096 x 1920.
One JSON line per point.  python tools/rank_sweep.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2301_09830_b200 import occ  # noqa: E402
from workloads import synth  # noqa: E402

PEAK = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"]


def time_sets(calls, steps=60):
    for c in calls[:4]:
        c()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for k in range(steps):
        calls[k % len(calls)]()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps * 1e3   # us


def sets_for(mats, r, nsets):
    """mats: list of (n, m) matrices compressed per step; returns nsets closures."""
    out = []
    for s in range(nsets):
        bufs = []
        for i, (n, m) in enumerate(mats):
            M = torch.from_numpy(synth.d2_gradlike(n, m, 500 + 10 * s + i)).cuda()
            bufs.append((M, torch.zeros_like(M), torch.from_numpy(synth.q0(m, r, 7)).cuda(),
                         torch.empty(n, r, device="cuda"), torch.empty_like(M), occ.alloc_workspace(n, m, r)))

        def call(bufs=bufs):
            for M, E, Q, P, R, ws in bufs:
                occ.occ_compress(M, E, Q, P, R, r=r, ws=ws)
        call.ws = bufs[0][5]
        out.append(call)
    return out


def main():
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    for name, mats in (("T 1024x3072", [(1024, 3072)]), ("configs[1] 4096x1920", [(4096, 1920)]),
                       ("configs[1] per-sample 4 x 1024x1920", [(1024, 1920)] * 4)):
        el = sum(n * m for n, m in mats)
        nsets = max(2, int(np.ceil(3 * l2 / (el * 12))))
        for r in (4, 8, 16, 32, 64):
            sets = sets_for(mats, r, nsets)
            us = time_sets(sets)
            alg = sum(n * m * 16 + r * (n + 2 * m) * 4 for n, m in mats)
            st = occ.occ_read_stats(sets[0].ws)
            print(json.dumps({"workload": name, "rank": r, "us_per_step": us, "GB_s": el * 4 / us / 1e3,
                              "roofline_frac": alg / us / 1e3 / PEAK, "path": st["path"],
                              "compression_ratio": sum(n * m for n, m in mats) / sum(r * (n + m) for n, m in mats)}),
                  flush=True)
            del sets
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
