"""How the measurement method changes the per-step time of occ_compress:
(a) flushed, events per step, CPU enqueues as it goes (round-1 bench);
(b) flushed, events per step, a GPU sleep ahead so the CPU never gates the GPU;
(c) back to back, warm L2 (same buffers every step);
(d) back to back, K rotating buffer sets larger than L2 (cold inputs every step).
Usage: python tools/timing_modes.py [n x m x r ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2301_09830_b200 import occ  # noqa: E402
from workloads import synth  # noqa: E402


def main(n, m, r, steps=200):
    dev = torch.device("cuda")
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    per_set = n * m * 4 * 4
    nsets = max(2, int(np.ceil(3 * l2 / per_set)))
    M0 = torch.from_numpy(synth.d2_gradlike(n, m, 5)).to(dev)
    E0 = torch.from_numpy(synth.e0(n, m, 6, like=M0.cpu().numpy())).to(dev)
    Q0 = torch.from_numpy(synth.q0(m, r, 7)).to(dev)
    sets = [(M0.clone(), E0.clone(), Q0.clone(), torch.empty(n, r, device=dev), torch.empty_like(M0))
            for _ in range(nsets)]
    ws = occ.alloc_workspace(n, m, r)
    flush = torch.empty(2 * l2 // 4, device=dev).uniform_()
    sink = torch.empty(1, device=dev)
    st = torch.cuda.current_stream()
    out = {"shape": [n, m, r], "nsets": nsets}

    def call(k):
        Md, Ed, Qd, Pd, Rd = sets[k % nsets]
        occ.occ_compress(Md, Ed, Qd, Pd, Rd, r=r, ws=ws)

    for mode in ("a", "b"):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for _ in range(5):
            torch.sum(flush, dim=0, out=sink[0]); call(0)
        torch.cuda.synchronize()
        if mode == "b":
            torch.cuda._sleep(int(2e9 * steps * 80e-6))   # ~steps x 80 us of GPU time ahead of the CPU
        for i in range(steps):
            torch.sum(flush, dim=0, out=sink[0])
            ev[i][0].record(st)
            call(0)
            ev[i][1].record(st)
        torch.cuda.synchronize()
        t = np.array([a.elapsed_time(b) * 1e3 for a, b in ev])
        out[mode] = {"median_us": float(np.median(t)), "p10": float(np.percentile(t, 10)), "p90": float(np.percentile(t, 90))}
    for mode, rot in (("c", False), ("d", True)):
        for i in range(10):
            call(i if rot else 0)
        torch.cuda.synchronize()
        torch.cuda._sleep(int(2e9 * steps * 80e-6))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for i in range(steps):
            call(i if rot else 0)
        b.record(st)
        torch.cuda.synchronize()
        out[mode] = {"mean_us": a.elapsed_time(b) * 1e3 / steps}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    for spec in sys.argv[1:] or ["1024x3072x16", "4096x1920x16"]:
        main(*map(int, spec.split("x")))
