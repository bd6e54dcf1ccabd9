"""The fused step (occ_compress) issued eagerly back to back vs replayed from a
CUDA graph captured over the same rotation of input sets: microseconds per
step and whether the outputs are bit-identical.  Usage: python tools/graph_probe.py [T|C2]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2301_09830_b200 import occ  # noqa: E402
from workloads import synth  # noqa: E402

SHAPES = {"T": (1024, 3072, 16), "C2": (4096, 1920, 16)}


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "T"
    n, m, r = SHAPES[name]
    nsets, reps = 8, 50
    sets = []
    for k in range(nsets):
        M = torch.from_numpy(synth.d2_gradlike(n, m, 10 + k)).cuda()
        E0 = torch.from_numpy(synth.e0(n, m, 20 + k, like=M.cpu().numpy())).cuda()
        Q0 = torch.from_numpy(synth.q0(m, r, 30 + k)).cuda()
        sets.append({"M": M, "E0": E0, "Q0": Q0, "E": E0.clone(), "Q": Q0.clone(),
                     "P": torch.empty(n, r, device="cuda"), "R": torch.empty_like(M),
                     "ws": occ.alloc_workspace(n, m, r)})

    def reset():
        for s in sets:
            s["E"].copy_(s["E0"])
            s["Q"].copy_(s["Q0"])

    def round_():
        for s in sets:
            occ.occ_compress(s["M"], s["E"], s["Q"], s["P"], s["R"], r=r, ws=s["ws"])

    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    # eager
    reset()
    round_()
    torch.cuda.synchronize()
    ref = [s["R"].clone() for s in sets]
    reset()
    for _ in range(2):
        round_()
    ev[0].record()
    for _ in range(reps):
        round_()
    ev[1].record()
    torch.cuda.synchronize()
    eager_us = ev[0].elapsed_time(ev[1]) * 1e3 / (reps * nsets)
    # graph: one round captured, replayed
    reset()
    s0 = torch.cuda.Stream()
    s0.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s0):
        round_()   # warm-up (plan cache, attributes) outside the capture
    torch.cuda.current_stream().wait_stream(s0)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        round_()
    reset()
    g.replay()
    torch.cuda.synchronize()
    same = all(torch.equal(a, s["R"]) for a, s in zip(ref, sets))
    for _ in range(2):
        g.replay()
    ev[0].record()
    for _ in range(reps):
        g.replay()
    ev[1].record()
    torch.cuda.synchronize()
    graph_us = ev[0].elapsed_time(ev[1]) * 1e3 / (reps * nsets)
    print(json.dumps({"config": name, "eager_us_per_step": eager_us, "graph_us_per_step": graph_us,
                      "outputs_bit_identical": same}), flush=True)


if __name__ == "__main__":
    main()
