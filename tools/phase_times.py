"""Per-phase device time of the fused step kernel (from %globaltimer stamps)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_09830_b200 import occ
from workloads import synth

NAMES = {0: "A sweep1", 1: "B reduce+gram", 3: "C orth", 6: "D sweep2", 7: "E Qreduce", 8: "F recon"}
NAMES2 = {0: "1 sweep1+tmem", 1: "2 Pband+gram", 2: "3a chol", 3: "3b Qpart", 4: "4 Qreduce", 5: "5 recon"}


def run(n, m, r, reps=20, bf16=False):
    M = torch.from_numpy(synth.d2_gradlike(n, m, 5)).cuda()
    if bf16:
        M = M.bfloat16()
    E = torch.from_numpy(synth.e0(n, m, 6, like=synth.d2_gradlike(8, 8, 1))).cuda() * 0
    Q = torch.from_numpy(synth.q0(m, r, 7)).cuda()
    P = torch.empty(n, r, device="cuda")
    R = torch.empty_like(M)
    ws = occ.alloc_workspace(n, m, r)
    flush = torch.ones(64 * 1024 * 1024, device="cuda")
    sink = torch.empty(1, device="cuda")
    acc = {}
    for i in range(reps):
        torch.sum(flush, dim=0, out=sink[0])   # clean read flush: no dirty lines left in L2
        occ.occ_compress(M, E, Q, P, R, r=r, ws=ws)
        torch.cuda.synchronize()
        st = occ.occ_read_stats(ws)
        t = st["t_ns"]
        if i < 3:
            continue
        names, end = (NAMES2, 6) if st["path"] == 3 else (NAMES, 9)
        marks = [k for k in sorted(names) if t[k]] + [end]
        for a, b in zip(marks, marks[1:]):
            acc.setdefault(names[a], []).append((t[b] - t[a]) / 1e3)
        acc.setdefault("total", []).append((t[end] - t[0]) / 1e3)
        if st["path"] == 3:
            acc.setdefault("1.prologue", []).append((t[7] - t[0]) / 1e3)
            acc.setdefault("1.wait_sum", []).append(t[8] / 1e3)
            acc.setdefault("3.reduceG", []).append((t[9] - t[2]) / 1e3)
            acc.setdefault("3.chol", []).append((t[10] - t[9]) / 1e3)
            acc.setdefault("3.inverse", []).append((t[11] - t[10]) / 1e3)
            acc.setdefault("3.apply", []).append((t[3] - t[11]) / 1e3)
    out = {k: sorted(v)[len(v) // 2] for k, v in acc.items()}
    print(json.dumps({"shape": [n, m, r], "bf16": bf16, "path": st["path"], "us": out, "grid": st["grid"]}))


if __name__ == "__main__":
    for spec in sys.argv[1:] or ["4096x1920x16", "1024x3072x16"]:
        n, m, r = map(int, spec.split("x"))
        run(n, m, r)
