"""The tcgen05 DP path (occ_umma.cu: sweeps + reconstruction) against the
mma.sync path on the same inputs (1-rank occ_allreduce_factors, no
communicator): relative differences of G (= M'), err, Q, P (fp32 rounding
level expected) and the time of both (CUDA events, back to back).
Usage: python tools/umma_dp_check.py [n x m x r ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2301_09830_b200 import occ  # noqa: E402
from workloads import synth  # noqa: E402


def run(shapes, r, flags, reps=10):
    mats = []
    for j, (n, m) in enumerate(shapes):
        M = torch.from_numpy(synth.d2_gradlike(n, m, 5 + j)).cuda()
        E0 = torch.from_numpy(synth.e0(n, m, 6 + j, like=M.cpu().numpy())).cuda()
        qrows = n if flags & occ.OCC_ORIENT_T else m
        prows = m if flags & occ.OCC_ORIENT_T else n
        Q0 = torch.from_numpy(synth.q0(qrows, r, 7 + j)).cuda()
        mats.append((M, E0, Q0, prows))
    res = {}
    for mode in ("0", "1"):
        os.environ["OCC_UMMA"] = mode
        G = [x[0].clone() for x in mats]
        E = [x[1].clone() for x in mats]
        Q = [x[2].clone() for x in mats]
        P = [torch.empty(x[3], r, device="cuda") for x in mats]
        ws = occ.occ_allreduce_factors(G, E, Q, P, r, 1.0, flags)
        torch.cuda.synchronize()
        res[mode] = (G, E, Q, P)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        for _ in range(2):
            occ.occ_allreduce_factors(G, E, Q, P, r, 1.0, flags, ws=ws)
        ev[0].record()
        for _ in range(reps):
            occ.occ_allreduce_factors(G, E, Q, P, r, 1.0, flags, ws=ws)
        ev[1].record()
        torch.cuda.synchronize()
        res[mode + "_us"] = ev[0].elapsed_time(ev[1]) * 1e3 / reps
    d = {}
    for i, name in enumerate(("G", "err", "Q", "P")):
        worst = 0.0
        for a, b in zip(res["0"][i], res["1"][i]):
            worst = max(worst, float((a - b).norm() / max(float(a.norm()), 1e-30)))
            d[name + "_finite"] = bool(torch.isfinite(b).all())
        d[name] = worst
    return {"shapes": shapes, "r": r, "flags": flags, "rel_diff": d, "us_mma_sync": res["0_us"], "us_umma": res["1_us"]}


def main():
    cases = [([(3072, 12288), (3072, 9216)], 64, 0), ([(1000, 776)], 64, 0), ([(1000, 776)], 32, occ.OCC_EF_GLOBAL),
             ([(333, 520)], 64, occ.OCC_ORIENT_T), ([(8192, 3072)], 64, occ.OCC_ORIENT_T)]
    for shapes, r, flags in cases:
        print(json.dumps(run(shapes, r, flags)), flush=True)


if __name__ == "__main__":
    main()
