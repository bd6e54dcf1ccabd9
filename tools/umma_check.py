"""The tcgen05 sweep (occ_umma.cu) against the mma.sync sweep on the same inputs:
relative differences of P_hat, Q, M', e_new (fp32 rounding level expected),
and the step time of both (CUDA events, back to back).
Usage: python tools/umma_check.py [n x m x r ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2301_09830_b200 import occ  # noqa: E402
from workloads import synth  # noqa: E402


def run(n, m, r, flags, reps=20):
    M = torch.from_numpy(synth.d2_gradlike(n, m, 5)).cuda()
    E0 = torch.from_numpy(synth.e0(n, m, 6, like=M.cpu().numpy())).cuda()
    Q0 = torch.from_numpy(synth.q0(m, r, 7)).cuda()
    ws = occ.alloc_workspace(n, m, r)
    res = {}
    for mode in ("0", "1"):
        os.environ["OCC_UMMA"] = mode
        E = E0.clone(); Q = Q0.clone()
        P = torch.empty(n, r, device="cuda"); out = torch.empty_like(M)
        occ.occ_compress(M, E, Q, P, out, r=r, flags=flags, ws=ws)
        torch.cuda.synchronize()
        res[mode] = (P.clone(), Q.clone(), out.clone(), E.clone())
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        Et = E0.clone(); Qt = Q0.clone()
        for _ in range(3):
            occ.occ_compress(M, Et, Qt, P, out, r=r, flags=flags, ws=ws)
        ev[0].record()
        for _ in range(reps):
            occ.occ_compress(M, Et, Qt, P, out, r=r, flags=flags, ws=ws)
        ev[1].record()
        torch.cuda.synchronize()
        res[mode + "_us"] = ev[0].elapsed_time(ev[1]) * 1e3 / reps
    d = {}
    for i, name in enumerate(("P", "Q", "recon", "err")):
        a, b = res["0"][i], res["1"][i]
        d[name] = float((a - b).norm() / max(float(a.norm()), 1e-30))
        d[name + "_finite"] = bool(torch.isfinite(b).all())
    return {"shape": [n, m, r], "flags": flags, "rel_diff": d, "us_mma_sync": res["0_us"], "us_umma": res["1_us"]}


def main():
    shapes = [tuple(int(x) for x in a.split("x")) for a in sys.argv[1:]] or \
        [(8192, 3072, 32), (3072, 12288, 64), (3072, 9216, 64), (1000, 776, 32), (333, 520, 64), (4096, 1920, 16)]
    for n, m, r in shapes:
        flags = occ.OCC_FORCE_MULTI if r == 16 or n * m < 2_000_000 else 0
        print(json.dumps(run(n, m, r, flags)), flush=True)


if __name__ == "__main__":
    main()
