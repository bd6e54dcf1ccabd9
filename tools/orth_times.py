"""Phase stamps of the per-phase path's cooperative kernel (P reduce + Gram,
orthonormalisation, sweep 2, Q reduce), from the instrumented build
(libocc_trace.so: CTA 0's %globaltimer at the boundaries, OCC_STAMP inside the
orthonormalisation).  Usage: OCC_LIB=trace python tools/orth_times.py [n x m x r ...]"""
import json
import os
import sys

os.environ.setdefault("OCC_LIB", "trace")
os.environ.setdefault("OCC_UMMA", "0")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2301_09830_b200 import build as occ_build, occ  # noqa: E402
from workloads import synth  # noqa: E402

# OCC_FAST_ORTH=0 (phases B, C1..C3 in every CTA) and the default one-CTA
# factorisation (orth_fast) stamp different slots; run with OCC_UMMA=0 so that
# the whole step is one cooperative launch (the stamps share its start)
NAMES_SLOW = {3: "P reduce + Gram partials (B)", 1: "C1 Gram reduce", 2: "C1 Cholesky", 4: "C1 L^-1",
              5: "C1 P_hat (+ 2nd Gram partials)", 9: "C3 Gram reduce (after barrier)", 10: "C3 Cholesky",
              11: "C3 L^-1", 6: "C3 P_hat + barrier", 7: "sweep 2 (D)", 8: "Q reduce (E)"}
NAMES_FAST = {1: "sweep 1 (A)", 9: "P reduce + Gram partials + reduce + barriers", 2: "factor: Gram load",
              3: "factor: LDL + inverse sweep", 4: "factor: Li, kappa", 10: "barrier",
              11: "apply P_hat", 6: "barrier", 7: "sweep 2 (D)", 8: "Q reduce (E)"}
FAST = os.environ.get("OCC_FAST_ORTH", "1") != "0"
NAMES = NAMES_FAST if FAST else NAMES_SLOW
ORDER = (1, 9, 2, 3, 4, 10, 11, 6, 7, 8) if FAST else (3, 1, 2, 4, 5, 9, 10, 11, 6, 7, 8)


def main():
    occ_build.build(trace=True)
    shapes = [tuple(int(x) for x in a.split("x")) for a in sys.argv[1:]] or [(3072, 12288, 64), (8192, 3072, 32)]
    for n, m, r in shapes:
        M = torch.from_numpy(synth.d2_gradlike(n, m, 5)).cuda()
        E = torch.from_numpy(synth.e0(n, m, 6, like=M.cpu().numpy())).cuda()
        Q = torch.from_numpy(synth.q0(m, r, 7)).cuda()
        P = torch.empty(n, r, device="cuda")
        out = torch.empty_like(M)
        ws = occ.alloc_workspace(n, m, r)
        for it in range(4):
            occ.occ_compress(M, E, Q, P, out, r=r, ws=ws)
            st = occ.occ_read_stats(ws)
            t = st["t_ns"]
            order = [k for k in ORDER if t[k] >= t[0] and t[k] - t[0] < 10**8]
            prev, res = t[0], {}
            for k in order:
                res[NAMES[k]] = round((t[k] - prev) / 1e3, 1)
                prev = t[k]
            print(json.dumps({"shape": [n, m, r], "iter": it, "second_pass": st["second_pass"],
                              "kappa": round(st["kappa_est"], 1), "us": res}), flush=True)


if __name__ == "__main__":
    main()
