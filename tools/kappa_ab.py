"""Per-step accuracy of the per-phase path (r = 64) on a warm-started D3 stream
against the oracle, under the CholQR2 threshold given by OCC_KAPPA_PHASE
(run once per setting: the library reads it once).  Usage:
  OCC_KAPPA_PHASE=1e4 python tools/kappa_ab.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2301_09830_b200 import occ  # noqa: E402
from workloads import synth  # noqa: E402


def main():
    n, m, r, T = 2048, 1536, 64, int(os.environ.get("STEPS", "6"))
    Ms = synth.d3_lep_stream(n, m, 83, T)
    Q0 = synth.q0(m, r, 84)
    Md = torch.empty(n, m, device="cuda")
    Ed = torch.zeros(n, m, device="cuda")
    Qd = torch.from_numpy(Q0).cuda()
    Pd = torch.empty(n, r, device="cuda")
    Rd = torch.empty(n, m, device="cuda")
    ws = occ.alloc_workspace(n, m, r)
    e_o = np.zeros((n, m))
    Q_o = Q0.astype(np.float64)
    for t, Mt in enumerate(Ms):
        Md.copy_(torch.from_numpy(Mt).cuda())
        occ.occ_compress(Md, Ed, Qd, Pd, Rd, r=r, ws=ws)
        torch.cuda.synchronize()
        st = occ.occ_read_stats(ws)
        A = Mt.astype(np.float64) + e_o
        o = oracle.compress_step(Mt, e_o, Q_o)
        rg, eg, ph = Rd.double().cpu().numpy(), Ed.double().cpu().numpy(), Pd.double().cpu().numpy()
        print(json.dumps({"kappa_phase": os.environ.get("OCC_KAPPA_PHASE"), "step": t, "kappa_est": st["kappa_est"],
                          "second_pass": st["second_pass"],
                          "recon_elem": float(np.abs(rg - o["recon"]).max() / np.abs(A).max()),
                          "recon_rel": float(np.linalg.norm(rg - o["recon"]) / np.linalg.norm(A)),
                          "err_elem": float(np.abs(eg - o["err"]).max() / np.abs(A).max()),
                          "orth": float(np.linalg.norm(ph.T @ ph - np.eye(r)))}), flush=True)
        e_o, Q_o = o["err"], o["Q"]


if __name__ == "__main__":
    main()
