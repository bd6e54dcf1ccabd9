"""Accuracy of the per-phase path against the fp64 oracle (element-wise and
Frobenius, as tests/test_gpu_parity.py measures them) under environment
settings given as KEY=VALUE arguments, one setting per run; e.g.
  python tools/umma_acc.py OCC_UMMA=0 OCC_UMMA=1 OCC_UMMA_KMAX=256"""
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
    n, m, r = (int(x) for x in os.environ.get("SHAPE", "8192x3072x32").split("x"))
    M = synth.d2_gradlike(n, m, 1000 + n)
    e = synth.e0(n, m, 1001 + n, like=M)
    Q0 = synth.q0(m, r, 1002)
    o = oracle.compress_step(M, e, Q0)
    A = M.astype(np.float64) + e
    amax = np.abs(A).max()
    nA = np.linalg.norm(A)
    for setting in sys.argv[1:] or ["OCC_UMMA=1"]:
        k, v = setting.split("=")
        old = os.environ.get(k)
        os.environ[k] = v
        Md, Ed, Qd = (torch.from_numpy(x).cuda() for x in (M, e.copy(), Q0.copy()))
        Pd = torch.empty(n, r, device="cuda")
        Rd = torch.empty_like(Md)
        occ.occ_compress(Md, Ed, Qd, Pd, Rd, r=r)
        torch.cuda.synchronize()
        rec = Rd.double().cpu().numpy()
        err = Ed.double().cpu().numpy()
        res = {"setting": setting, "shape": [n, m, r],
               "recon_elem": float(np.abs(rec - o["recon"]).max() / amax),
               "recon_rel": float(np.linalg.norm(rec - o["recon"]) / nA),
               "err_elem": float(np.abs(err - o["err"]).max() / amax),
               "Q_rel": float(np.linalg.norm(Qd.double().cpu().numpy() - o["Q"]) / np.linalg.norm(o["Q"])),
               "P_hat_rel": float(np.linalg.norm(Pd.double().cpu().numpy() - o["P_hat"]) / np.linalg.norm(o["P_hat"]))}
        print(json.dumps(res), flush=True)
        if old is None:
            del os.environ[k]
        else:
            os.environ[k] = old


if __name__ == "__main__":
    main()
