"""Debug driver: one occ_compress call on a small matrix, prints stats and parity."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2301_09830_b200 import occ
import oracle
from workloads import synth
n, m, r = (int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "128x256x4").split("x"))
M = synth.d2_gradlike(n, m, 3); e = synth.e0(n, m, 4, like=M); Q0 = synth.q0(m, r, 5)
Md, Ed, Qd = (torch.from_numpy(x).cuda() for x in (M, e, Q0))
Pd = torch.empty(n, r, device="cuda"); Rd = torch.empty_like(Md)
t = time.time()
ws = occ.occ_compress(Md, Ed, Qd, Pd, Rd, r=r)
torch.cuda.synchronize()
st = occ.occ_read_stats(ws)
o = oracle.compress_step(M, e, Q0)
A = M.astype(np.float64) + e
err = np.linalg.norm(Rd.double().cpu().numpy() - o["recon"]) / np.linalg.norm(A)
print(json.dumps({"shape": [n, m, r], "path": st["path"], "recon_rel": err, "sec": time.time() - t}), flush=True)
