"""Per-phase launches of the per-phase (v1) path for one shape, for an ncu
launch list (OCC_FORCE_MULTI).  Not part of the product."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_09830_b200 import occ
from workloads import synth
n, m, r = (int(x) for x in sys.argv[1].split("x"))
M = torch.from_numpy(synth.d2_gradlike(n, m, 5)).cuda(); E = torch.zeros_like(M)
Q = torch.from_numpy(synth.q0(m, r, 7)).cuda(); P = torch.empty(n, r, device="cuda"); R = torch.empty_like(M)
ws = occ.alloc_workspace(n, m, r)
for _ in range(3):
    occ.occ_compress(M, E, Q, P, R, r=r, ws=ws, flags=occ.OCC_FORCE_MULTI)
torch.cuda.synchronize(); print("ok")
