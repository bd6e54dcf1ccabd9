import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2301_09830_b200 import occ
from workloads import synth
shapes = [(3072, 12288), (3072, 9216)]
r = 64
G = [torch.from_numpy(synth.d2_gradlike(n, m, 5 + j)).cuda() for j, (n, m) in enumerate(shapes)]
E = [torch.from_numpy(synth.e0(n, m, 6 + j, like=G[j].cpu().numpy())).cuda() for j, (n, m) in enumerate(shapes)]
Q = [torch.from_numpy(synth.q0(m, r, 7 + j)).cuda() for j, (n, m) in enumerate(shapes)]
P = [torch.empty(n, r, device="cuda") for n, m in shapes]
ws = None
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    ws = occ.occ_allreduce_factors(G, E, Q, P, r, 1.0, 0, ws=ws)
torch.cuda.synchronize()
print("ok")
