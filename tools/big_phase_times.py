"""One occ_compress (C3 shape) and one occ_allreduce_factors bucket (C4) per
call, for an ncu launch list: the per-kernel device time of the large-shape
path.  Usage: python tools/big_phase_times.py [multi]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2301_09830_b200 import occ  # noqa: E402
from workloads import synth  # noqa: E402

flags = occ.OCC_FORCE_MULTI if "multi" in sys.argv else 0
n, m, r = 8192, 3072, 32
M = torch.from_numpy(synth.d2_gradlike(n, m, 5)).cuda()
E = torch.zeros_like(M)
Q = torch.from_numpy(synth.q0(m, r, 7)).cuda()
P = torch.empty(n, r, device="cuda")
out = torch.empty_like(M)
for _ in range(2):
    occ.occ_compress(M, E, Q, P, None, r=r, flags=flags)
    occ.occ_decompress(P, Q, out)
shapes = [(3072, 12288), (3072, 9216)]
G = [torch.from_numpy(synth.d2_gradlike(a, b, 9)).cuda() for a, b in shapes]
Es = [torch.zeros_like(g) for g in G]
Qs = [torch.from_numpy(synth.q0(b, 64, 7)).cuda() for _, b in shapes]
Ps = [torch.empty(a, 64, device="cuda") for a, _ in shapes]
for _ in range(2):
    occ.occ_allreduce_factors(G, Es, Qs, Ps, 64, 1.0, flags=flags)
torch.cuda.synchronize()
print("ok")
