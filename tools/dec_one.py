import os, sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2301_09830_b200 import occ
n, m, r = 4096, 1920, 16
P = torch.randn(n, r, device="cuda"); Q = torch.randn(m, r, device="cuda"); out = torch.empty(n, m, device="cuda")
for _ in range(3): occ.occ_decompress(P, Q, out)
torch.cuda.synchronize(); print("ok")
