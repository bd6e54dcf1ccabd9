"""Device time of occ_decompress (fp32 out) per rank for one shape, L2 flushed
before every call, CUDA events, median of 20; with the HBM bytes the output
write alone needs (the floor).  Not part of the product.
    python tools/dec_times.py [n m]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json
import torch
from paper_2301_09830_b200 import occ
n, m = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (3072, 12288)
flush = torch.empty(2 * torch.cuda.get_device_properties(0).L2_cache_size // 4, device="cuda").uniform_()
sink = torch.empty(1, device="cuda")
out = torch.empty(n, m, device="cuda")
for r in (8, 16, 32, 64):
    P = torch.randn(n, r, device="cuda"); Q = torch.randn(m, r, device="cuda")
    for _ in range(3):
        occ.occ_decompress(P, Q, out)
    ts = []
    for _ in range(20):
        torch.sum(flush, dim=0, out=sink[0])
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); occ.occ_decompress(P, Q, out); b.record()
        torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    us = sorted(ts)[10] * 1e3
    print(json.dumps({"n": n, "m": m, "r": r, "us": round(us, 1), "write_GB_s": round(n * m * 4 / us / 1e3, 1)}), flush=True)
