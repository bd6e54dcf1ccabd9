"""Device time of one occ_compress step (with the fused reconstruction) for
each BASELINE.json config shape on one GPU, L2 flushed before every step,
CUDA events on the launching stream.  Not part of the bench contract; the
numbers are recorded in DESIGN.md."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_09830_b200 import occ
from workloads import synth

CONFIGS = [("configs[0] 128x256 r4", 128, 256, 4), ("T 1024x3072 r16", 1024, 3072, 16),
           ("configs[1] 4096x1920 r16", 4096, 1920, 16), ("configs[2] 8192x3072 r32", 8192, 3072, 32),
           ("configs[3] MLP 3072x12288 r64", 3072, 12288, 64), ("configs[3] QKV 3072x9216 r64", 3072, 9216, 64)]
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json"))).get("hbm_gbs", 6551) if os.path.exists("MEASURED_PEAKS.json") else 6551
flush = torch.empty(2 * torch.cuda.get_device_properties(0).L2_cache_size // 4, device="cuda").uniform_()
sink = torch.empty(1, device="cuda")
for name, n, m, r in CONFIGS:
    M = torch.from_numpy(synth.d2_gradlike(n, m, 5)).cuda()
    E = torch.zeros_like(M); Q = torch.from_numpy(synth.q0(m, r, 7)).cuda()
    P = torch.empty(n, r, device="cuda"); R = torch.empty_like(M)
    ws = occ.alloc_workspace(n, m, r)
    for _ in range(5):
        occ.occ_compress(M, E, Q, P, R, r=r, ws=ws)
    ts = []
    for _ in range(20):
        torch.sum(flush, dim=0, out=sink[0])
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); occ.occ_compress(M, E, Q, P, R, r=r, ws=ws); b.record()
        torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    ts.sort(); us = ts[len(ts) // 2] * 1e3
    st = occ.occ_read_stats(ws)
    alg = n * m * 16 + (n + m) * r * 8
    print(json.dumps({"config": name, "path": st["path"], "us": round(us, 1), "GB_s": round(n * m * 4 / us / 1e3, 1),
                      "roofline_frac": round(alg / us / 1e3 / peak, 3)}), flush=True)
