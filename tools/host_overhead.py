"""Host-side cost of one occ_compress call (Python binding + C-ABI validation +
planning + launch), and the device-side gap it can open between a start event
and the kernel.  Not part of the product."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_09830_b200 import occ
from workloads import synth

n, m, r = (int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1024x3072x16").split("x"))
M = torch.from_numpy(synth.d2_gradlike(n, m, 5)).cuda()
E = torch.zeros_like(M)
Q = torch.from_numpy(synth.q0(m, r, 7)).cuda()
P = torch.empty(n, r, device="cuda")
R = torch.empty_like(M)
ws = occ.alloc_workspace(n, m, r)
for _ in range(20):
    occ.occ_compress(M, E, Q, P, R, r=r, ws=ws)
torch.cuda.synchronize()
# host time per call (GPU busy far ahead: a long sleep kernel keeps the queue full)
t0 = time.perf_counter()
N = 200
torch.cuda._sleep(int(2e8))
for _ in range(N):
    occ.occ_compress(M, E, Q, P, R, r=r, ws=ws)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"host time per occ_compress call: {(t1 - t0) / N * 1e6:.1f} us")
# device time per call, back to back (CPU far ahead)
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda._sleep(int(2e8))
ev0.record()
for _ in range(N):
    occ.occ_compress(M, E, Q, P, R, r=r, ws=ws)
ev1.record()
torch.cuda.synchronize()
print(f"device time per call, back to back, warm L2: {ev0.elapsed_time(ev1) / N * 1e3:.1f} us")
