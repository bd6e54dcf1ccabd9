"""Per-component device time of the pipeline ring step on 2+ GPUs (torchrun):
occ_compress (no recon), occ_decompress, and the full occ_sendrecv_factors.
Not part of the product."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
from paper_2301_09830_b200 import occ
from workloads import synth

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
dev = torch.device("cuda", torch.cuda.current_device())
dist.init_process_group("nccl", device_id=dev)
comm = occ.Comm.from_process_group()
n, m, r = (int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "4096x1920x16").split("x"))
M = torch.from_numpy(synth.d2_gradlike(n, m, 5 + rank)).to(dev)
E = torch.zeros_like(M); Q = torch.from_numpy(synth.q0(m, r, 7)).to(dev)
P = torch.empty(n, r, device=dev); out = torch.empty_like(M)
Pr, Qr = torch.empty(n, r, device=dev), torch.empty(m, r, device=dev)
ws = occ.alloc_workspace(n, m, r, device=dev)
snd, rcv = (rank - 1) % world, (rank + 1) % world
none = None
cases = {
    "compress (no recon)": lambda: occ.occ_compress(M, E, Q, P, None, r=r, ws=ws),
    "decompress": lambda: occ.occ_decompress(P, Q, out),
    "sendrecv_factors (full step)": lambda: occ.occ_sendrecv_factors(M, E, Q, P, r, snd, out, Pr, Qr, rcv, comm, ws=ws),
}
for name, f in cases.items():
    for _ in range(10): f()
    torch.cuda.synchronize(); dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50): f()
    e1.record(); torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / 50 * 1e3], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0: print(f"{name:32s} {t.item():8.1f} us (back to back, warm L2, max over ranks)", flush=True)
comm.destroy(); dist.destroy_process_group()
