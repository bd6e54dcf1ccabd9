"""NCCL point-to-point / allreduce latency over the box's interconnect for the
factor-message sizes of the hot path (torchrun, 2+ ranks).  Not part of the
product.  Prints the transport lines NCCL_DEBUG=INFO reports on rank 0."""
import os, sys, time
import torch, torch.distributed as dist

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
dev = torch.device("cuda", torch.cuda.current_device())
dist.init_process_group("nccl", device_id=dev)
snd, rcv = (rank - 1) % world, (rank + 1) % world
for kb in (4, 64, 256, 1024, 4096):
    a = torch.zeros(kb * 256, device=dev); b = torch.zeros_like(a)
    def x():
        for r in dist.batch_isend_irecv([dist.P2POp(dist.isend, a, snd), dist.P2POp(dist.irecv, b, rcv)]):
            r.wait()
    for _ in range(10): x()
    torch.cuda.synchronize(); dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(100): x()
    e1.record(); torch.cuda.synchronize()
    t_p2p = e0.elapsed_time(e1) / 100 * 1e3
    for _ in range(10): dist.all_reduce(a)
    torch.cuda.synchronize(); dist.barrier()
    e0.record()
    for _ in range(100): dist.all_reduce(a)
    e1.record(); torch.cuda.synchronize()
    t_ar = e0.elapsed_time(e1) / 100 * 1e3
    if rank == 0:
        print(f"{kb:6d} KB: sendrecv ring {t_p2p:8.1f} us ({kb / 1024 / t_p2p * 1e6 / 1e3:7.1f} GB/s)   allreduce {t_ar:8.1f} us", flush=True)
dist.destroy_process_group()
