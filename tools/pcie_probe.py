"""Host-link probe for the e2e figure: every rank copies the bench's M (4096 x 1920
fp32, 31.5 MB) pinned-host -> device and M' device -> pinned-host, on two streams
at once (as bench.py's e2e loop does), with no compute.  Prints per-rank and
aggregate GB/s per direction; the e2e step cannot beat this.

    torchrun --nproc-per-node N tools/pcie_probe.py
"""
import json
import os

import torch
import torch.distributed as dist


def main():
    rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(dev)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    nbytes = 4096 * 1920 * 4
    hin = torch.empty(nbytes // 4, dtype=torch.float32).pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    din, dout = torch.empty_like(hin, device=dev), torch.empty_like(hin, device=dev)
    s1, s2 = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    res = {}
    for mode in ("h2d", "d2h", "both"):
        for it in range(2):   # warm-up, timed
            k = 20
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record()
            s1.wait_stream(torch.cuda.current_stream())
            s2.wait_stream(torch.cuda.current_stream())
            for _ in range(k):
                if mode in ("h2d", "both"):
                    with torch.cuda.stream(s1):
                        din.copy_(hin, non_blocking=True)
                if mode in ("d2h", "both"):
                    with torch.cuda.stream(s2):
                        hout.copy_(dout, non_blocking=True)
            torch.cuda.current_stream().wait_stream(s1)
            torch.cuda.current_stream().wait_stream(s2)
            t1.record()
            torch.cuda.synchronize()
        ms = torch.tensor([t0.elapsed_time(t1) / k], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        res[mode] = {"ms_per_copy": ms.item(), "per_rank_gbs_per_direction": nbytes / (ms.item() * 1e-3) / 1e9,
                     "aggregate_gbs_per_direction": world * nbytes / (ms.item() * 1e-3) / 1e9}
    if rank == 0:
        print(json.dumps({"world": world, "bytes_per_copy": nbytes, **res}), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
