"""occ_dplink_allreduce vs ncclAllReduce (torch.distributed) on fp32 buffers of
several sizes, µs per call (CUDA events, max over ranks).  torchrun, N GPUs:
  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/dplink_probe.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2301_09830_b200 import occ  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", rank)))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    comm = occ.Comm.from_process_group()
    sizes = [1 << 10, 1 << 14, 1 << 18, 1 << 20, 1 << 22, 1 << 24]
    dl = occ.DpLink.open(comm, max(sizes))
    reps = 30

    def timed(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) / reps * 1e3], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    for n in sizes:
        x = torch.ones(n, device=dev)
        us_link = timed(lambda: dl.allreduce(x, x))
        y = torch.ones(n, device=dev)
        us_nccl = timed(lambda: dist.all_reduce(y))
        if rank == 0:
            print(json.dumps({"world": world, "floats": n, "bytes": 4 * n, "dplink_us": us_link, "nccl_us": us_nccl,
                              "dplink_GBs_per_rank_pushed": 4 * n * (world - 1) / us_link / 1e3}), flush=True)
    dl.close()
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
