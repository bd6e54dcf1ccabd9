"""Timing of one iteration's communication of the 2 PP x D DP step at the
BASELINE configs[4] (C5) sizes (paper_2301_09830_b200/threed.py): 16 micro-batches
of the 8192 x 3072 inter-stage gradient at r 16 under the epilogue mask,
stage DP sync of 3072 x 12288 + 3072 x 9216 weight gradients at r 64 (SC), and
the 50257 x 3072 fused embedding sync at r 64 as G^T over the 2D ranks.
Synthetic device gradients (no oracle; tests/threed_check.py checks parity at
small sizes).  torchrun --nproc-per-node 4 tools/run_3d.py [--link] [--iters 3]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2301_09830_b200 import occ, policy as pol, threed  # noqa: E402


def main():
    use_link = "--link" in sys.argv
    iters = int(sys.argv[sys.argv.index("--iters") + 1]) if "--iters" in sys.argv else 3
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    P, D = 2, world // 2
    comm = occ.Comm.from_process_group()
    sh = threed.StepShapes(weights=[(3072, 12288), (3072, 9216)])
    policy = pol.Policy(warmup_iters=0)
    step = threed.ThreeDStep(policy, P, D, comm, sh, dev, use_link=use_link)
    g = torch.Generator(device=dev).manual_seed(rank)
    base = torch.randn(sh.act_rows, sh.hidden, device=dev, generator=g) * 1e-2
    acts = [base + 1e-3 * torch.randn(sh.act_rows, sh.hidden, device=dev, generator=g) for _ in range(2)]
    Ws0 = [torch.randn(a, b, device=dev, generator=g) * 1e-2 for a, b in sh.weights]
    Vs0 = [torch.randn(v, device=dev, generator=g) for v in sh.vectors]
    G0 = torch.randn(sh.vocab, sh.hidden, device=dev, generator=g) * 1e-3 if step.stage in (0, P - 1) else None
    res = []
    for it in range(iters):
        Ws, Vs = [w.clone() for w in Ws0], [v.clone() for v in Vs0]
        G = G0.clone() if G0 is not None else None
        torch.cuda.synchronize()
        dist.barrier()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record()
        step.backward_sends(it, lambda k: acts[k % 2])
        ev[1].record()
        step.dp_sync(it, Ws, Vs)
        ev[2].record()
        if G is not None:
            step.embedding_sync(it, G)
        ev[3].record()
        torch.cuda.synchronize()
        t = [ev[i].elapsed_time(ev[i + 1]) for i in range(3)]
        tt = torch.tensor(t, device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        res.append(tt.tolist())
    occ.occ_check_status(comm=comm)
    if rank == 0:
        last = res[-1]
        print(json.dumps({"workload": "C5: 2 PP x %d DP, 16 micro-batches 8192x3072 r16 (epilogue mask: k=15), "
                                      "DP {3072x12288, 3072x9216} r64 (SC both stages), EMB 50257x3072 r64 as G^T "
                                      "over %d ranks" % (D, 2 * D),
                          "exchange": "link" if use_link else "nccl", "world": world, "iters": iters,
                          "backward_sends_ms": last[0], "dp_sync_ms": last[1], "embedding_sync_ms": last[2],
                          "all_iters_ms": res, "note": "device time, max over ranks, last iteration; dense "
                                                       "micro-batch sends are torch.distributed (the baseline)"}),
              flush=True)
    step.close()
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
