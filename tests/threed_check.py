"""3D-parallel integration check, run under torchrun with
world = 2 (2 PP x 1 DP) or 4 (2 PP x 2 DP):

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 tests/threed_check.py [--link]

Two iterations of paper_2301_09830_b200.threed.ThreeDStep with warm-up = 1:
iteration 0 is all dense (warm-up bypass, reading C17), iteration 1 applies the
epilogue mask (C10), SC (C11), compressed FE (C14), rank-1 tensors dense (C16).
Rank 0 re-creates every rank's seeded gradients and checks what it received /
holds against the fp64 oracle simulating all ranks: the backward link's LEP
stream (compressed micro-batches vs oracle.compress_step, dense ones vs
M + e_pending with the flush of C9), its stage's DP sync (oracle.dp_step or the
exact mean), the fused embedding sync (embed_sync_fused, or dp_step on the 2D
ranks as G^T), and the rank-1 means.  One JSON line per check on rank 0.
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2301_09830_b200 import occ, policy as pol, threed  # noqa: E402
from workloads import synth  # noqa: E402

SH = threed.StepShapes(act_rows=1024, hidden=768, microbatches=4, cb_rank=16, dp_rank=128,
                       weights=[(512, 1024), (384, 768)], vectors=[768], vocab=2048, emb_rank=16)
ITERS = 2


def act(it, stage, rep, k):
    return synth.d2_gradlike(SH.act_rows, SH.hidden, 10000 + 1000 * it + 100 * stage + 10 * rep + k)


def weight(it, rank, j):
    a, b = SH.weights[j]
    return synth.d2_gradlike(a, b, 20000 + 1000 * it + 10 * rank + j)


def vector(it, rank, j):
    return np.random.default_rng(40000 + 1000 * it + 10 * rank + j).standard_normal(SH.vectors[j]).astype(np.float32)


def emb(it, rank, stage):
    if stage == 0:
        return synth.d5_embedding_sparse(SH.vocab, SH.hidden, 30000 + 1000 * it + rank, tokens=1024)
    return synth.d2_gradlike(SH.vocab, SH.hidden, 30000 + 1000 * it + rank)


def rel(a, b, ref):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(ref), 1e-300))


def main():
    use_link = "--link" in sys.argv
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    P, D = 2, world // 2
    comm = occ.Comm.from_process_group()
    policy = pol.Policy(warmup_iters=1)

    def init_q(Q, seed):   # the oracle's Q0 (reading C5: the same on every rank)
        Q.copy_(torch.from_numpy(synth.q0(Q.shape[0], Q.shape[1], seed)))

    step = threed.ThreeDStep(policy, P, D, comm, SH, dev, use_link=use_link, init_q=init_q)
    stage, rep = step.stage, step.replica
    records = []
    saved = None
    for it in range(ITERS):
        if it == ITERS - 1:
            saved = step.state_dict()   # checkpoint before the last iteration (replayed below)
        rec = {}
        step.backward_sends(it, lambda k: torch.from_numpy(act(it, stage, rep, k)).to(dev), record=rec)
        Ws = [torch.from_numpy(weight(it, rank, j)).to(dev) for j in range(len(SH.weights))]
        Vs = [torch.from_numpy(vector(it, rank, j)).to(dev) for j in range(len(SH.vectors))]
        step.dp_sync(it, Ws, Vs, record=rec)
        G = torch.from_numpy(emb(it, rank, stage)).to(dev) if stage in (0, P - 1) else None
        if G is not None:
            step.embedding_sync(it, G, record=rec)
        torch.cuda.synchronize()
        rec["W"] = [w.double().cpu().numpy() for w in Ws]
        rec["V"] = [v.double().cpu().numpy() for v in Vs]
        rec["G"] = G.double().cpu().numpy() if G is not None else None
        rec["recv"] = [(k, c, o.double().cpu().numpy()) for k, c, o in rec.get("recv", [])]
        records.append(rec)
    # resume: restore the checkpoint and replay the last iteration; every output must repeat bit for bit
    step.load_state_dict(saved)
    it = ITERS - 1
    rec2 = {}
    step.backward_sends(it, lambda k: torch.from_numpy(act(it, stage, rep, k)).to(dev), record=rec2)
    Ws = [torch.from_numpy(weight(it, rank, j)).to(dev) for j in range(len(SH.weights))]
    Vs = [torch.from_numpy(vector(it, rank, j)).to(dev) for j in range(len(SH.vectors))]
    step.dp_sync(it, Ws, Vs)
    G = torch.from_numpy(emb(it, rank, stage)).to(dev) if stage in (0, P - 1) else None
    if G is not None:
        step.embedding_sync(it, G)
    torch.cuda.synchronize()
    same = all(np.array_equal(w.double().cpu().numpy(), records[it]["W"][j]) for j, w in enumerate(Ws))
    same = same and (G is None or np.array_equal(G.double().cpu().numpy(), records[it]["G"]))
    same = same and all(np.array_equal(o.double().cpu().numpy(), r[2])
                        for (_, _, o), r in zip(rec2.get("recv", []), records[it]["recv"]))
    same_t = torch.tensor([1 if same else 0], device=dev)
    dist.all_reduce(same_t, op=dist.ReduceOp.MIN)
    occ.occ_check_status(comm=comm)
    ok = True
    if rank == 0:
        x = {"check": "threed_checkpoint_resume", "bit_identical_replay": bool(same_t.item()), "ok": bool(same_t.item()),
             "world": world, "exchange": "link" if use_link else "nccl"}
        print(json.dumps(x), flush=True)
        ok = ok and x["ok"]
        out = []
        # (1) the backward link into stage 0, replica 0: the sender is stage 1, replica 0
        e = np.zeros((SH.act_rows, SH.hidden))
        Q = synth.q0(SH.hidden, 16, 1234).astype(np.float64)
        worst_c, worst_d, n_c = 0.0, 0.0, 0
        for it in range(ITERS):
            for k, comp, got in records[it]["recv"]:
                M = act(it, 1, 0, k).astype(np.float64)
                want_c = pol.cb_compressed(policy, it, k, SH.microbatches, P, 1)
                assert comp == want_c
                if comp:
                    o = oracle.compress_step(M, e, Q)
                    worst_c = max(worst_c, rel(got, o["recon"], M + e))
                    e, Q = o["err"], o["Q"]
                    n_c += 1
                else:
                    worst_d = max(worst_d, rel(got, (M + e).astype(np.float32), M + e))
                    e = np.zeros_like(e)
        good = worst_c <= 1e-4 and worst_d <= 1e-6 and n_c == ITERS - 1
        out.append({"check": "threed_backward_link", "compressed_microbatches": n_c, "recon_rel_compressed": worst_c,
                    "rel_dense": worst_d, "ok": good})
        # (2) stage 0's DP sync (ranks 0 .. D-1)
        e_dp = [[None] * D for _ in SH.weights]
        Qd = [synth.q0(b, 64, 99).astype(np.float64) for _, b in SH.weights]
        worst = 0.0
        for it in range(ITERS):
            comp = pol.dp_compressed(policy, it, 0, P, 2)
            assert records[it]["dp_compressed"] == comp
            for j in range(len(SH.weights)):
                Ms = [weight(it, pol.rank_of(0, d, D), j) for d in range(D)]
                if comp:
                    o = oracle.dp_step(Ms, e_dp[j], Qd[j], scale=1.0 / D)
                    want = o["recon"]
                    e_dp[j], Qd[j] = o["err"], o["Q"]
                else:
                    want = sum(x.astype(np.float64) for x in Ms) / D
                worst = max(worst, rel(records[it]["W"][j], want, want))
        out.append({"check": "threed_dp_sync_stage0", "recon_rel": worst, "ok": worst <= 1e-4})
        # (3) rank-1 tensors: dense mean
        wv = max(rel(records[it]["V"][j], sum(vector(it, pol.rank_of(0, d, D), j).astype(np.float64)
                                               for d in range(D)) / D, records[it]["V"][j])
                 for it in range(ITERS) for j in range(len(SH.vectors)))
        out.append({"check": "threed_rank1_dense", "rel": wv, "ok": wv <= 1e-6})
        # (4) fused embedding sync over the 2D ranks of the first and last stage
        fe_ranks = pol.fe_group(D, P)
        e_fe, Q_fe = None, synth.q0(SH.vocab, 16, 77).astype(np.float64)
        worst = 0.0
        for it in range(ITERS):
            Gs = [emb(it, rr, rr // D) for rr in fe_ranks]
            comp = records[it]["emb_compressed"]
            assert comp == pol.dp_compressed(policy, it, 0, P, 2)
            if comp:
                o = oracle.dp_step(Gs, e_fe, Q_fe, scale=1.0 / D, orient_t=True)
                want = o["recon"]
                e_fe, Q_fe = o["err"], o["Q"]
            else:
                want = oracle.embed_sync_fused(Gs, D)
            worst = max(worst, rel(records[it]["G"], want, want))
        out.append({"check": "threed_embedding_sync", "ranks": len(fe_ranks), "recon_rel": worst, "ok": worst <= 1e-4})
        for x in out:
            x.update({"world": world, "stages": P, "replicas": D, "exchange": "link" if use_link else "nccl"})
            print(json.dumps(x), flush=True)
            ok = ok and x["ok"]
    flag = torch.tensor([1 if ok else 0], device=dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    step.close()
    comm.destroy()
    dist.destroy_process_group()
    sys.exit(0 if flag.item() else 1)


if __name__ == "__main__":
    main()
