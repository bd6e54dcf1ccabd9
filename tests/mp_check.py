"""Multi-GPU parity check, run under torchrun (one rank per GPU, NCCL):

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tests/mp_check.py

Checks, against the fp64 oracle simulating all ranks in-process:
  * DP   occ_allreduce_factors over all ranks (local and global EF, reading C1/C2)
  * PP   occ_send_factors (rank 1) -> occ_recv_factors (rank 0) and the sendrecv ring;
         the receiver's M' must equal the sender's own decompression bit for bit
         (reading C8); fp32 and bf16 (OCC_WIRE_BF16, C7) wire factors
  * EMB  occ_embed_sync dense (r = 0, reading C12) and compressed (r > 0, C14)
Prints one JSON line per check on rank 0 and exits non-zero on any failure.
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
from paper_2301_09830_b200 import occ  # noqa: E402
from workloads import synth  # noqa: E402


def rel(a, b, ref):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(ref), 1e-300))


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    comm = occ.Comm.from_process_group()
    assert comm.rank == rank and comm.nranks == world
    ok = True

    def report(name, **kw):
        nonlocal ok
        good = kw.pop("ok")
        ok = ok and good
        if rank == 0:
            print(json.dumps({"check": name, "world": world, "ok": bool(good), **kw}), flush=True)

    def gather_np(t):
        out = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(out, t.contiguous())
        return [x.double().cpu().numpy() for x in out]

    # ------------------------------------------------------------------ DP
    for flags, name in ((0, "dp_local_ef"), (occ.OCC_EF_GLOBAL, "dp_global_ef")):
        n, m, r = 768, 1024, 16
        Ms = [synth.d2_gradlike(n, m, 500 + w) for w in range(world)]
        Es = [synth.e0(n, m, 600 + w, like=Ms[w]) for w in range(world)]
        Q0 = synth.q0(m, r, 7)
        G = torch.from_numpy(Ms[rank]).to(dev)
        E = torch.from_numpy(Es[rank]).to(dev)
        Q = torch.from_numpy(Q0).to(dev)
        P = torch.empty(n, r, device=dev)
        occ.occ_allreduce_factors([G], [E], [Q], [P], r, 1.0 / world, flags=flags, comm=comm)
        torch.cuda.synchronize()
        o = oracle.dp_step(Ms, Es, Q0, scale=1.0 / world, ef_global=bool(flags & occ.OCC_EF_GLOBAL))
        A = sum(Ms[w].astype(np.float64) + Es[w] for w in range(world))
        gs, es = gather_np(G), gather_np(E)
        e_recon = max(rel(gs[w], o["recon"], A / world) for w in range(world))
        e_err = max(rel(es[w], o["err"][w], Ms[w].astype(np.float64) + Es[w]) for w in range(world))
        same = all(np.array_equal(gs[0], gs[w]) for w in range(world))
        orth = float(np.linalg.norm(P.double().cpu().numpy().T @ P.double().cpu().numpy() - np.eye(r)))
        q_rel = rel(Q.double().cpu().numpy(), o["Q"], o["Q"])
        report(name, recon_rel=e_recon, err_rel=e_err, q_rel=q_rel, orth=orth, identical_on_ranks=same,
               ok=e_recon <= 1e-4 and e_err <= 1e-4 and same and orth <= 1e-5 and q_rel <= 1e-3)

    # ------------------------------------------------------------------ DP, OCC_ORIENT_T (reading C6)
    for flags, name in ((occ.OCC_ORIENT_T, "dp_orient_t_local_ef"),
                        (occ.OCC_ORIENT_T | occ.OCC_EF_GLOBAL, "dp_orient_t_global_ef")):
        n, m, r = 1536, 512, 16      # tall, like the 50257 x 3072 embedding
        Ms = [synth.d2_gradlike(n, m, 520 + w) for w in range(world)]
        Es = [synth.e0(n, m, 620 + w, like=Ms[w]) for w in range(world)]
        Q0 = synth.q0(n, r, 13)      # row side with OCC_ORIENT_T
        G = torch.from_numpy(Ms[rank]).to(dev)
        E = torch.from_numpy(Es[rank]).to(dev)
        Q = torch.from_numpy(Q0).to(dev)
        P = torch.empty(m, r, device=dev)
        occ.occ_allreduce_factors([G], [E], [Q], [P], r, 1.0 / world, flags=flags, comm=comm)
        torch.cuda.synchronize()
        o = oracle.dp_step(Ms, Es, Q0, scale=1.0 / world, ef_global=bool(flags & occ.OCC_EF_GLOBAL), orient_t=True)
        A = sum(Ms[w].astype(np.float64) + Es[w] for w in range(world))
        gs, es = gather_np(G), gather_np(E)
        e_recon = max(rel(gs[w], o["recon"], A / world) for w in range(world))
        e_err = max(rel(es[w], o["err"][w], Ms[w].astype(np.float64) + Es[w]) for w in range(world))
        same = all(np.array_equal(gs[0], gs[w]) for w in range(world))
        Ph = P.double().cpu().numpy()
        orth = float(np.linalg.norm(Ph.T @ Ph - np.eye(r)))
        q_rel = rel(Q.double().cpu().numpy(), o["Q"], o["Q"])
        report(name, recon_rel=e_recon, err_rel=e_err, q_rel=q_rel, orth=orth, identical_on_ranks=same,
               ok=e_recon <= 1e-4 and e_err <= 1e-4 and same and orth <= 1e-5 and q_rel <= 1e-3)

    # ------------------------------------------------------------------ DP over the in-kernel exchange (occ_dplink, f1)
    dl = occ.DpLink.open(comm, (12288 + 9216) * 64)
    for flags, name, (n, m, r) in ((0, "dp_link_local_ef", (768, 1024, 16)),
                                   (occ.OCC_EF_GLOBAL, "dp_link_global_ef", (768, 1024, 16)),
                                   (occ.OCC_ORIENT_T, "dp_link_orient_t", (1536, 512, 16)),
                                   (0, "dp_link_c4_mlp_r64", (3072, 12288, 64))):
        ot = bool(flags & occ.OCC_ORIENT_T)
        Ms = [synth.d2_gradlike(n, m, 540 + w) for w in range(world)]
        Es = [synth.e0(n, m, 640 + w, like=Ms[w]) for w in range(world)]
        Q0 = synth.q0(n if ot else m, r, 17)
        G = torch.from_numpy(Ms[rank]).to(dev)
        E = torch.from_numpy(Es[rank]).to(dev)
        Q = torch.from_numpy(Q0).to(dev)
        P = torch.empty(m if ot else n, r, device=dev)
        occ.occ_allreduce_factors_link([G], [E], [Q], [P], r, 1.0 / world, dl, flags=flags)
        occ.occ_check_status(comm=comm)
        o = oracle.dp_step(Ms, Es, Q0, scale=1.0 / world, ef_global=bool(flags & occ.OCC_EF_GLOBAL), orient_t=ot)
        A = sum(Ms[w].astype(np.float64) + Es[w] for w in range(world))
        gs, es = gather_np(G), gather_np(E)
        e_recon = max(rel(gs[w], o["recon"], A / world) for w in range(world))
        e_err = max(rel(es[w], o["err"][w], Ms[w].astype(np.float64) + Es[w]) for w in range(world))
        same = all(np.array_equal(gs[0], gs[w]) for w in range(world))
        Ph = P.double().cpu().numpy()
        orth = float(np.linalg.norm(Ph.T @ Ph - np.eye(r)))
        q_rel = rel(Q.double().cpu().numpy(), o["Q"], o["Q"])
        report(name, recon_rel=e_recon, err_rel=e_err, q_rel=q_rel, orth=orth, identical_on_ranks=same,
               ok=e_recon <= 1e-4 and e_err <= 1e-4 and same and orth <= 1e-5 and q_rel <= 1e-3)
    # slot reuse: 6 back-to-back calls (each slot three times), every rank identical
    n, m, r = 512, 768, 16
    G = torch.from_numpy(synth.d2_gradlike(n, m, 560 + rank)).to(dev)
    E = torch.zeros(n, m, device=dev)
    Q = torch.from_numpy(synth.q0(m, r, 19)).to(dev)
    P = torch.empty(n, r, device=dev)
    for _ in range(6):
        occ.occ_allreduce_factors_link([G], [E], [Q], [P], r, 1.0 / world, dl)
    occ.occ_check_status(comm=comm)
    qs = gather_np(Q)
    report("dp_link_slot_reuse", calls=6, identical_on_ranks=all(np.array_equal(qs[0], x) for x in qs),
           finite=bool(torch.isfinite(Q).all()),
           ok=all(np.array_equal(qs[0], x) for x in qs) and bool(torch.isfinite(Q).all()))
    dl.close()

    # PP checks run twice: fp32 factors, and OCC_WIRE_BF16 (reading C7: bf16 factors on
    # the wire, e_new against them; the oracle rounds its fp64 factors the same way,
    # so a few elements may differ by one bf16 ulp -> 1e-3)
    for wflags, sfx, wb, tolr in ((0, "", False, 1e-4), (occ.OCC_WIRE_BF16, "_wire_bf16", True, 1e-3)):
        # ------------------------------------------------------------------ PP (pairs 1 -> 0, 3 -> 2, ...)
        if world >= 2:
            n, m, r = 8192, 3072, 32      # BASELINE configs[2]: GPT-8.3B inter-stage, 1024 tokens x mb 8
            sender = rank % 2 == 1
            peer = rank - 1 if sender else rank + 1
            pair = rank // 2
            M = synth.d2_gradlike(n, m, 700 + pair)
            E0 = synth.e0(n, m, 800 + pair, like=M)
            Q0 = synth.q0(m, r, 9)
            if peer < world:
                if sender:
                    Md, Ed, Qd = (torch.from_numpy(x).to(dev) for x in (M, E0, Q0))
                    Pd = torch.empty(n, r, device=dev)
                    occ.occ_send_factors(Md, Ed, Qd, Pd, r, peer, comm, flags=wflags)
                    own = torch.empty(n, m, device=dev)
                    occ.occ_decompress(Pd, Qd, own)          # what the sender's residual assumes
                    torch.cuda.synchronize()
                    dist.send(own, peer)
                    dist.send(Ed, peer)
                else:
                    out = torch.empty(n, m, device=dev)
                    Pr = torch.empty(n, r, device=dev)
                    Qr = torch.empty(m, r, device=dev)
                    occ.occ_recv_factors(out, Pr, Qr, r, peer, comm, flags=wflags)
                    torch.cuda.synchronize()
                    own, e_snd = torch.empty(n, m, device=dev), torch.empty(n, m, device=dev)
                    dist.recv(own, peer)
                    dist.recv(e_snd, peer)
                    own, e_snd = own.cpu(), e_snd.cpu()
                    o = oracle.compress_step(M, E0, Q0, wire_bf16=wb)
                    A = M.astype(np.float64) + E0
                    got = out.double().cpu().numpy()
                    r_rel = rel(got, o["recon"], A)
                    bit = bool(torch.equal(out.cpu(), own))
                    ef = rel(got + e_snd.double().numpy(), A, A)   # sender's e_new + receiver's M' = A
                    good = r_rel <= tolr and bit and ef <= 1e-6
                    flag = torch.tensor([1 if good else 0], device=dev)
            flags_t = torch.tensor([1], device=dev)
            if peer < world and not sender:
                flags_t = flag
            dist.all_reduce(flags_t, op=dist.ReduceOp.MIN)
            if rank == 0:
                report("pp_send_recv" + sfx, recon_rel=r_rel, bitwise_equal_to_sender=bit, ef_identity=ef,
                       ok=bool(flags_t.item()))
            else:
                ok = ok and bool(flags_t.item())

        # ------------------------------------------------------------------ PP ring (1F1B steady state)
        # every rank compresses its own gradient and sends the factors to rank - 1
        # while receiving rank + 1's and decompressing them (occ_sendrecv_factors)
        if world >= 2:
            n, m, r = 1024, 3072, 16      # north-star target T
            mats = [synth.d2_gradlike(n, m, 1100 + w) for w in range(world)]
            errs = [synth.e0(n, m, 1200 + w, like=mats[w]) for w in range(world)]
            Q0 = synth.q0(m, r, 17)
            Md, Ed, Qd = (torch.from_numpy(x).to(dev) for x in (mats[rank], errs[rank], Q0))
            Pd = torch.empty(n, r, device=dev)
            out = torch.empty(n, m, device=dev)
            Pr, Qr = torch.empty(n, r, device=dev), torch.empty(m, r, device=dev)
            snd, rcv = (rank - 1) % world, (rank + 1) % world
            occ.occ_sendrecv_factors(Md, Ed, Qd, Pd, r, snd, out, Pr, Qr, rcv, comm, flags=wflags)
            own = torch.empty(n, m, device=dev)
            occ.occ_decompress(Pd, Qd, own)          # what this rank's residual assumes
            torch.cuda.synchronize()
            owns = gather_np(own)
            o = oracle.compress_step(mats[rcv], errs[rcv], Q0, wire_bf16=wb)
            A = mats[rcv].astype(np.float64) + errs[rcv]
            got = out.double().cpu().numpy()
            r_rel = rel(got, o["recon"], A)
            bit = bool(np.array_equal(got, owns[rcv]))
            good = torch.tensor([1 if (r_rel <= tolr and bit) else 0], device=dev)
            dist.all_reduce(good, op=dist.ReduceOp.MIN)
            report("pp_ring_sendrecv" + sfx, recon_rel=r_rel, bitwise_equal_to_sender=bit, ok=bool(good.item()))

    # ------------------------------------------------------------------ PP ring over occ_link (f1)
    # the same 1F1B ring with the in-kernel NVLink exchange: the compression
    # kernel pushes (P_hat, Q) into rank - 1's mailbox, rank + 1's factors are
    # decompressed straight from ours; 4 steps (both mailbox slots reused)
    if world >= 2:
        for wflags, sfx, wb, tolr, (n, m, r) in ((0, "", False, 1e-4, (1024, 3072, 16)),
                                                  (occ.OCC_WIRE_BF16, "_wire_bf16", True, 1e-3, (1024, 3072, 16)),
                                                  (0, "_r64_perphase", False, 1e-4, (1536, 2048, 64))):
            steps = 4
            snd, rcv = (rank - 1) % world, (rank + 1) % world
            link = occ.Link.open(comm, snd, rcv, n, m, r)
            streams = [synth.d3_lep_stream(n, m, 1500 + w, steps) for w in range(world)]
            e0s = [synth.e0(n, m, 1600 + w, like=streams[w][0]) for w in range(world)]
            Q0 = synth.q0(m, r, 21)
            Ed, Qd = torch.from_numpy(e0s[rank]).to(dev), torch.from_numpy(Q0).to(dev)
            Pd = torch.empty(n, r, device=dev)
            out = torch.empty(n, m, device=dev)
            Pr, Qr = torch.empty(n, r, device=dev), torch.empty(m, r, device=dev)
            e_o, Q_o = e0s[rcv].astype(np.float64), Q0.astype(np.float64)   # the oracle follows rank + 1's stream
            worst, bit = 0.0, True
            for t in range(steps):
                Md = torch.from_numpy(streams[rank][t]).to(dev)
                occ.occ_sendrecv_factors_link(Md, Ed, Qd, Pd, r, out, Pr, Qr, link, flags=wflags)
                own = torch.empty_like(out)
                occ.occ_decompress(Pd, Qd, own)
                torch.cuda.synchronize()
                owns = gather_np(own)
                got = out.double().cpu().numpy()
                bit = bit and bool(np.array_equal(got, owns[rcv]))
                o = oracle.compress_step(streams[rcv][t], e_o, Q_o, wire_bf16=wb)
                worst = max(worst, rel(got, o["recon"], streams[rcv][t].astype(np.float64) + e_o))
                e_o, Q_o = o["err"], o["Q"]
            occ.occ_check_status(comm=comm)
            link.close()
            good = torch.tensor([1 if (worst <= tolr and bit) else 0], device=dev)
            dist.all_reduce(good, op=dist.ReduceOp.MIN)
            report("pp_ring_link" + sfx, steps=steps, recon_rel_worst=worst, bitwise_equal_to_sender=bit,
                   ok=bool(good.item()))

    # ------------------------------------------------------------------ EMB dense (fused, reading C12)
    V, h = 4096, 1024
    D = max(1, world // 2)
    Gs = [synth.d5_embedding_sparse(V, h, 900 + w) if w < D else synth.d2_gradlike(V, h, 900 + w)
          for w in range(world)]
    G = torch.from_numpy(Gs[rank]).to(dev)
    occ.occ_embed_sync(G, None, None, None, 0, 1.0 / D, comm)
    torch.cuda.synchronize()
    want = oracle.embed_sync_fused(Gs, D)
    got = G.double().cpu().numpy()
    e1 = rel(got, want, want)
    report("emb_dense", rel=e1, ok=e1 <= 1e-6)

    # ------------------------------------------------------------------ EMB compressed (r > 0)
    r = 16
    G = torch.from_numpy(Gs[rank]).to(dev)
    E = torch.zeros(V, h, device=dev)
    Q0 = synth.q0(h, r, 11)
    Q = torch.from_numpy(Q0).to(dev)
    P = torch.empty(V, r, device=dev)
    occ.occ_embed_sync(G, E, Q, P, r, 1.0 / D, comm)
    torch.cuda.synchronize()
    o = oracle.dp_step(Gs, None, Q0, scale=1.0 / D)
    A = sum(g.astype(np.float64) for g in Gs)
    e2 = rel(G.double().cpu().numpy(), o["recon"], A / D)
    report("emb_compressed", recon_rel=e2, ok=e2 <= 1e-4)

    # ------------------------------------------------------------------ EMB compressed as G^T (C5, reading C6)
    G = torch.from_numpy(Gs[rank]).to(dev)
    E = torch.zeros(V, h, device=dev)
    Q0 = synth.q0(V, r, 12)
    Q = torch.from_numpy(Q0).to(dev)
    P = torch.empty(h, r, device=dev)
    occ.occ_embed_sync(G, E, Q, P, r, 1.0 / D, comm, flags=occ.OCC_ORIENT_T)
    torch.cuda.synchronize()
    o = oracle.dp_step(Gs, None, Q0, scale=1.0 / D, orient_t=True)
    e3 = rel(G.double().cpu().numpy(), o["recon"], A / D)
    report("emb_compressed_orient_t", recon_rel=e3, ok=e3 <= 1e-4)

    # ------------------------------------------------------------------ C5 EMB at full size (BASELINE configs[4])
    # the 50257 x 3072 tied-embedding gradient, compressed as G^T (OCC_ORIENT_T,
    # reading C6) at r = 64 over all ranks (first stage ranks: row-sparse D5,
    # last stage ranks: dense D2), scale 1/D (reading C12/C14).  Rank 0 runs the
    # oracle on every rank's input; M' must be bit-identical on all ranks.
    if os.environ.get("OCC_MP_FULL_EMB", "1") == "1":
        V, h, r = 50257, 3072, 64
        D = max(1, world // 2)
        mk = lambda w: synth.d5_embedding_sparse(V, h, 1400 + w) if w < D else synth.d2_gradlike(V, h, 1400 + w)
        Gw = mk(rank)
        Q0 = synth.q0(V, r, 15)
        G = torch.from_numpy(Gw).to(dev)
        E = torch.zeros(V, h, device=dev)
        Q = torch.from_numpy(Q0).to(dev)
        P = torch.empty(h, r, device=dev)
        occ.occ_embed_sync(G, E, Q, P, r, 1.0 / D, comm, flags=occ.OCC_ORIENT_T)
        torch.cuda.synchronize()
        csum = torch.tensor([float(G.double().sum()), float((G.double() ** 2).sum())], device=dev, dtype=torch.float64)
        allc = [torch.empty_like(csum) for _ in range(world)]
        dist.all_gather(allc, csum)
        same = all(torch.equal(allc[0], c) for c in allc)
        if rank == 0:
            Gs = [mk(w) for w in range(world)]
            o = oracle.dp_step(Gs, None, Q0, scale=1.0 / D, orient_t=True)
            A = sum(g.astype(np.float64) for g in Gs)
            got = G.double().cpu().numpy()
            e4 = rel(got, o["recon"], A / D)
            el = float(np.abs(got - o["recon"]).max() / np.abs(A / D).max())
            ee = rel(E.double().cpu().numpy(), o["err"][0], Gs[0].astype(np.float64))
            Ph = P.double().cpu().numpy()
            orth = float(np.linalg.norm(Ph.T @ Ph - np.eye(r)))
            good = e4 <= 1e-4 and el <= 1e-5 and ee <= 1e-4 and orth <= 1e-5 and same
            del Gs, o, A
        else:
            e4 = el = ee = orth = None
            good = True
        g_t = torch.tensor([1 if good else 0], device=dev)
        dist.all_reduce(g_t, op=dist.ReduceOp.MIN)
        report("emb_compressed_orient_t_full_50257x3072_r64", recon_rel=e4, recon_elem=el, err_rel_rank0=ee,
               orth=orth, identical_on_ranks=same, ok=bool(g_t.item()))
        del G, E, Q, P, Gw

    # ------------------------------------------------------------------ occ_comm_wrap (torch's communicator)
    try:
        ptr = dist.distributed_c10d._get_default_group()._get_backend(dev)._comm_ptr()
    except Exception as exc:   # private torch API: report, do not fail
        ptr = None
        report("comm_wrap", skipped=str(exc)[:80], ok=True)
    if ptr:
        wrapped = occ.Comm.wrap(ptr)
        n, m, r = 512, 768, 8
        Ms = [synth.d2_gradlike(n, m, 1300 + w) for w in range(world)]
        Q0 = synth.q0(m, r, 19)
        outs = []
        for cm in (wrapped, comm):
            G = torch.from_numpy(Ms[rank]).to(dev)
            Q = torch.from_numpy(Q0).to(dev)
            P = torch.empty(n, r, device=dev)
            occ.occ_allreduce_factors([G], None, [Q], [P], r, 1.0 / world, flags=occ.OCC_NO_EF, comm=cm)
            torch.cuda.synchronize()
            outs.append(G.cpu())
        same = bool(torch.equal(outs[0], outs[1]))
        report("comm_wrap", nranks=wrapped.nranks, same_result_as_own_comm=same,
               ok=same and wrapped.nranks == world and wrapped.rank == rank)
        wrapped.destroy()   # frees only the handle

    comm.destroy()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
