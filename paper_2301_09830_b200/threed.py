"""3D-parallel integration of the compression path.

One training iteration's communication of a P-stage x D-replica pipeline, the
way Optimus-CC drives it (§Background 1F1B; 351-396 §CB;
527-540 epilogue; 562-618 §FE; 627-665 §SC; 684-689 §Impl), on synthetic
gradients: there is no model compute here (training runs, datasets and
weights are out of scope), only the traffic the paper
compresses and the host switches that decide it (policy.py, row a10):

  * backward inter-stage sends of the 1F1B schedule, micro-batch k from stage s
    to s - 1: compressed (occ_send_factors / occ_recv_factors, or the occ_link
    in-kernel exchange) iff policy.cb_compressed(...) -- the epilogue mask
    (reading C10) after the warm-up bypass (C17); otherwise a dense send of
    M + e_pending with the pending lazy error flushed (LEP add-and-flush, C9);
  * the data-parallel gradient sync of every stage: matrices of stages in the SC
    set (ceil(0.75 P) earliest, C11) go through occ_allreduce_factors on the
    stage's DP communicator, rank-1 tensors (bias, LayerNorm) always dense (C16);
  * the tied-embedding sync of the first and last stage fused into one group of
    2D ranks (FE, C12; the group found by name, policy.is_embedding): dense
    occ_embed_sync, or compressed (C14) when the first stage is SC-selected.

Communicators: one occ_comm over all P*D ranks, split into the DP groups
(color = stage), the PP pairs (color = replica) and the FE group (first and
last stage; other ranks take NCCL_SPLIT_NOCOLOR).  Ranks are stage-major
(policy.rank_of).  Every step of the path runs in libocc (occ.py is the ctypes
binding); torch.distributed only carries the dense baseline traffic (the sends
the policy leaves uncompressed) and the rank-1 allreduces.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional

from . import occ, policy as pol

NOCOLOR = -1   # NCCL_SPLIT_NOCOLOR


@dataclass
class StepShapes:
    """Shapes of one iteration's traffic (C5: 8192 x 3072 inter-stage at r 16,
    EMB 50257 x 3072 at r 64 compressed as G^T, weight gradients at r 64)."""
    act_rows: int = 8192            # seq 1024 x micro-batch 8 (reading C6)
    hidden: int = 3072
    microbatches: int = 16          # 512 / (4 replicas x 8)
    cb_rank: int = 16
    dp_rank: int = 64               # the paper's 128, run at the largest built rank (Policy.kernel_rank)
    weights: List[tuple] = field(default_factory=lambda: [(3072, 12288)])   # per stage, 2-D
    vectors: List[int] = field(default_factory=lambda: [3072, 3072])        # per stage, rank-1
    vocab: int = 50257
    emb_rank: int = 64


class ThreeDStep:
    """The communication of one iteration for this rank (stage, replica)."""

    def __init__(self, policy: pol.Policy, stages: int, replicas: int, comm: occ.Comm, shapes: StepShapes,
                 device, use_link: bool = False, init_q: Optional[Callable] = None):
        """init_q(Q, seed) fills a warm-start factor (default occ_init_q; the same
        seed on every rank of a group, reading C5)."""
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.pol, self.P, self.D, self.sh, self.dev = policy, stages, replicas, shapes, device
        self.rank, self.world = comm.rank, comm.nranks
        if self.world != stages * replicas:
            raise ValueError("world size must be stages x replicas")
        self.stage, self.replica = divmod(self.rank, replicas)   # stage-major (policy.rank_of)
        self.comm = comm
        self.dp = comm.split(self.stage, self.replica)
        self.pp = comm.split(self.replica, self.stage)            # pp rank == stage
        in_fe = self.stage in (0, stages - 1)
        self.fe = comm.split(0 if in_fe else NOCOLOR, self.rank)
        # torch groups for the dense baseline traffic (every rank creates every group)
        self.pp_groups = [dist.new_group(pol.pp_group(d, replicas, stages)) for d in range(replicas)]
        self.dp_groups = [dist.new_group(pol.dp_group(s, replicas)) for s in range(stages)]
        n, h, r = shapes.act_rows, shapes.hidden, policy.kernel_rank(shapes.cb_rank)
        f32 = torch.float32
        self.cb_r = r
        # LEP state of this stage's backward link (stage s -> s-1): e and the warm-start Q (C5: same seed)
        self.send = stage_has_send = self.stage >= 1
        self.recv = self.stage < stages - 1
        if stage_has_send:
            self.e = torch.zeros(n, h, device=device, dtype=f32)
            self.Q = torch.empty(h, r, device=device, dtype=f32)
            (init_q or occ.occ_init_q)(self.Q, 1234)
            self.Pbuf = torch.empty(n, r, device=device, dtype=f32)
            self.ws = occ.alloc_workspace(n, h, r, device=device)
        if self.recv:
            self.Pr = torch.empty(n, r, device=device, dtype=f32)
            self.Qr = torch.empty(h, r, device=device, dtype=f32)
        # occ_link: this stage sends to stage - 1, receives from stage + 1 (the pp comm's ranks are stages)
        self.link = None
        if use_link:
            self.link = occ.Link.open(self.pp, self.stage - 1 if self.send else -1,
                                      self.stage + 1 if self.recv else -1, n, h, r)
        # DP error feedback state per weight matrix (SC stages only)
        self.dp_r = policy.kernel_rank(shapes.dp_rank)
        self.dp_state = []
        for (a, b) in shapes.weights:
            q = torch.empty(b, self.dp_r, device=device, dtype=f32)
            (init_q or occ.occ_init_q)(q, 99)
            self.dp_state.append({"e": torch.zeros(a, b, device=device, dtype=f32), "Q": q,
                                  "P": torch.empty(a, self.dp_r, device=device, dtype=f32)})
        nmax = max(a for a, _ in shapes.weights)
        mmax = max(b for _, b in shapes.weights)
        self.dp_ws = occ.alloc_workspace(nmax, mmax, self.dp_r, nmat=len(shapes.weights), device=device)
        # FE state: the embedding gradient compressed as G^T (reading C6): P on the hidden side, Q on the vocab side
        self.emb_r = policy.kernel_rank(shapes.emb_rank)
        if in_fe:
            V = shapes.vocab
            self.emb_e = torch.zeros(V, h, device=device, dtype=f32)
            self.emb_Q = torch.empty(V, self.emb_r, device=device, dtype=f32)
            (init_q or occ.occ_init_q)(self.emb_Q, 77)
            self.emb_P = torch.empty(h, self.emb_r, device=device, dtype=f32)
            self.emb_ws = occ.alloc_workspace(V, h, self.emb_r, device=device)

    # -------------------------------------------------------------- backward sends (1F1B)
    def backward_sends(self, iteration: int, grad: Callable[[int], "object"], record: Optional[Dict] = None):
        """All M micro-batches of the backward link(s) of this rank.  grad(k)
        is stage s's activation gradient for micro-batch k (device, n x h)."""
        torch, dist = self.torch, self.dist
        M, r = self.sh.microbatches, self.cb_r
        g = self.pp_groups[self.replica]
        peer_dn = pol.rank_of(self.stage - 1, self.replica, self.D) if self.send else None
        peer_up = pol.rank_of(self.stage + 1, self.replica, self.D) if self.recv else None
        n, h = self.sh.act_rows, self.sh.hidden
        out = torch.empty(n, h, device=self.dev) if self.recv else None
        for k in range(M):
            # what this stage sends down (it is stage s >= 1) and what it receives from s + 1
            send_c = self.send and pol.cb_compressed(self.pol, iteration, k, M, self.P, self.stage)
            recv_c = self.recv and pol.cb_compressed(self.pol, iteration, k, M, self.P, self.stage + 1)
            if self.link is not None and (send_c or recv_c):
                # one call for both directions; a side with null arguments is skipped
                occ.occ_sendrecv_factors_link(grad(k) if send_c else None, self.e if send_c else None,
                                              self.Q if send_c else None, self.Pbuf if send_c else None, r,
                                              out if recv_c else None, self.Pr if recv_c else None,
                                              self.Qr if recv_c else None, self.link,
                                              ws=self.ws if send_c else None)
            else:
                if send_c:
                    occ.occ_send_factors(grad(k), self.e, self.Q, self.Pbuf, r, self.stage - 1, self.pp, ws=self.ws)
                if recv_c:
                    occ.occ_recv_factors(out, self.Pr, self.Qr, r, self.stage + 1, self.pp)
            if self.send and not send_c:
                # dense send of M + e_pending, then the pending error is flushed (reading C9)
                dense = grad(k) + self.e
                self.e.zero_()
                dist.send(dense, peer_dn, group=g)
            if self.recv and not recv_c:
                dist.recv(out, peer_up, group=g)
            if self.recv and record is not None:
                record.setdefault("recv", []).append((k, recv_c, out.clone()))

    # -------------------------------------------------------------- DP gradient sync (SC)
    def dp_sync(self, iteration: int, weights: List, vectors: List, record: Optional[Dict] = None):
        """weights: this rank's 2-D gradients (in place: the synced mean), vectors: rank-1 ones."""
        dist = self.dist
        g = self.dp_groups[self.stage]
        comp = pol.dp_compressed(self.pol, iteration, self.stage, self.P, 2)
        if comp:
            occ.occ_allreduce_factors(weights, [s["e"] for s in self.dp_state], [s["Q"] for s in self.dp_state],
                                      [s["P"] for s in self.dp_state], self.dp_r, 1.0 / self.D, comm=self.dp,
                                      ws=self.dp_ws)
        else:
            for w in weights:
                dist.all_reduce(w, group=g)
                w.mul_(1.0 / self.D)
        for v in vectors:   # rank-1 tensors: always dense (reading C16)
            dist.all_reduce(v, group=g)
            v.mul_(1.0 / self.D)
        if record is not None:
            record["dp_compressed"] = comp

    # -------------------------------------------------------------- fused embedding sync (FE)
    def embedding_sync(self, iteration: int, G, record: Optional[Dict] = None):
        """G: this rank's tied-embedding gradient (first / last stage only; in place)."""
        if self.stage not in (0, self.P - 1):
            return
        comp = self.pol.fe and pol.dp_compressed(self.pol, iteration, 0, self.P, 2)   # the first stage is in SC
        scale = pol.fe_scale(self.D)
        if comp:
            occ.occ_embed_sync(G, self.emb_e, self.emb_Q, self.emb_P, self.emb_r, scale, self.fe,
                               flags=occ.OCC_ORIENT_T, ws=self.emb_ws)
        else:
            occ.occ_embed_sync(G, None, None, None, 0, scale, self.fe)
        if record is not None:
            record["emb_compressed"] = comp

    # -------------------------------------------------------------- checkpoint / resume
    def state_dict(self) -> Dict:
        """The compression state a resumed run needs: the lazy
        error and warm-start factor of the backward link, the DP error-feedback
        buffers and factors, and the embedding's; tensors are copied."""
        st = {}
        if self.send:
            st["link.e"], st["link.Q"] = self.e.clone(), self.Q.clone()
        for j, d in enumerate(self.dp_state):
            st[f"dp.{j}.e"], st[f"dp.{j}.Q"] = d["e"].clone(), d["Q"].clone()
        if self.stage in (0, self.P - 1):
            st["emb.e"], st["emb.Q"] = self.emb_e.clone(), self.emb_Q.clone()
        return st

    def load_state_dict(self, st: Dict):
        if self.send:
            self.e.copy_(st["link.e"])
            self.Q.copy_(st["link.Q"])
        for j, d in enumerate(self.dp_state):
            d["e"].copy_(st[f"dp.{j}.e"])
            d["Q"].copy_(st[f"dp.{j}.Q"])
        if self.stage in (0, self.P - 1):
            self.emb_e.copy_(st["emb.e"])
            self.emb_Q.copy_(st["emb.Q"])

    def close(self):
        if self.link is not None:
            self.link.close()
        for c in (self.fe, self.pp, self.dp):
            if c is not None:
                c.destroy()


def timed(fn, *a, **kw):
    """(result, device ms) of fn on the current stream."""
    import torch
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    t0 = time.perf_counter()
    res = fn(*a, **kw)
    e.record()
    torch.cuda.synchronize()
    return res, s.elapsed_time(e), (time.perf_counter() - t0) * 1e3
