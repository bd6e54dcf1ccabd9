"""Thin ctypes binding of libocc.so (include/occ.h).  Argument marshalling only:
every step of the hot path runs in the library's CUDA kernels / NCCL calls.

The function names are the C names.  Tensors are torch CUDA tensors (torch is
used for device memory, streams and process groups only).  There is no CPU
fallback: if libocc.so is missing or fails to load, every call raises.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

HERE = os.path.dirname(os.path.abspath(__file__))
# OCC_LIB=trace selects the instrumented build (libocc_trace.so, tools/trace.py)
LIB_PATH = os.path.join(HERE, "libocc_trace.so" if os.environ.get("OCC_LIB") == "trace" else "libocc.so")

OCC_F32, OCC_BF16 = 0, 1
OCC_NO_EF = 1
OCC_EF_GLOBAL = 2
OCC_CHECK_FINITE = 4
OCC_WIRE_BF16 = 8
OCC_ORIENT_T = 16
OCC_FORCE_MULTI = 64
OCC_FORCE_TWO_PASS = 128
SUPPORTED_RANKS = (4, 8, 16, 32, 64)

STATUS = ["OCC_OK", "OCC_ERR_INVALID_ARG", "OCC_ERR_SHAPE", "OCC_ERR_DTYPE", "OCC_ERR_RANK",
          "OCC_ERR_ALIGN", "OCC_ERR_ALIAS", "OCC_ERR_WORKSPACE", "OCC_ERR_CUDA", "OCC_ERR_NCCL",
          "OCC_ERR_NONFINITE", "OCC_ERR_UNSUPPORTED"]


class occ_mat(ctypes.Structure):
    _fields_ = [("ptr", ctypes.c_void_p), ("rows", ctypes.c_int64), ("cols", ctypes.c_int64),
                ("ld", ctypes.c_int64), ("dtype", ctypes.c_int)]


class occ_stats(ctypes.Structure):
    _fields_ = [("fallback_columns", ctypes.c_int32), ("second_pass", ctypes.c_int32),
                ("kappa_est", ctypes.c_double), ("path", ctypes.c_int32), ("grid", ctypes.c_int32),
                ("t_ns", ctypes.c_uint64 * 12), ("q_amp", ctypes.c_double), ("q_fused", ctypes.c_int32)]


class OccError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        self.status = status
        self.name = STATUS[status] if 0 <= status < len(STATUS) else f"status {status}"
        super().__init__(f"{where}: {self.name}: {detail}")


_lib = None


def lib():
    """Load libocc.so (raises if it is absent: no silent fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} not built; run `python -m paper_2301_09830_b200.build`")
    L = ctypes.CDLL(LIB_PATH)
    vp, i64, c_int, u32, u64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_uint32, ctypes.c_uint64
    M = occ_mat
    sig = {
        "occ_status_string": ([c_int], ctypes.c_char_p),
        "occ_last_error": ([], ctypes.c_char_p),
        "occ_version": ([], ctypes.c_char_p),
        "occ_workspace_bytes": ([i64, i64, c_int, c_int, u32], ctypes.c_size_t),
        "occ_init_q": ([M, u64, vp], c_int),
        "occ_compress": ([M, M, M, M, M, c_int, u32, vp, ctypes.c_size_t, vp], c_int),
        "occ_decompress": ([M, M, M, vp], c_int),
        "occ_allreduce_factors": ([c_int, ctypes.POINTER(M), ctypes.POINTER(M), ctypes.POINTER(M),
                                   ctypes.POINTER(M), ctypes.POINTER(c_int), ctypes.c_float, u32, vp, vp,
                                   ctypes.c_size_t, vp], c_int),
        "occ_send_factors": ([M, M, M, M, c_int, c_int, u32, vp, vp, ctypes.c_size_t, vp], c_int),
        "occ_recv_factors": ([M, M, M, c_int, c_int, u32, vp, vp], c_int),
        "occ_sendrecv_factors": ([M, M, M, M, c_int, c_int, M, M, M, c_int, u32, vp, vp, ctypes.c_size_t, vp], c_int),
        "occ_embed_sync": ([M, M, M, M, c_int, ctypes.c_float, u32, vp, vp, ctypes.c_size_t, vp], c_int),
        "occ_link_open": ([vp, c_int, c_int, i64, i64, c_int, ctypes.POINTER(vp)], c_int),
        "occ_link_close": ([vp], c_int),
        "occ_sendrecv_factors_link": ([M, M, M, M, c_int, M, M, M, u32, vp, vp, ctypes.c_size_t, vp], c_int),
        "occ_dplink_open": ([vp, i64, ctypes.POINTER(vp)], c_int),
        "occ_dplink_close": ([vp], c_int),
        "occ_dplink_allreduce": ([vp, vp, vp, i64, vp], c_int),
        "occ_allreduce_factors_link": ([c_int, ctypes.POINTER(M), ctypes.POINTER(M), ctypes.POINTER(M),
                                        ctypes.POINTER(M), ctypes.POINTER(c_int), ctypes.c_float, u32, vp, vp,
                                        ctypes.c_size_t, vp], c_int),
        "occ_get_unique_id": ([ctypes.c_char_p], c_int),
        "occ_comm_init": ([ctypes.POINTER(vp), ctypes.c_char_p, c_int, c_int], c_int),
        "occ_comm_split": ([vp, c_int, c_int, ctypes.POINTER(vp)], c_int),
        "occ_comm_wrap": ([ctypes.POINTER(vp), vp], c_int),
        "occ_comm_rank": ([vp, ctypes.POINTER(c_int), ctypes.POINTER(c_int)], c_int),
        "occ_comm_destroy": ([vp], c_int),
        "occ_check_status": ([vp, vp], c_int),
        "occ_read_stats": ([vp, ctypes.POINTER(occ_stats), vp], c_int),
        "occ_read_trace": ([vp, ctypes.POINTER(ctypes.c_uint64), c_int, vp], c_int),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def _check(status: int, where: str):
    if status != 0:
        raise OccError(status, where, lib().occ_last_error().decode())


def _stream(stream) -> int:
    import torch
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def mat(t) -> occ_mat:
    """2-D row-major view of a torch tensor (None -> null view)."""
    if t is None:
        return occ_mat(None, 0, 0, 0, OCC_F32)
    import torch
    if t.dim() != 2:
        raise ValueError("occ tensors are 2-D")
    if t.stride(1) != 1:
        raise ValueError("occ tensors must be row-major (stride(1) == 1)")
    if t.dtype == torch.float32:
        dt = OCC_F32
    elif t.dtype == torch.bfloat16:
        dt = OCC_BF16
    else:
        raise TypeError(f"unsupported dtype {t.dtype}")
    return occ_mat(t.data_ptr(), t.shape[0], t.shape[1], t.stride(0), dt)


def occ_version() -> str:
    return lib().occ_version().decode()


def occ_status_string(s: int) -> str:
    return lib().occ_status_string(s).decode()


def occ_workspace_bytes(n: int, m: int, r: int, nmat: int = 1, flags: int = 0) -> int:
    return int(lib().occ_workspace_bytes(n, m, r, nmat, flags))


def alloc_workspace(n: int, m: int, r: int, nmat: int = 1, flags: int = 0, device=None):
    """Zeroed workspace (the library keeps it zeroed between calls)."""
    import torch
    nb = occ_workspace_bytes(n, m, r, nmat, flags)
    return torch.zeros(nb, dtype=torch.uint8, device=device or "cuda")


def occ_init_q(Q, seed: int, stream=None):
    _check(lib().occ_init_q(mat(Q), seed, _stream(stream)), "occ_init_q")


def occ_compress(M, err, Q, P, recon=None, r: Optional[int] = None, flags: int = 0, ws=None, stream=None):
    r = Q.shape[1] if r is None else r
    ws = alloc_workspace(M.shape[0], M.shape[1], r, device=M.device) if ws is None else ws
    _check(lib().occ_compress(mat(M), mat(err), mat(Q), mat(P), mat(recon), r, flags,
                              ws.data_ptr(), ws.numel() * ws.element_size(), _stream(stream)),
           "occ_compress")
    return ws


def occ_decompress(P, Q, out, stream=None):
    _check(lib().occ_decompress(mat(P), mat(Q), mat(out), _stream(stream)), "occ_decompress")


def occ_allreduce_factors(G: Sequence, err: Optional[Sequence], Q: Sequence, P: Sequence, r: int,
                          scale: float, flags: int = 0, comm: Optional["Comm"] = None, ws=None, stream=None):
    n = len(G)
    arr = occ_mat * n
    g_, q_, p_ = arr(*[mat(x) for x in G]), arr(*[mat(x) for x in Q]), arr(*[mat(x) for x in P])
    e_ = arr(*[mat(x) for x in err]) if err is not None else None
    rs = (ctypes.c_int * n)(*([r] * n))
    if ws is None:
        ws = alloc_workspace(max(x.shape[0] for x in G), max(x.shape[1] for x in G), r, nmat=n,
                             device=G[0].device)
    _check(lib().occ_allreduce_factors(n, g_, e_, q_, p_, rs, scale, flags, comm.handle if comm else None,
                                       ws.data_ptr(), ws.numel(), _stream(stream)), "occ_allreduce_factors")
    return ws


def occ_allreduce_factors_link(G: Sequence, err: Optional[Sequence], Q: Sequence, P: Sequence, r: int,
                               scale: float, link: "DpLink", flags: int = 0, ws=None, stream=None):
    """occ_allreduce_factors with the two factor sums done in-kernel over the
    DP group's NVLink mailboxes (include/occ.h occ_dplink)."""
    n = len(G)
    arr = occ_mat * n
    g_, q_, p_ = arr(*[mat(x) for x in G]), arr(*[mat(x) for x in Q]), arr(*[mat(x) for x in P])
    e_ = arr(*[mat(x) for x in err]) if err is not None else None
    rs = (ctypes.c_int * n)(*([r] * n))
    if ws is None:
        ws = alloc_workspace(max(x.shape[0] for x in G), max(x.shape[1] for x in G), r, nmat=n,
                             device=G[0].device)
    _check(lib().occ_allreduce_factors_link(n, g_, e_, q_, p_, rs, scale, flags, link.handle, ws.data_ptr(),
                                            ws.numel(), _stream(stream)), "occ_allreduce_factors_link")
    return ws


def occ_send_factors(M, err, Q, P, r: int, peer: int, comm: "Comm", flags: int = 0, ws=None, stream=None):
    ws = alloc_workspace(M.shape[0], M.shape[1], r, device=M.device) if ws is None else ws
    _check(lib().occ_send_factors(mat(M), mat(err), mat(Q), mat(P), r, peer, flags, comm.handle,
                                  ws.data_ptr(), ws.numel(), _stream(stream)), "occ_send_factors")
    return ws


def occ_recv_factors(out, P, Q, r: int, peer: int, comm: "Comm", flags: int = 0, stream=None):
    _check(lib().occ_recv_factors(mat(out), mat(P), mat(Q), r, peer, flags, comm.handle, _stream(stream)),
           "occ_recv_factors")


def occ_sendrecv_factors(M, err, Q, P, r: int, send_peer: int, out, Prcv, Qrcv, recv_peer: int, comm: "Comm",
                         flags: int = 0, ws=None, stream=None):
    """PP steady state: compress M and send (P, Q) to send_peer while receiving
    recv_peer's factors and decompressing them into out (one NCCL group).
    M None: send P, Q as they are; out None: receive without decompressing."""
    if send_peer >= 0 and ws is None and M is not None:
        ws = alloc_workspace(M.shape[0], M.shape[1], r, device=M.device)
    _check(lib().occ_sendrecv_factors(mat(M) if send_peer >= 0 and M is not None else mat(None), mat(err), mat(Q),
                                      mat(P), r, send_peer,
                                      mat(out), mat(Prcv), mat(Qrcv), recv_peer, flags, comm.handle,
                                      ws.data_ptr() if ws is not None else None,
                                      ws.numel() if ws is not None else 0, _stream(stream)), "occ_sendrecv_factors")
    return ws


def occ_sendrecv_factors_link(M, err, Q, P, r: int, out, Prcv, Qrcv, link: "Link", flags: int = 0, ws=None,
                              stream=None):
    """occ_sendrecv_factors over an occ_link (NVLink peer memory, no NCCL call):
    compress M and push (P, Q) into send_peer's mailbox from the kernel, receive
    recv_peer's factors from our mailbox and decompress them into out.
    M None: push P, Q as they are; out None: receive into Prcv, Qrcv only."""
    if M is not None and ws is None:
        ws = alloc_workspace(M.shape[0], M.shape[1], r, device=M.device)
    _check(lib().occ_sendrecv_factors_link(mat(M), mat(err), mat(Q), mat(P), r, mat(out), mat(Prcv), mat(Qrcv),
                                           flags, link.handle, ws.data_ptr() if ws is not None else None,
                                           ws.numel() if ws is not None else 0, _stream(stream)),
           "occ_sendrecv_factors_link")
    return ws


def occ_embed_sync(G, err, Q, P, r: int, scale: float, comm: Optional["Comm"], flags: int = 0, ws=None,
                   stream=None):
    if r > 0 and ws is None:
        ws = alloc_workspace(G.shape[0], G.shape[1], r, device=G.device)
    _check(lib().occ_embed_sync(mat(G), mat(err), mat(Q), mat(P), r, scale, flags,
                                comm.handle if comm else None, ws.data_ptr() if ws is not None else None,
                                ws.numel() if ws is not None else 0, _stream(stream)), "occ_embed_sync")
    return ws


def occ_read_stats(ws, stream=None) -> dict:
    st = occ_stats()
    _check(lib().occ_read_stats(ws.data_ptr(), ctypes.byref(st), _stream(stream)), "occ_read_stats")
    return {"fallback_columns": st.fallback_columns, "second_pass": st.second_pass,
            "kappa_est": st.kappa_est, "path": st.path, "grid": st.grid, "t_ns": list(st.t_ns),
            "q_amp": st.q_amp, "q_fused": st.q_fused}


def occ_check_status(stream=None, comm: Optional["Comm"] = None):
    _check(lib().occ_check_status(_stream(stream), comm.handle if comm else None), "occ_check_status")


class Comm:
    """An NCCL communicator owned by libocc (occ_comm)."""

    def __init__(self, handle: int):
        self.handle = ctypes.c_void_p(handle)
        r, n = ctypes.c_int(), ctypes.c_int()
        _check(lib().occ_comm_rank(self.handle, ctypes.byref(r), ctypes.byref(n)), "occ_comm_rank")
        self.rank, self.nranks = r.value, n.value

    @classmethod
    def from_process_group(cls, group=None) -> "Comm":
        """Bootstrap: rank 0 creates the NCCL unique id, torch.distributed
        broadcasts it (any backend), every rank calls occ_comm_init."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        buf = ctypes.create_string_buffer(128)
        if rank == 0:
            _check(lib().occ_get_unique_id(buf), "occ_get_unique_id")
        obj = [bytes(buf.raw)]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group else 0, group=group)
        h = ctypes.c_void_p()
        _check(lib().occ_comm_init(ctypes.byref(h), obj[0], world, rank), "occ_comm_init")
        return cls(h.value)

    @classmethod
    def single(cls) -> "Comm":
        """A communicator of one rank (no process group needed): its NCCL
        calls still run (an allreduce copies, a send to self lands in the
        matching recv), which is how the 1-GPU tests exercise the exchange."""
        buf = ctypes.create_string_buffer(128)
        _check(lib().occ_get_unique_id(buf), "occ_get_unique_id")
        h = ctypes.c_void_p()
        _check(lib().occ_comm_init(ctypes.byref(h), bytes(buf.raw), 1, 0), "occ_comm_init")
        return cls(h.value)

    @classmethod
    def wrap(cls, nccl_comm_ptr: int) -> "Comm":
        """Adopt an existing ncclComm_t (not destroyed by destroy()), e.g. the
        communicator of a torch ProcessGroupNCCL (its private _comm_ptr())."""
        h = ctypes.c_void_p()
        _check(lib().occ_comm_wrap(ctypes.byref(h), ctypes.c_void_p(nccl_comm_ptr)), "occ_comm_wrap")
        return cls(h.value)

    def split(self, color: int, key: int) -> Optional["Comm"]:
        h = ctypes.c_void_p()
        _check(lib().occ_comm_split(self.handle, color, key, ctypes.byref(h)), "occ_comm_split")
        return Comm(h.value) if h.value else None

    def destroy(self):
        if self.handle:
            _check(lib().occ_comm_destroy(self.handle), "occ_comm_destroy")
            self.handle = None


class Link:
    """An occ_link: this stage's NVLink mailboxes towards its pipeline
    neighbours (include/occ.h).  open() is collective over the communicator."""

    def __init__(self, handle: int):
        self.handle = ctypes.c_void_p(handle)

    @classmethod
    def open(cls, comm: "Comm", send_peer: int, recv_peer: int, max_rows: int, max_cols: int, r: int) -> "Link":
        h = ctypes.c_void_p()
        _check(lib().occ_link_open(comm.handle, send_peer, recv_peer, max_rows, max_cols, r, ctypes.byref(h)),
               "occ_link_open")
        return cls(h.value)

    def close(self):
        if self.handle:
            _check(lib().occ_link_close(self.handle), "occ_link_close")
            self.handle = None


class DpLink:
    """An occ_dplink: the DP group's NVLink mailboxes for the in-kernel factor
    sums (include/occ.h).  open() is collective over the communicator."""

    def __init__(self, handle: int):
        self.handle = ctypes.c_void_p(handle)

    @classmethod
    def open(cls, comm: "Comm", max_floats: int) -> "DpLink":
        h = ctypes.c_void_p()
        _check(lib().occ_dplink_open(comm.handle, max_floats, ctypes.byref(h)), "occ_dplink_open")
        return cls(h.value)

    def allreduce(self, src, dst, stream=None):
        """dst = sum over the group of src (fp32 device tensors), in rank order."""
        _check(lib().occ_dplink_allreduce(self.handle, src.data_ptr(), dst.data_ptr(), src.numel(), _stream(stream)),
               "occ_dplink_allreduce")

    def close(self):
        if self.handle:
            _check(lib().occ_dplink_close(self.handle), "occ_dplink_close")
            self.handle = None
