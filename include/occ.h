/* occ.h -- C ABI of the B200-native Optimus-CC compression hot path.
 *
 * Optimus-CC (arXiv 2301.09830, PAPER.md) compresses three kinds of 3D-parallel
 * training traffic with PowerSGD-style rank-r low-rank approximation plus error
 * feedback (§Background, 676-677 §Impl):
 *   - the backward inter-stage activation gradient (compressed backpropagation
 *     with lazy error propagation, §CB),
 *   - data-parallel weight gradients (selective stage compression, PAPER.md:
 *     627-665 §SC, error feedback PAPER.md:657),
 *   - the tied-embedding gradient sync, fused into one allreduce over 2D ranks
 *     (§FE).
 * For each matrix M (n x m, row-major) one call performs
 *     A = M + e                (a1, lazy error / error feedback)
 *     P = A Q_prev             (a2)
 *     P_hat = orth(P)          (a4; P^T P reduced over ranks first in DP, a3)
 *     Q = A^T P_hat            (a5; summed over ranks in DP, a6)
 *     M' = round(P_hat Q^T)    (a7, M's dtype)
 *     e = A - M'               (a8)    and Q_prev <- Q  (a9, warm start).
 *
 * Conventions (every entry point):
 *  - Tensors are caller-owned DEVICE memory (torch allocations), row-major
 *    views {ptr, rows, cols, ld (elements), dtype}.  Nothing on the hot path
 *    allocates device memory; calls are asynchronous and stream ordered.
 *  - M and recon are OCC_F32 or OCC_BF16; err, P, Q are OCC_F32 always
 *    (reading C7 in DESIGN.md).  P is n x r, Q is m x r, both contiguous
 *    (ld == r).  r must be one of 4, 8, 16, 32, 64 and r <= min(n, m)
 *    (the kernels are template instances per rank; the paper's ranks are 16
 *    for CB and 128 for DP; 128 is not built: OCC_ERR_UNSUPPORTED).
 *    M.cols must be a multiple of 8 (one 8-column MMA k-step; the paper's
 *    hidden sizes 1920 / 3072 and every weight width are).
 *  - Alignment: 16-byte aligned pointers and ld*elsize % 16 == 0 (128-bit
 *    loads), else OCC_ERR_ALIGN.  M must not alias err, P or Q.
 *  - Argument errors are detected on the host before anything is enqueued;
 *    the buffers are then untouched.  Launch failures map to OCC_ERR_CUDA /
 *    OCC_ERR_NCCL.  No C++ exception crosses the ABI.  occ_last_error()
 *    returns a thread-local detail string for the last non-OK status.
 *  - Workspace: `ws` of at least occ_workspace_bytes(...) bytes of device
 *    memory, ZEROED ONCE by the caller when allocated; every call leaves it
 *    in the zeroed state it needs (its grid-barrier words are self-resetting).
 *    One workspace must not be used by two concurrently executing calls.
 *  - The library holds no state besides occ_comm handles.
 */
#ifndef OCC_H_
#define OCC_H_

#include <stddef.h>
#include <stdint.h>
#include <cuda_runtime.h>

#ifdef __cplusplus
extern "C" {
#endif

/* libocc is built with -fvisibility=hidden; only these declarations export. */
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

typedef enum {
  OCC_OK = 0,
  OCC_ERR_INVALID_ARG = 1,
  OCC_ERR_SHAPE = 2,
  OCC_ERR_DTYPE = 3,
  OCC_ERR_RANK = 4,
  OCC_ERR_ALIGN = 5,
  OCC_ERR_ALIAS = 6,
  OCC_ERR_WORKSPACE = 7,
  OCC_ERR_CUDA = 8,
  OCC_ERR_NCCL = 9,
  OCC_ERR_NONFINITE = 10,
  OCC_ERR_UNSUPPORTED = 11
} occ_status;

typedef enum { OCC_F32 = 0, OCC_BF16 = 1 } occ_dtype;

/* Row-major matrix view.  ld is the row stride in ELEMENTS. */
typedef struct {
  void* ptr;
  int64_t rows, cols, ld;
  occ_dtype dtype;
} occ_mat;

typedef struct occ_comm_s* occ_comm; /* wraps an ncclComm_t */

/* flags */
enum {
  OCC_NO_EF = 1u,          /* do not add err (Non-LEP / naive compression); err, if given, receives M - M' */
  OCC_EF_GLOBAL = 2u,      /* DP only: e_w = A_w - M' instead of the local A_w - P_hat Q_w^T (reading C2) */
  OCC_CHECK_FINITE = 4u,   /* set a device status word when M or err holds a NaN / Inf (detected on the Gram
                              diagonal, r checks per step; outputs still propagate it); occ_check_status
                              reports OCC_ERR_NONFINITE and clears it */
  OCC_WIRE_BF16 = 8u,      /* reading C7: P_hat and Q are rounded to bf16 before the reconstruction (so e_new
                              and the returned factors use the rounded values) and sent as bf16 by the
                              send / recv calls (half the bytes).  Not for occ_allreduce_factors. */
  OCC_ORIENT_T = 16u,      /* compress A^T (reading C6, the 50257-row embedding): P is m x r (orthonormal,
                              column side), Q is n x r (row side, the warm start); M, err, recon keep their
                              stored n x m layout.  Runs on the per-phase kernels (not the fused one). */
  OCC_FORCE_MULTI = 64u,   /* debug: one launch per phase instead of the fused persistent kernel */
  OCC_FORCE_TWO_PASS = 128u /* always run the second CholQR pass */
};

/* Per-call diagnostics written into the workspace (read with occ_read_stats). */
typedef struct {
  int32_t fallback_columns; /* columns replaced by their deterministic fallback vector (reading C3) */
  int32_t second_pass;      /* 1 if the second CholQR pass ran */
  double kappa_est;         /* ||L||_F * ||L^-1||_F of the first Cholesky factor (>= cond_2(P)) */
  int32_t path;             /* 1 = fused persistent kernel (v1), 2 = one launch per phase, 3 = TMEM-resident fused kernel (v2) */
  int32_t grid;             /* CTAs of the persistent kernel */
  uint64_t t_ns[12];        /* %globaltimer stamps of CTA 0 at phase boundaries (diagnostic; the v2 kernel fills them only in the OCC_TRACE build) */
  double q_amp;             /* v2: ||S Li^T||_F, the rounding amplification of the fused Q = (A^T P) Li^T; -1 if not computed */
  int32_t q_fused;          /* v2: 1 if Q was formed as (A^T P) Li^T (reading C20), 0 if as A^T P_hat */
} occ_stats;

const char* occ_status_string(occ_status s);
const char* occ_last_error(void);
const char* occ_version(void);

/* Bytes of workspace one call on an n x m matrix at rank r needs.  nmat > 1
 * sizes a DP bucket of nmat matrices of at most n x m each. */
size_t occ_workspace_bytes(int64_t n, int64_t m, int r, int nmat, uint32_t flags);

/* Q (rows x r, f32, contiguous) <- N(0,1) from a counter-based generator
 * keyed by `seed` (same seed => same Q on every rank; reading C5). */
occ_status occ_init_q(occ_mat Q, uint64_t seed, cudaStream_t stream);

/* One compression step on one GPU (the north-star path; SPEC.md:114-136
 * lowrank_compress / lazy_step).  PAPER.md:383-389 (LEP), 269-270 (PowerSGD).
 *   M      n x m, f32 or bf16, read only
 *   err    n x m f32: in e_old, out e_new = A - M'   (may be NULL ptr with OCC_NO_EF)
 *   Q      m x r f32: in Q_prev, out Q = A^T P_hat   (warm start for the next call)
 *   P      n x r f32: out P_hat (orthonormal columns)
 *   recon  n x m in M's dtype: out M' = round(P_hat Q^T), or NULL ptr to skip
 *          (err is still computed against the rounded M' the receiver would see). */
occ_status occ_compress(occ_mat M, occ_mat err, occ_mat Q, occ_mat P, occ_mat recon,
                        int r, uint32_t flags, void* ws, size_t ws_bytes, cudaStream_t stream);

/* SPEC.md:123-131 lowrank_decompress: out = round(P Q^T).  P n x r, Q m x r
 * f32; out n x m f32 or bf16. */
occ_status occ_decompress(occ_mat P, occ_mat Q, occ_mat out, cudaStream_t stream);

/* Data-parallel step over the group `dp` (§SC, 657 EF;
 * reading C1 order: allreduce-sum P before orthonormalisation, allreduce-sum
 * Q after Q_w = A_w^T P_hat; one NCCL call per factor for the whole bucket).
 * For each i < nmat: G[i] (in: local gradient; out: M' = round(P_hat (scale*sum_w Q_w)^T)),
 * err[i] (EF state), Q[i] (in: Q_prev identical on all ranks; out: scale*sum_w Q_w),
 * P[i] (out: P_hat).  All matrices share rank r[i] == r[0]. dp == NULL means a
 * group of one rank (no communication). */
occ_status occ_allreduce_factors(int nmat, const occ_mat* G, const occ_mat* err, const occ_mat* Q,
                                 const occ_mat* P, const int* r, float scale, uint32_t flags,
                                 occ_comm dp, void* ws, size_t ws_bytes, cudaStream_t stream);

/* Pipeline backward link, sender side (stage s+1 -> s): compressed
 * backpropagation of the inter-stage activation gradient (PAPER.md:351-396
 * §CB; 386-389 lazy error propagation: err keeps e_new for the link's next
 * micro-batch; 681-682 §Impl, the P2P low-rank send).  occ_compress without
 * recon, then one NCCL group of two ncclSend calls: P_hat (n x r, or m x r
 * with OCC_ORIENT_T) and Q (m x r / n x r) to `peer` of `pp`; OCC_WIRE_BF16
 * sends them as bf16 (staged in ws).  Every argument check (shapes, peer,
 * staging size) runs before anything is enqueued.  The call returns once the
 * sends are enqueued on `stream`; a matching occ_recv_factors must be posted
 * by `peer` (NCCL semantics: an unmatched send blocks the stream). */
occ_status occ_send_factors(occ_mat M, occ_mat err, occ_mat Q, occ_mat P, int r, int peer,
                            uint32_t flags, occ_comm pp, void* ws, size_t ws_bytes,
                            cudaStream_t stream);

/* Receiver side of the same link (§CB; 681-682 §Impl):
 * one NCCL group of two ncclRecv calls into P (n x r) and Q (m x r) (caller-
 * owned, overwritten; m x r / n x r with OCC_ORIENT_T) from `peer`, then
 * out = round(P_hat Q^T) in out's dtype, bit-identical to
 * the M' the sender's e_new was taken against (reading C8).  out must not
 * overlap P or Q; with OCC_WIRE_BF16 out also stages the bf16 factors. */
occ_status occ_recv_factors(occ_mat out, occ_mat P, occ_mat Q, int r, int peer, uint32_t flags,
                            occ_comm pp, cudaStream_t stream);

/* Pipeline steady state (1F1B, PAPER.md:331-337 / 386): this stage compresses
 * its backward gradient M (occ_compress without recon) and sends (P, Q) to
 * send_peer while it receives the next stage's factors into (Prcv, Qrcv) from
 * recv_peer and decompresses them into out (occ_decompress).  The sends and
 * receives form ONE NCCL group, so a ring of stages cannot deadlock.
 * send_peer / recv_peer = -1 skip that side (the pipeline ends).  Shapes as
 * occ_send_factors / occ_recv_factors (out is recv_peer's matrix shape).
 * M.ptr == NULL sends the factors already in P and Q (exchange only, e.g. to
 * time the link); out.ptr == NULL receives into Prcv / Qrcv without
 * decompressing.  Neither form takes OCC_WIRE_BF16 (OCC_ERR_UNSUPPORTED).
 * A stage may name itself as both peers (a ring of one: the NCCL send and
 * receive still run, matched inside the group). */
occ_status occ_sendrecv_factors(occ_mat M, occ_mat err, occ_mat Q, occ_mat P, int r, int send_peer,
                                occ_mat out, occ_mat Prcv, occ_mat Qrcv, int recv_peer, uint32_t flags,
                                occ_comm pp, void* ws, size_t ws_bytes, cudaStream_t stream);

/* Fused embedding synchronisation over the 2D-rank group `emb` (PAPER.md:
 * 598-618).  r == 0: one dense allreduce-sum of scale*G in place (lossless FE).
 * r > 0: occ_allreduce_factors on the group (compressed FE, reading C14). */
occ_status occ_embed_sync(occ_mat G, occ_mat err, occ_mat Q, occ_mat P, int r, float scale,
                          uint32_t flags, occ_comm emb, void* ws, size_t ws_bytes,
                          cudaStream_t stream);

/* In-kernel factor exchange over NVLink peer memory (
 * PAPER.md:681-682 §Impl, the P2P low-rank send of compressed
 * backpropagation, here without a host-issued collective).  A link is this
 * stage's pair of pipeline neighbours: it sends to send_peer and receives from
 * recv_peer (ranks of `pp`; -1: none; both may be this rank, a ring of one).
 * occ_link_open is collective over `pp`: every rank allocates a mailbox of two
 * slots of (max_rows + max_cols) x r fp32 plus flag words, exports it with
 * CUDA IPC and maps its neighbours' (handles all-gathered over `pp`).
 *   sender:   the compression kernel itself writes P_hat and Q into slot
 *             seq % 2 of send_peer's mailbox with NVLink stores (the fused
 *             kernel's producer warp does it during phase 5; other paths use
 *             a push kernel) and releases flag = seq (system scope).
 *   receiver: the decompression kernel acquires its flag >= seq, decompresses
 *             straight from the slot, copies the factors to Prcv / Qrcv, and
 *             acknowledges seq to recv_peer (which reuses the slot two steps
 *             later).
 * No NCCL call is on this path.  A wait that exceeds ~2 s (peer gone) aborts
 * the kernel's wait and occ_check_status reports OCC_ERR_NCCL. */
typedef struct occ_link_s* occ_link;
occ_status occ_link_open(occ_comm pp, int send_peer, int recv_peer, int64_t max_rows, int64_t max_cols, int r,
                         occ_link* out);
occ_status occ_link_close(occ_link link);
/* occ_sendrecv_factors over a link (same arguments and semantics, M.ptr == NULL:
 * push the factors already in P / Q; out.ptr == NULL: receive into Prcv / Qrcv
 * only).  A side whose arguments are all NULL (M and P; out and Prcv) is
 * skipped this call, so a stage can send compressed while it receives dense.
 * OCC_WIRE_BF16 is allowed: the factors are bf16-exact fp32 values. */
occ_status occ_sendrecv_factors_link(occ_mat M, occ_mat err, occ_mat Q, occ_mat P, int r, occ_mat out, occ_mat Prcv,
                                     occ_mat Qrcv, uint32_t flags, occ_link link, void* ws, size_t ws_bytes,
                                     cudaStream_t stream);

/* In-kernel factor sums of a data-parallel group over NVLink peer memory
 * (§Impl, the DP allreduce of PowerSGD's
 * P and Q; reading C1).  occ_dplink_open is collective over `dp` (at most 8
 * ranks): every rank allocates a mailbox of two slots of max_floats fp32 plus
 * flag / acknowledgement words, exports it with CUDA IPC and maps every other
 * member's (handles all-gathered over `dp`).  max_floats bounds the largest
 * bucket one call sums (the P bucket sum_i rows_i r, or the Q bucket
 * sum_i cols_i r).
 * occ_allreduce_factors_link is occ_allreduce_factors (same arguments, layout,
 * ownership and errors) with each of its two sums done by one kernel instead of
 * ncclAllReduce: a rank copies its bucket into slot seq % 2 of its own mailbox
 * and releases its flag (system scope); every rank acquires every member's
 * flag >= seq, sums the D slots in rank order (so the sum is bit-identical on
 * every rank) into its output and acknowledges; a slot is rewritten two calls
 * later, after every member's acknowledgement.  No NCCL call is on this path;
 * a wait that exceeds ~2 s (peer gone) ends the kernel's wait and
 * occ_check_status reports OCC_ERR_NCCL.  Every rank of the group must issue
 * the same sequence of calls.  OCC_ERR_WORKSPACE: a bucket larger than
 * max_floats. */
typedef struct occ_dplink_s* occ_dplink;
occ_status occ_dplink_open(occ_comm dp, int64_t max_floats, occ_dplink* out);
occ_status occ_dplink_close(occ_dplink link);
/* The exchange alone: dst[i] = sum over the group of src[i] (count <= max_floats
 * fp32, 16-byte aligned device pointers, dst may equal src), in rank order. */
occ_status occ_dplink_allreduce(occ_dplink link, const float* src, float* dst, int64_t count, cudaStream_t stream);
occ_status occ_allreduce_factors_link(int nmat, const occ_mat* G, const occ_mat* err, const occ_mat* Q, const occ_mat* P,
                                      const int* r, float scale, uint32_t flags, occ_dplink link, void* ws,
                                      size_t ws_bytes, cudaStream_t stream);

/* Communicators (NCCL over NVLink / NVSwitch). */
occ_status occ_get_unique_id(uint8_t id[128]);
occ_status occ_comm_init(occ_comm* comm, const uint8_t id[128], int nranks, int rank);
occ_status occ_comm_split(occ_comm parent, int color, int key, occ_comm* out);
/* Adopt an existing ncclComm_t (e.g. torch's ProcessGroupNCCL communicator);
 * occ_comm_destroy then frees only the handle, never the caller's communicator. */
occ_status occ_comm_wrap(occ_comm* comm, void* nccl_comm);
occ_status occ_comm_rank(occ_comm comm, int* rank, int* nranks);
occ_status occ_comm_destroy(occ_comm comm);

/* Synchronises `stream`, then reports the first pending CUDA error, the
 * asynchronous NCCL error of `comm` (may be NULL: SURVEY.md §8(b) lists
 * occ_check_status(stream); the communicator argument is needed because NCCL
 * reports asynchronous errors per communicator), and OCC_ERR_NONFINITE. */
occ_status occ_check_status(cudaStream_t stream, occ_comm comm);

/* Copies the diagnostics of the last call that used `ws` (synchronises). */
occ_status occ_read_stats(const void* ws, occ_stats* out, cudaStream_t stream);

/* Debug (libocc_trace.so, built with -DOCC_TRACE; the product library leaves
 * the trace zero): per-CTA phase trace of the last fused (v2) call on ws: out[cta*48 + k],
 * k < 24 clock64 at phase boundaries, k >= 24 the matching %globaltimer (ns).
 * Copies min(count, 160*48) words (synchronises). */
occ_status occ_read_trace(const void* ws, uint64_t* out, int count, cudaStream_t stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif
#endif /* OCC_H_ */
