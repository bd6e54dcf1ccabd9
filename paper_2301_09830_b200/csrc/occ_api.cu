// occ_api.cu -- the extern "C" boundary (include/occ.h): argument validation,
// workspace carving, orchestration of the step phases and the NCCL exchanges.
#include "occ.h"
#include "occ_kernels.cuh"
#include "occ_internal.h"

#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

using namespace occ;

struct occ_comm_s {
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;
  bool owned = true;   // false for occ_comm_wrap: the caller's communicator is not destroyed
  // occ_embed_sync's PreMulSum op (scale * G summed), created once per (dtype, scale)
  bool has_premul = false;
  ncclRedOp_t premul_op{};
  ncclDataType_t premul_dt{};
  float premul_scale = 0.f;
};

namespace {

thread_local std::string g_err;

// NVTX range per API call (header-only NVTX 3: a no-op unless a profiler
// injects itself), so nsys / ncu timelines show which call launched what.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

occ_status fail(occ_status s, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
occ_status fail(occ_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

occ_status cuda_fail(cudaError_t e, const char* what) {
  return fail(OCC_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

constexpr int kGeomSms = 148;              // geometry is device independent (B200 SM count)
constexpr double kTau = 1e-5;              // reading C3
constexpr double kKappaTwoPass = 1e4;      // CholQR2 trigger on ||L||_F ||L^-1||_F (fused kernel)
// The per-phase path forms P_hat = P Li^T from an fp64 Gram of the fp32 P, so
// the first pass's loss of orthogonality is ~ kappa^2 u_64 (<= 1e-8 at 1e4,
// 1e-4 at the worst kappa_est 1e6 only if kappa_est is tight; it overestimates
// kappa by up to sqrt(r)) next to the fp32 rounding of P_hat itself, which no
// second pass removes: CholQR2 runs there only above 1e6 (reading C3)
constexpr double kKappaTwoPassPhase = 1e6;
constexpr unsigned long long kFbSeed = 0;  // fallback-vector seed (oracle default)

size_t esize(occ_dtype d) { return d == OCC_BF16 ? 2 : 4; }

bool rank_supported(int r) { return r == 4 || r == 8 || r == 16 || r == 32 || r == 64; }

struct Span { uintptr_t lo, hi; };
Span span_of(const occ_mat& a) {
  if (!a.ptr || a.rows <= 0) return {0, 0};
  uintptr_t lo = reinterpret_cast<uintptr_t>(a.ptr);
  return {lo, lo + (uintptr_t)((a.rows - 1) * a.ld + a.cols) * esize(a.dtype)};
}
bool overlap(const occ_mat& a, const occ_mat& b) {
  Span x = span_of(a), y = span_of(b);
  if (x.lo == x.hi || y.lo == y.hi) return false;
  return x.lo < y.hi && y.lo < x.hi;
}

occ_status check_view(const occ_mat& a, const char* name, int64_t rows, int64_t cols, bool f32_only,
                      bool contiguous) {
  if (!a.ptr) return fail(OCC_ERR_INVALID_ARG, "%s: null pointer", name);
  if (a.dtype != OCC_F32 && a.dtype != OCC_BF16) return fail(OCC_ERR_DTYPE, "%s: unknown dtype %d", name, (int)a.dtype);
  if (f32_only && a.dtype != OCC_F32) return fail(OCC_ERR_DTYPE, "%s: must be OCC_F32", name);
  if (a.rows != rows || a.cols != cols)
    return fail(OCC_ERR_SHAPE, "%s: shape %lldx%lld, expected %lldx%lld", name, (long long)a.rows,
                (long long)a.cols, (long long)rows, (long long)cols);
  if (a.ld < a.cols) return fail(OCC_ERR_SHAPE, "%s: ld %lld < cols %lld", name, (long long)a.ld, (long long)a.cols);
  if (contiguous && a.ld != a.cols) return fail(OCC_ERR_SHAPE, "%s: must be contiguous (ld == cols)", name);
  if ((reinterpret_cast<uintptr_t>(a.ptr) & 15) != 0) return fail(OCC_ERR_ALIGN, "%s: pointer not 16-byte aligned", name);
  if ((a.ld * (int64_t)esize(a.dtype)) % 16 != 0) return fail(OCC_ERR_ALIGN, "%s: ld*elsize not a multiple of 16", name);
  return OCC_OK;
}

occ_status check_rank(int r, int64_t n, int64_t m) {
  if (r < 1 || r > std::min(n, m)) return fail(OCC_ERR_RANK, "rank %d outside [1, min(n,m)=%lld]", r, (long long)std::min(n, m));
  if (!rank_supported(r)) return fail(OCC_ERR_UNSUPPORTED, "rank %d not built (supported: 4, 8, 16, 32, 64)", r);
  return OCC_OK;
}

// Validates one (M, err, Q, P, recon) set for the compression step.
occ_status check_step(const occ_mat& M, const occ_mat& err, const occ_mat& Q, const occ_mat& P,
                      const occ_mat* recon, int r, uint32_t flags) {
  if (!M.ptr) return fail(OCC_ERR_INVALID_ARG, "M: null pointer");
  if (M.rows < 1 || M.cols < 1) return fail(OCC_ERR_SHAPE, "M: empty matrix %lldx%lld", (long long)M.rows, (long long)M.cols);
  occ_status s = check_rank(r, M.rows, M.cols);
  if (s) return s;
  if ((s = check_view(M, "M", M.rows, M.cols, false, false))) return s;
  if (M.cols % 8 != 0) return fail(OCC_ERR_SHAPE, "M: cols %lld must be a multiple of 8", (long long)M.cols);
  const bool need_err = !(flags & OCC_NO_EF);
  if (need_err || err.ptr) {
    if ((s = check_view(err, "err", M.rows, M.cols, true, false))) return s;
  }
  const bool ot = (flags & OCC_ORIENT_T) != 0;   // P on the column side, Q on the row side
  if ((s = check_view(Q, "Q", ot ? M.rows : M.cols, r, true, true))) return s;
  if ((s = check_view(P, "P", ot ? M.cols : M.rows, r, true, true))) return s;
  if (recon && recon->ptr) {
    if ((s = check_view(*recon, "recon", M.rows, M.cols, false, false))) return s;
    if (recon->dtype != M.dtype) return fail(OCC_ERR_DTYPE, "recon: dtype must equal M's");
  }
  const occ_mat* bufs[] = {&err, &Q, &P};
  const char* names[] = {"err", "Q", "P"};
  for (int x = 0; x < 3; x++)
    if (overlap(M, *bufs[x]))
      return fail(OCC_ERR_ALIAS, "M aliases %s", names[x]);
  for (int x = 0; x < 3; x++)
    for (int y = x + 1; y < 3; y++)
      if (overlap(*bufs[x], *bufs[y])) return fail(OCC_ERR_ALIAS, "%s aliases %s", names[x], names[y]);
  if (recon && recon->ptr) {
    for (int x = 0; x < 3; x++)
      if (overlap(*recon, *bufs[x])) return fail(OCC_ERR_ALIAS, "recon aliases %s", names[x]);
    if (overlap(*recon, M) && (recon->ptr != M.ptr || recon->ld != M.ld))
      return fail(OCC_ERR_ALIAS, "recon partially aliases M");
  }
  return OCC_OK;
}

Params base_params(const occ_mat& M, const occ_mat& err, const occ_mat& Q, const occ_mat& P, uint32_t flags) {
  Params p;
  memset(&p, 0, sizeof p);
  p.M = M.ptr;
  p.ldm = M.ld;
  p.m_bf16 = M.dtype == OCC_BF16;
  p.err_in = (flags & OCC_NO_EF) ? nullptr : static_cast<const float*>(err.ptr);
  p.lde_in = err.ld;
  p.err_out = static_cast<float*>(err.ptr);
  p.lde_out = err.ld;
  p.r_bf16 = M.dtype == OCC_BF16;
  p.n = (int)M.rows;
  p.m = (int)M.cols;
  p.Qprev = static_cast<const float*>(Q.ptr);
  p.P = static_cast<float*>(P.ptr);
  p.Qloc = static_cast<float*>(Q.ptr);
  p.Qrec = static_cast<const float*>(Q.ptr);
  p.Qstate_out = nullptr;
  p.scale = 1.0f;
  p.fb_seed = kFbSeed;
  p.tau = kTau;
  p.kappa_thr = kKappaTwoPass;
  p.kappa_thr_phase = kKappaTwoPassPhase;
  static const double kphase_env = [] {   // experiment knob (tools/kappa_ab.py)
    const char* e = getenv("OCC_KAPPA_PHASE");
    return e ? atof(e) : 0.0;
  }();
  if (kphase_env > 0.0) p.kappa_thr_phase = kphase_env;
  p.force_two_pass = (flags & OCC_FORCE_TWO_PASS) ? 1 : 0;
  p.check_finite = (flags & OCC_CHECK_FINITE) ? 1 : 0;
  p.wire_bf16 = (flags & OCC_WIRE_BF16) ? 1 : 0;
  return p;
}

bool want_multi(uint32_t flags) {
  if (flags & OCC_FORCE_MULTI) return true;
  const char* e = getenv("OCC_FORCE_MULTI");
  return e && e[0] == '1';
}

bool want_v1() {
  const char* e = getenv("OCC_PATH");
  return e && e[0] == 'v' && e[1] == '1';
}

occ_status nccl_fail(ncclResult_t r, const char* what) {
  return fail(OCC_ERR_NCCL, "%s: %s", what, ncclGetErrorString(r));
}

// Inside an NCCL group: the first failing ncclSend / ncclRecv is kept in *first
// (the group is still closed by the caller, which then reports it).
void nccl_keep(ncclResult_t r, ncclResult_t* first) {
  if (r != ncclSuccess && *first == ncclSuccess) *first = r;
}

// Closes a group and reports the first error of its calls, or of the close.
occ_status group_end(ncclResult_t first, const char* what) {
  const ncclResult_t e = ncclGroupEnd();
  if (first != ncclSuccess) return nccl_fail(first, what);
  if (e != ncclSuccess) return nccl_fail(e, what);
  return OCC_OK;
}

// Phase ranges of run_phases (occ_step.cu PhaseId): [0,2) = sweep 1 + P reduce,
// [2,6) = Gram + orthonormalisation, [6,8) = sweep 2 + Q reduce, [8,9) = reconstruct.
constexpr int kPhA = 0, kPhOrth = 2, kPhD = 6, kPhF = 8, kPhEnd = 9;

// phase F of a per-phase occ_compress (M' and e_new): the v2 decompress
// arithmetic for every supported rank (r = 4..64), so occ_decompress
// reproduces the sender's M' bit for bit (C8) whichever path compressed; v1
// phase F only under OCC_PATH=v1, where occ_decompress is v1 as well.
cudaError_t reconstruct(const Params& p, const Geometry& g, int r, bool multi, cudaStream_t st) {
  if (!want_v1()) {
    cudaError_t e = run_v2_reconstruct(p, r, st);
    if (e != cudaErrorNotSupported) return e;
  }
  return run_phases(p, g, kPhF, kPhEnd, multi, false, st);
}

// Orthonormalise the column-side factor U (m x R, in place) with the per-phase
// kernels: the Gram phases run with the factor length m (OCC_ORIENT_T).
cudaError_t orth_column_factor(const Params& base, float* U, int64_t m, int64_t n, int R, const WsLayout& L,
                               void* ws, bool multi, cudaStream_t st) {
  Params p2 = base;
  p2.n = (int)m;
  p2.m = (int)n;
  p2.P = U;
  Geometry gT = make_geometry(m, n, R, kGeomSms);
  fill_ws(p2, gT, L, ws);
  return run_phases(p2, gT, kPhOrth, kPhD, multi, false, st);
}

// OCC_WIRE_BF16 send side: the (already bf16-exact) factors packed into the
// workspace's factor buckets, then sent as bf16.  Queues the ncclSends (inside
// the caller's group).
// OCC_WIRE_BF16 staging space check of the send side (before anything is enqueued).
occ_status check_send_stage_bf16(int64_t prows, int64_t qrows, int r, size_t ws_bytes, int64_t n, int64_t m) {
  const WsLayout L = make_layout(make_geometry(n, m, r, kGeomSms), 1);
  const size_t need = 2 * ((size_t)prows + (size_t)qrows) * r;
  if (L.qs_bucket - L.p_bucket < need || ws_bytes < L.total) return fail(OCC_ERR_WORKSPACE, "bf16 staging");
  return OCC_OK;
}

// Packs the (already bf16-exact) factors (stream ordered, before the group).
occ_status pack_factors_bf16(const occ_mat& P, const occ_mat& Q, int r, void* ws, int64_t n, int64_t m,
                             cudaStream_t st) {
  const WsLayout L = make_layout(make_geometry(n, m, r, kGeomSms), 1);
  char* stage = static_cast<char*>(ws) + L.p_bucket;
  cudaError_t e = run_pack_bf16(static_cast<const float*>(P.ptr), stage, (long long)P.rows * r, st);
  if (e == cudaSuccess) e = run_pack_bf16(static_cast<const float*>(Q.ptr), stage + 2 * (size_t)P.rows * r, (long long)Q.rows * r, st);
  return e == cudaSuccess ? OCC_OK : cuda_fail(e, "bf16 pack");
}

// Queues the bf16 sends of the packed factors (inside the caller's group).
void send_factors_bf16(const occ_mat& P, const occ_mat& Q, int r, int peer, occ_comm pp, void* ws, int64_t n,
                       int64_t m, cudaStream_t st, ncclResult_t* first) {
  const WsLayout L = make_layout(make_geometry(n, m, r, kGeomSms), 1);
  char* stage = static_cast<char*>(ws) + L.p_bucket;
  nccl_keep(ncclSend(stage, (size_t)P.rows * r, ncclBfloat16, peer, pp->comm, st), first);
  nccl_keep(ncclSend(stage + 2 * (size_t)P.rows * r, (size_t)Q.rows * r, ncclBfloat16, peer, pp->comm, st), first);
}

// OCC_WIRE_BF16 receive side: bf16 factors land in `out` (not yet written), are
// expanded into Prcv / Qrcv, and `out` is then overwritten by the decompression.
occ_status check_recv_stage_bf16(const occ_mat& out, const occ_mat& Prcv, const occ_mat& Qrcv, int r) {
  const size_t need = 2 * ((size_t)Prcv.rows + (size_t)Qrcv.rows) * r;
  const size_t have = (size_t)out.rows * out.ld * (out.dtype == OCC_BF16 ? 2 : 4);
  if (have < need) return fail(OCC_ERR_UNSUPPORTED, "OCC_WIRE_BF16: out too small to stage the factors");
  return OCC_OK;
}
void recv_factors_bf16(const occ_mat& out, const occ_mat& Prcv, const occ_mat& Qrcv, int r, int peer, occ_comm pp,
                       cudaStream_t st, ncclResult_t* first) {
  char* stage = static_cast<char*>(out.ptr);
  nccl_keep(ncclRecv(stage, (size_t)Prcv.rows * r, ncclBfloat16, peer, pp->comm, st), first);
  nccl_keep(ncclRecv(stage + 2 * (size_t)Prcv.rows * r, (size_t)Qrcv.rows * r, ncclBfloat16, peer, pp->comm, st), first);
}

// Receiver-side checks (before anything is enqueued): the output view, the
// factor shapes, aliasing between out and the factors (and, for the ring, the
// sender's buffers), and the bf16 staging size.
occ_status check_recv_side(const occ_mat& out, const occ_mat& Prcv, const occ_mat& Qrcv, int r, uint32_t flags,
                           const occ_mat* snd_bufs, int nsnd) {
  if (!out.ptr) return fail(OCC_ERR_INVALID_ARG, "out: null pointer");
  occ_status s = check_rank(r, out.rows, out.cols);
  if (s) return s;
  if ((s = check_view(out, "out", out.rows, out.cols, false, false))) return s;
  if (out.cols % 8 != 0) return fail(OCC_ERR_SHAPE, "out: cols must be a multiple of 8");
  const bool ot = (flags & OCC_ORIENT_T) != 0;   // P m x r, Q n x r; out = Q P^T
  if ((s = check_view(Prcv, "P", ot ? out.cols : out.rows, r, true, true))) return s;
  if ((s = check_view(Qrcv, "Q", ot ? out.rows : out.cols, r, true, true))) return s;
  if (overlap(out, Prcv) || overlap(out, Qrcv) || overlap(Prcv, Qrcv))
    return fail(OCC_ERR_ALIAS, "out and the received factors must not overlap");
  for (int i = 0; i < nsnd; i++)
    if (overlap(snd_bufs[i], out) || overlap(snd_bufs[i], Prcv) || overlap(snd_bufs[i], Qrcv))
      return fail(OCC_ERR_ALIAS, "receive buffers alias the sender's M / err / Q / P");
  if ((flags & OCC_WIRE_BF16) && (s = check_recv_stage_bf16(out, Prcv, Qrcv, r))) return s;
  return OCC_OK;
}
occ_status unpack_factors_bf16(const occ_mat& out, const occ_mat& Prcv, const occ_mat& Qrcv, int r, cudaStream_t st) {
  const char* stage = static_cast<const char*>(out.ptr);
  cudaError_t e = run_unpack_bf16(stage, static_cast<float*>(Prcv.ptr), (long long)Prcv.rows * r, st);
  if (e == cudaSuccess)
    e = run_unpack_bf16(stage + 2 * (size_t)Prcv.rows * r, static_cast<float*>(Qrcv.ptr), (long long)Qrcv.rows * r, st);
  return e == cudaSuccess ? OCC_OK : cuda_fail(e, "bf16 unpack");
}

}  // namespace

static occ_status compress_impl(occ_mat M, occ_mat err, occ_mat Q, occ_mat P, occ_mat recon, int r, uint32_t flags,
                                void* ws, size_t ws_bytes, cudaStream_t stream, const LinkPush* push, bool* pushed);

extern "C" {

const char* occ_status_string(occ_status s) {
  switch (s) {
    case OCC_OK: return "OCC_OK";
    case OCC_ERR_INVALID_ARG: return "OCC_ERR_INVALID_ARG";
    case OCC_ERR_SHAPE: return "OCC_ERR_SHAPE";
    case OCC_ERR_DTYPE: return "OCC_ERR_DTYPE";
    case OCC_ERR_RANK: return "OCC_ERR_RANK";
    case OCC_ERR_ALIGN: return "OCC_ERR_ALIGN";
    case OCC_ERR_ALIAS: return "OCC_ERR_ALIAS";
    case OCC_ERR_WORKSPACE: return "OCC_ERR_WORKSPACE";
    case OCC_ERR_CUDA: return "OCC_ERR_CUDA";
    case OCC_ERR_NCCL: return "OCC_ERR_NCCL";
    case OCC_ERR_NONFINITE: return "OCC_ERR_NONFINITE";
    case OCC_ERR_UNSUPPORTED: return "OCC_ERR_UNSUPPORTED";
  }
  return "OCC_ERR_UNKNOWN";
}

const char* occ_last_error(void) { return g_err.c_str(); }

const char* occ_version(void) { return "occ 0.1 (sm_100a)"; }

size_t occ_workspace_bytes(int64_t n, int64_t m, int r, int nmat, uint32_t flags) {
  (void)flags;
  if (n < 1 || m < 1 || r < 1 || nmat < 1) return 0;
  Geometry g = make_geometry(n, m, r, kGeomSms);
  return make_layout(g, nmat).total;
}

occ_status occ_init_q(occ_mat Q, uint64_t seed, cudaStream_t stream) {
  occ_status s = check_view(Q, "Q", Q.rows, Q.cols, true, false);
  if (s) return s;
  if (Q.rows < 1 || Q.cols < 1) return fail(OCC_ERR_SHAPE, "Q: empty");
  cudaError_t e = run_init_q(static_cast<float*>(Q.ptr), Q.rows, (int)Q.cols, Q.ld, seed, stream);
  return e == cudaSuccess ? OCC_OK : cuda_fail(e, "occ_init_q launch");
}

occ_status occ_compress(occ_mat M, occ_mat err, occ_mat Q, occ_mat P, occ_mat recon, int r, uint32_t flags,
                        void* ws, size_t ws_bytes, cudaStream_t stream) {
  NvtxRange nvtx_("occ_compress");
  return compress_impl(M, err, Q, P, recon, r, flags, ws, ws_bytes, stream, nullptr, nullptr);
}

}  // extern "C"

// occ_compress; with `push` (occ_link sender) the fused kernel also pushes the
// factors to the peer's mailbox (*pushed = true) -- the other paths leave it to
// the caller (*pushed = false).
static occ_status compress_impl(occ_mat M, occ_mat err, occ_mat Q, occ_mat P, occ_mat recon, int r, uint32_t flags,
                                void* ws, size_t ws_bytes, cudaStream_t stream, const LinkPush* push, bool* pushed) {
  if (pushed) *pushed = false;
  occ_status s = check_step(M, err, Q, P, &recon, r, flags);
  if (s) return s;
  Geometry g = make_geometry(M.rows, M.cols, r, kGeomSms);
  WsLayout L = make_layout(g, 1);
  if (!ws || ws_bytes < L.total)
    return fail(OCC_ERR_WORKSPACE, "workspace %zu bytes < required %zu", ws_bytes, L.total);
  if (reinterpret_cast<uintptr_t>(ws) & 255) return fail(OCC_ERR_ALIGN, "workspace not 256-byte aligned");
  Params p = base_params(M, err, Q, P, flags);
  p.recon = recon.ptr;
  p.ldr = recon.ptr ? recon.ld : 0;
  fill_ws(p, g, L, ws);
  const bool multi = want_multi(flags);
  if (flags & OCC_ORIENT_T) {
    // the step on A^T in A's layout (reading C6): U = A^T Q_prev (sweep 2 with the
    // row-side warm start), U_hat = orth(U) into P, V = A U_hat (sweep 1) into Q
    // (the next warm start), M' = V U_hat^T, e_new = A - M'
    float* Pp = static_cast<float*>(P.ptr);
    float* Qp = static_cast<float*>(Q.ptr);
    Params p1 = p;
    p1.P = Qp;
    p1.Qloc = Pp;
    cudaError_t e = run_phases(p1, g, kPhD, kPhF, multi, false, stream);
    if (e == cudaSuccess) e = orth_column_factor(p, Pp, M.cols, M.rows, r, L, ws, multi, stream);
    if (e == cudaSuccess) {
      Params p3 = p;
      p3.Qprev = Pp;
      p3.P = Qp;
      e = run_phases(p3, g, kPhA, kPhOrth, multi, false, stream);
    }
    if (e == cudaSuccess && p.wire_bf16) e = run_round_bf16(Pp, M.cols * (long long)r, stream);
    if (e == cudaSuccess && p.wire_bf16) e = run_round_bf16(Qp, M.rows * (long long)r, stream);
    if (e == cudaSuccess) {
      Params p4 = p;
      p4.P = Qp;
      p4.Qrec = Pp;
      e = reconstruct(p4, g, r, multi, stream);
    }
    return e == cudaSuccess ? OCC_OK : cuda_fail(e, "occ_compress (OCC_ORIENT_T) launch");
  }
  if (!multi && !want_v1() && L.v2_tail_bytes > 0) {
    if (push) p.push = *push;
    cudaError_t e2 = run_v2(p, r, static_cast<char*>(ws) + L.v2_tail, L.v2_tail_bytes, kGeomSms, stream);
    if (e2 == cudaSuccess) {
      if (pushed) *pushed = push != nullptr;
      return OCC_OK;
    }
    p.push = LinkPush{};
    if (e2 != cudaErrorNotSupported) return cuda_fail(e2, "occ_compress (fused v2) launch");
  }
  cudaError_t e;
  e = run_phases(p, g, kPhA, kPhF, multi, false, stream);
  if (p.wire_bf16) {   // reading C7: the reconstruction uses the bf16-rounded factors
    if (e == cudaSuccess) e = run_round_bf16(p.P, M.rows * (long long)r, stream);
    if (e == cudaSuccess) e = run_round_bf16(p.Qloc, M.cols * (long long)r, stream);
  }
  if (e == cudaSuccess) e = reconstruct(p, g, r, multi, stream);
  return e == cudaSuccess ? OCC_OK : cuda_fail(e, "occ_compress launch");
}

extern "C" {

occ_status occ_decompress(occ_mat P, occ_mat Q, occ_mat out, cudaStream_t stream) {
  NvtxRange nvtx_("occ_decompress");
  if (!out.ptr) return fail(OCC_ERR_INVALID_ARG, "out: null pointer");
  const int r = (int)P.cols;
  occ_status s = check_rank(r, out.rows, out.cols);
  if (s) return s;
  if ((s = check_view(out, "out", out.rows, out.cols, false, false))) return s;
  if (out.cols % 8 != 0) return fail(OCC_ERR_SHAPE, "out: cols must be a multiple of 8");
  if ((s = check_view(P, "P", out.rows, r, true, true))) return s;
  if ((s = check_view(Q, "Q", out.cols, r, true, true))) return s;
  if (overlap(out, P) || overlap(out, Q)) return fail(OCC_ERR_ALIAS, "out aliases a factor");
  Params p;
  memset(&p, 0, sizeof p);
  p.n = (int)out.rows;
  p.m = (int)out.cols;
  p.P = static_cast<float*>(P.ptr);
  p.Qrec = static_cast<const float*>(Q.ptr);
  p.scale = 1.0f;
  p.recon = out.ptr;
  p.ldr = out.ld;
  p.r_bf16 = out.dtype == OCC_BF16;
  cudaError_t e = want_v1() ? cudaErrorNotSupported
                            : run_v2_decompress(p.P, p.Qrec, p.recon, p.ldr, p.n, p.m, r, p.r_bf16 != 0, stream);
  if (e == cudaErrorNotSupported) e = run_decompress(p, r, stream);   // OCC_PATH=v1
  return e == cudaSuccess ? OCC_OK : cuda_fail(e, "occ_decompress launch");
}

}  // extern "C"

// ------------------------------------------------------------------ occ_dplink (f1, DP)
// Mailbox of one rank: two slots of D sub-slots of cap fp32 (sub-slot q is
// written by member q), then the words: +4 q flag from member q (its sub-slot
// of sequence seq is complete), +64 + 4 q ack from member q (q has summed its
// slot of sequence seq, so ours may be rewritten), +1024 / +1088 the local
// CTA-exit counters.  Every rank maps every member's mailbox with CUDA IPC.
struct occ_dplink_s {
  occ_comm dp = nullptr;
  int D = 1, rank = 0;
  size_t cap = 0, words_off = 0;
  char* local = nullptr;
  char* base[kDplinkMax] = {};
  bool ipc[kDplinkMax] = {};
  unsigned seq = 0;
};

static cudaError_t run_dplink_allreduce(occ_dplink L, const float* src, float* dst, size_t count, cudaStream_t st) {
  DplinkArgs a{};
  a.D = L->D;
  a.rank = L->rank;
  a.seq = ++L->seq;
  a.cap = (long long)L->cap;
  a.words_off = (long long)L->words_off;
  for (int q = 0; q < L->D; q++) a.base[q] = L->base[q];
  a.src = src;
  a.dst = dst;
  a.count = (long long)count;
  return run_dplink_kernel(a, st);
}

static occ_status allreduce_factors_impl(int nmat, const occ_mat* G, const occ_mat* err, const occ_mat* Q,
                                         const occ_mat* P, const int* r, float scale, uint32_t flags, occ_comm dp,
                                         occ_dplink dl, void* ws, size_t ws_bytes, cudaStream_t stream);

extern "C" {

occ_status occ_allreduce_factors(int nmat, const occ_mat* G, const occ_mat* err, const occ_mat* Q, const occ_mat* P,
                                 const int* r, float scale, uint32_t flags, occ_comm dp, void* ws, size_t ws_bytes,
                                 cudaStream_t stream) {
  NvtxRange nvtx_("occ_allreduce_factors");
  return allreduce_factors_impl(nmat, G, err, Q, P, r, scale, flags, dp, nullptr, ws, ws_bytes, stream);
}

}  // extern "C"

// The DP step (occ_allreduce_factors / occ_allreduce_factors_link): the factor
// sums run over NCCL (dp) or in-kernel over NVLink peer memory (dl).
static occ_status allreduce_factors_impl(int nmat, const occ_mat* G, const occ_mat* err, const occ_mat* Q,
                                         const occ_mat* P, const int* r, float scale, uint32_t flags, occ_comm dp,
                                         occ_dplink dl, void* ws, size_t ws_bytes, cudaStream_t stream) {
  if (nmat < 1 || !G || !Q || !P || !r) return fail(OCC_ERR_INVALID_ARG, "null array or nmat < 1");
  if (!(flags & OCC_NO_EF) && !err) return fail(OCC_ERR_INVALID_ARG, "err array required unless OCC_NO_EF");
  if (flags & OCC_WIRE_BF16) return fail(OCC_ERR_UNSUPPORTED, "OCC_WIRE_BF16 applies to the send / recv calls");
  const int R = r[0];
  int64_t nmax = 0, mmax = 0;
  for (int i = 0; i < nmat; i++) {
    if (r[i] != R) return fail(OCC_ERR_RANK, "all matrices of a bucket must share one rank");
    occ_mat e = err ? err[i] : occ_mat{nullptr, 0, 0, 0, OCC_F32};
    occ_status s = check_step(G[i], e, Q[i], P[i], nullptr, R, flags);
    if (s) return fail(s, "matrix %d: %s", i, g_err.c_str());
    nmax = std::max<int64_t>(nmax, G[i].rows);
    mmax = std::max<int64_t>(mmax, G[i].cols);
  }
  Geometry gmax = make_geometry(nmax, mmax, R, kGeomSms);
  WsLayout L = make_layout(gmax, nmat);
  if (!ws || ws_bytes < L.total)
    return fail(OCC_ERR_WORKSPACE, "workspace %zu bytes < required %zu", ws_bytes, L.total);
  if (reinterpret_cast<uintptr_t>(ws) & 255) return fail(OCC_ERR_ALIGN, "workspace not 256-byte aligned");
  const bool multi = want_multi(flags);
  const bool dpl = !(flags & OCC_EF_GLOBAL);
  const bool comm = dp != nullptr || dl != nullptr;   // a 1-rank group still runs its exchange (tested on 1 GPU)
  // sum over the group: NCCL, or the in-kernel exchange over the dplink
  auto allreduce = [&](const float* src, float* dst, size_t count, const char* what) -> occ_status {
    if (dl) {
      if (count > dl->cap) return fail(OCC_ERR_WORKSPACE, "%s: %zu floats > dplink capacity %zu", what, count, dl->cap);
      cudaError_t e = run_dplink_allreduce(dl, src, dst, count, stream);
      return e == cudaSuccess ? OCC_OK : cuda_fail(e, what);
    }
    ncclResult_t nr = ncclAllReduce(src, dst, count, ncclFloat, ncclSum, dp->comm, stream);
    return nr == ncclSuccess ? OCC_OK : nccl_fail(nr, what);
  };
  char* base = static_cast<char*>(ws);
  float* pb = reinterpret_cast<float*>(base + L.p_bucket);
  float* qwb = reinterpret_cast<float*>(base + L.qw_bucket);
  float* qsb = reinterpret_cast<float*>(base + L.qs_bucket);
  size_t poff[64], qoff[64];
  if (nmat > 64) return fail(OCC_ERR_INVALID_ARG, "at most 64 matrices per bucket");
  size_t ptot = 0, qtot = 0;
  for (int i = 0; i < nmat; i++) {
    poff[i] = ptot; ptot += (size_t)G[i].rows * R;
    qoff[i] = qtot; qtot += (size_t)G[i].cols * R;
  }
  if (dl && std::max(ptot, qtot) > dl->cap)   // before anything is enqueued (occ.h conventions)
    return fail(OCC_ERR_WORKSPACE, "factor bucket of %zu floats > dplink capacity %zu", std::max(ptot, qtot), dl->cap);
  auto params_for = [&](int i) {
    occ_mat e = err ? err[i] : occ_mat{nullptr, 0, 0, 0, OCC_F32};
    Params p = base_params(G[i], e, Q[i], P[i], flags);
    Geometry g = make_geometry(G[i].rows, G[i].cols, R, kGeomSms);
    fill_ws(p, g, L, ws);
    return std::make_pair(p, g);
  };
  if (flags & OCC_ORIENT_T) {
    // DP step on A_w^T (reading C6), in A's layout: U_w = A_w^T V_prev (column
    // side) -> allreduce-sum U -> U_hat = orth(U) into P -> V_w = A_w U_hat (row
    // side) -> allreduce-sum V -> M' = (scale V_sum) U_hat^T, e_w = A_w - V_w U_hat^T
    // (local, reading C2) or A_w - M'; Q <- scale V_sum (the warm start).
    for (int i = 0; i < nmat; i++) {
      auto [p, g] = params_for(i);
      p.P = static_cast<float*>(Q[i].ptr);
      p.Qloc = qwb + qoff[i];
      cudaError_t e = run_phases(p, g, kPhD, kPhF, multi, false, stream);
      if (e != cudaSuccess) return cuda_fail(e, "dp (ORIENT_T) sweep launch");
    }
    if (comm) {
      if (occ_status sa = allreduce(qwb, qwb, qtot, "allreduce(U)")) return sa;
    }
    for (int i = 0; i < nmat; i++) {
      auto [p, g] = params_for(i);
      float* Up = static_cast<float*>(P[i].ptr);
      cudaError_t e = cudaMemcpyAsync(Up, qwb + qoff[i], (size_t)G[i].cols * R * 4, cudaMemcpyDeviceToDevice, stream);
      if (e != cudaSuccess) return cuda_fail(e, "U copy");
      e = orth_column_factor(p, Up, G[i].cols, G[i].rows, R, L, ws, multi, stream);
      if (e != cudaSuccess) return cuda_fail(e, "dp (ORIENT_T) orthonormalise launch");
      p.Qprev = Up;
      p.P = pb + poff[i];
      e = run_phases(p, g, kPhA, kPhOrth, multi, false, stream);
      if (e != cudaSuccess) return cuda_fail(e, "dp (ORIENT_T) sweep launch");
    }
    float* vsum = pb;
    if (comm) {
      if (occ_status sa = allreduce(pb, qsb, ptot, "allreduce(V)")) return sa;
      vsum = qsb;
    }
    for (int i = 0; i < nmat; i++) {
      auto [p, g] = params_for(i);
      p.P = vsum + poff[i];
      p.Qrec = static_cast<const float*>(P[i].ptr);
      p.Ploc = dpl ? pb + poff[i] : nullptr;
      p.Pstate_out = static_cast<float*>(Q[i].ptr);
      p.scale = scale;
      p.dp_local_err = dpl ? 1 : 0;
      p.recon = G[i].ptr;
      p.ldr = G[i].ld;
      p.f_tc = 1;
      cudaError_t e = run_phases(p, g, kPhF, kPhEnd, multi, dpl, stream);
      if (e != cudaSuccess) return cuda_fail(e, "dp (ORIENT_T) reconstruct launch");
    }
    return OCC_OK;
  }
  // (a1-a2) sweep 1 + P reduce for every matrix into the P bucket
  for (int i = 0; i < nmat; i++) {
    auto [p, g] = params_for(i);
    p.P = pb + poff[i];
    cudaError_t e = run_phases(p, g, 0, 2, multi, dpl, stream);
    if (e != cudaSuccess) return cuda_fail(e, "dp sweep1 launch");
  }
  // (a3) allreduce-sum P over the DP group (reading C1)
  if (comm) {
    if (occ_status sa = allreduce(pb, pb, ptot, "allreduce(P)")) return sa;
  }
  // (a4-a5) Gram + orthonormalise + sweep 2 + Q reduce into the Q_w bucket
  for (int i = 0; i < nmat; i++) {
    auto [p, g] = params_for(i);
    cudaError_t e = cudaMemcpyAsync(P[i].ptr, pb + poff[i], (size_t)G[i].rows * R * 4, cudaMemcpyDeviceToDevice, stream);
    if (e != cudaSuccess) return cuda_fail(e, "P copy");
    p.Qloc = qwb + qoff[i];
    e = run_phases(p, g, 2, 8, multi, dpl, stream);
    if (e != cudaSuccess) return cuda_fail(e, "dp sweep2 launch");
  }
  // (a6) allreduce-sum Q
  float* qsum = qwb;
  if (comm) {
    if (occ_status sa = allreduce(qwb, qsb, qtot, "allreduce(Q)")) return sa;
    qsum = qsb;
  }
  // (a7-a9) M' = round(P_hat (scale sum Q)^T) over G, residual, warm start
  for (int i = 0; i < nmat; i++) {
    auto [p, g] = params_for(i);
    p.Qloc = qwb + qoff[i];
    p.Qrec = qsum + qoff[i];
    p.scale = scale;
    p.Qstate_out = static_cast<float*>(Q[i].ptr);
    p.dp_local_err = dpl ? 1 : 0;
    p.recon = G[i].ptr;
    p.ldr = G[i].ld;
    p.f_tc = 1;
    cudaError_t e = run_phases(p, g, 8, 9, multi, dpl, stream);
    if (e != cudaSuccess) return cuda_fail(e, "dp reconstruct launch");
  }
  return OCC_OK;
}

extern "C" {

occ_status occ_send_factors(occ_mat M, occ_mat err, occ_mat Q, occ_mat P, int r, int peer, uint32_t flags,
                            occ_comm pp, void* ws, size_t ws_bytes, cudaStream_t stream) {
  NvtxRange nvtx_("occ_send_factors");
  if (!pp) return fail(OCC_ERR_INVALID_ARG, "pp communicator is null");
  if (peer < 0 || peer >= pp->nranks || peer == pp->rank) return fail(OCC_ERR_INVALID_ARG, "bad peer %d", peer);
  occ_mat none = {nullptr, 0, 0, 0, M.dtype};
  occ_status s = check_step(M, err, Q, P, nullptr, r, flags);
  if (s) return s;
  if ((flags & OCC_WIRE_BF16) && (s = check_send_stage_bf16(P.rows, Q.rows, r, ws_bytes, M.rows, M.cols))) return s;
  if ((s = occ_compress(M, err, Q, P, none, r, flags, ws, ws_bytes, stream))) return s;
  if ((flags & OCC_WIRE_BF16) && (s = pack_factors_bf16(P, Q, r, ws, M.rows, M.cols, stream))) return s;
  ncclResult_t nr, first = ncclSuccess;
  if ((nr = ncclGroupStart()) != ncclSuccess) return nccl_fail(nr, "ncclGroupStart");
  if (flags & OCC_WIRE_BF16) {
    send_factors_bf16(P, Q, r, peer, pp, ws, M.rows, M.cols, stream, &first);
  } else {
    nccl_keep(ncclSend(P.ptr, (size_t)P.rows * r, ncclFloat, peer, pp->comm, stream), &first);   // (OCC_ORIENT_T: P is m x r)
    nccl_keep(ncclSend(Q.ptr, (size_t)Q.rows * r, ncclFloat, peer, pp->comm, stream), &first);
  }
  return group_end(first, "ncclSend(P,Q)");
}

occ_status occ_recv_factors(occ_mat out, occ_mat P, occ_mat Q, int r, int peer, uint32_t flags, occ_comm pp,
                            cudaStream_t stream) {
  NvtxRange nvtx_("occ_recv_factors");
  if (!pp) return fail(OCC_ERR_INVALID_ARG, "pp communicator is null");
  if (peer < 0 || peer >= pp->nranks || peer == pp->rank) return fail(OCC_ERR_INVALID_ARG, "bad peer %d", peer);
  if ((int)P.cols != r) return fail(OCC_ERR_SHAPE, "P: cols must equal r");
  occ_status s = check_recv_side(out, P, Q, r, flags, nullptr, 0);
  if (s) return s;
  const bool ot = (flags & OCC_ORIENT_T) != 0;   // P m x r, Q n x r; out = Q P^T
  const bool wire = (flags & OCC_WIRE_BF16) != 0;
  ncclResult_t nr, first = ncclSuccess;
  if ((nr = ncclGroupStart()) != ncclSuccess) return nccl_fail(nr, "ncclGroupStart");
  if (wire) {
    recv_factors_bf16(out, P, Q, r, peer, pp, stream, &first);
  } else {
    nccl_keep(ncclRecv(P.ptr, (size_t)P.rows * r, ncclFloat, peer, pp->comm, stream), &first);
    nccl_keep(ncclRecv(Q.ptr, (size_t)Q.rows * r, ncclFloat, peer, pp->comm, stream), &first);
  }
  if ((s = group_end(first, "ncclRecv(P,Q)"))) return s;
  if (wire && (s = unpack_factors_bf16(out, P, Q, r, stream))) return s;
  return ot ? occ_decompress(Q, P, out, stream) : occ_decompress(P, Q, out, stream);
}

occ_status occ_sendrecv_factors(occ_mat M, occ_mat err, occ_mat Q, occ_mat P, int r, int send_peer, occ_mat out,
                                occ_mat Prcv, occ_mat Qrcv, int recv_peer, uint32_t flags, occ_comm pp, void* ws,
                                size_t ws_bytes, cudaStream_t stream) {
  NvtxRange nvtx_("occ_sendrecv_factors");
  if (!pp) return fail(OCC_ERR_INVALID_ARG, "pp communicator is null");
  const bool snd = send_peer >= 0, rcv = recv_peer >= 0;
  // a stage may be its own peer only when it both sends and receives in this
  // one group (a ring of one stage, e.g. a 1-GPU check of the NCCL exchange)
  const bool self_ok = snd && rcv && send_peer == pp->rank && recv_peer == pp->rank;
  if (snd && (send_peer >= pp->nranks || (send_peer == pp->rank && !self_ok)))
    return fail(OCC_ERR_INVALID_ARG, "bad send_peer %d", send_peer);
  if (rcv && (recv_peer >= pp->nranks || (recv_peer == pp->rank && !self_ok)))
    return fail(OCC_ERR_INVALID_ARG, "bad recv_peer %d", recv_peer);
  const bool wire = (flags & OCC_WIRE_BF16) != 0;
  // M.ptr == NULL: P and Q already hold the factors to send (exchange only);
  // out.ptr == NULL: receive the factors only (no decompression)
  const bool compress = snd && M.ptr != nullptr, decompress = rcv && out.ptr != nullptr;
  if ((!compress && snd && wire) || (!decompress && rcv && wire))
    return fail(OCC_ERR_UNSUPPORTED, "OCC_WIRE_BF16 needs M and out (the bf16 staging lives in ws / out)");
  // every argument check before anything is enqueued (occ.h conventions)
  occ_status s;
  if (compress) {
    if ((s = check_step(M, err, Q, P, nullptr, r, flags))) return s;
    if (wire && (s = check_send_stage_bf16(P.rows, Q.rows, r, ws_bytes, M.rows, M.cols))) return s;
  } else if (snd) {
    if ((s = check_rank(r, P.rows, Q.rows))) return s;
    if ((s = check_view(P, "P", P.rows, r, true, true))) return s;
    if ((s = check_view(Q, "Q", Q.rows, r, true, true))) return s;
  }
  if (decompress) {
    const occ_mat sb[4] = {M, err, Q, P};
    if ((s = check_recv_side(out, Prcv, Qrcv, r, flags, sb, snd ? 4 : 0))) return s;
  } else if (rcv) {
    if ((s = check_view(Prcv, "Prcv", Prcv.rows, r, true, true))) return s;
    if ((s = check_view(Qrcv, "Qrcv", Qrcv.rows, r, true, true))) return s;
    if (overlap(Prcv, Qrcv) || (snd && (overlap(Prcv, P) || overlap(Prcv, Q) || overlap(Qrcv, P) || overlap(Qrcv, Q))))
      return fail(OCC_ERR_ALIAS, "receive buffers overlap");
  }
  if (compress) {
    occ_mat none = {nullptr, 0, 0, 0, M.dtype};
    if ((s = occ_compress(M, err, Q, P, none, r, flags, ws, ws_bytes, stream))) return s;
    if (wire && (s = pack_factors_bf16(P, Q, r, ws, M.rows, M.cols, stream))) return s;
  }
  ncclResult_t nr, first = ncclSuccess;
  if ((nr = ncclGroupStart()) != ncclSuccess) return nccl_fail(nr, "ncclGroupStart");
  if (snd) {
    if (wire) {
      send_factors_bf16(P, Q, r, send_peer, pp, ws, M.rows, M.cols, stream, &first);
    } else {
      nccl_keep(ncclSend(P.ptr, (size_t)P.rows * r, ncclFloat, send_peer, pp->comm, stream), &first);
      nccl_keep(ncclSend(Q.ptr, (size_t)Q.rows * r, ncclFloat, send_peer, pp->comm, stream), &first);
    }
  }
  if (rcv) {
    if (wire) {
      recv_factors_bf16(out, Prcv, Qrcv, r, recv_peer, pp, stream, &first);
    } else {
      nccl_keep(ncclRecv(Prcv.ptr, (size_t)Prcv.rows * r, ncclFloat, recv_peer, pp->comm, stream), &first);
      nccl_keep(ncclRecv(Qrcv.ptr, (size_t)Qrcv.rows * r, ncclFloat, recv_peer, pp->comm, stream), &first);
    }
  }
  if ((s = group_end(first, "ncclSendRecv(P,Q)"))) return s;
  if (!decompress) return OCC_OK;
  if (wire && (s = unpack_factors_bf16(out, Prcv, Qrcv, r, stream))) return s;
  const bool ot = (flags & OCC_ORIENT_T) != 0;
  return ot ? occ_decompress(Qrcv, Prcv, out, stream) : occ_decompress(Prcv, Qrcv, out, stream);
}

occ_status occ_embed_sync(occ_mat G, occ_mat err, occ_mat Q, occ_mat P, int r, float scale, uint32_t flags,
                          occ_comm emb, void* ws, size_t ws_bytes, cudaStream_t stream) {
  NvtxRange nvtx_("occ_embed_sync");
  if (r > 0) return occ_allreduce_factors(1, &G, &err, &Q, &P, &r, scale, flags, emb, ws, ws_bytes, stream);
  occ_status s = check_view(G, "G", G.rows, G.cols, false, true);
  if (s) return s;
  if (!emb) {   // no group: the identity when scale == 1 (a group of one rank)
    if (scale == 1.0f) return OCC_OK;
    return fail(OCC_ERR_INVALID_ARG, "emb communicator is null");
  }
  ncclDataType_t dt = G.dtype == OCC_BF16 ? ncclBfloat16 : ncclFloat;
  const size_t count = (size_t)G.rows * G.cols;
  ncclResult_t nr;
  // one PreMulSum op per communicator, re-created only when the dtype or the
  // scale changes (the FE scale 1/D is fixed for a run, reading C12)
  if (!emb->has_premul || emb->premul_dt != dt || emb->premul_scale != scale) {
    if (emb->has_premul) {
      ncclRedOpDestroy(emb->premul_op, emb->comm);
      emb->has_premul = false;
    }
    if (G.dtype == OCC_BF16) {
      __nv_bfloat16 sb = __float2bfloat16_rn(scale);   // the scalar's type must match the data type
      nr = ncclRedOpCreatePreMulSum(&emb->premul_op, &sb, dt, ncclScalarHostImmediate, emb->comm);
    } else {
      nr = ncclRedOpCreatePreMulSum(&emb->premul_op, &scale, dt, ncclScalarHostImmediate, emb->comm);
    }
    if (nr != ncclSuccess) return nccl_fail(nr, "ncclRedOpCreatePreMulSum");
    emb->has_premul = true;
    emb->premul_dt = dt;
    emb->premul_scale = scale;
  }
  nr = ncclAllReduce(G.ptr, G.ptr, count, dt, emb->premul_op, emb->comm, stream);
  if (nr != ncclSuccess) return nccl_fail(nr, "ncclAllReduce(EMB)");
  return OCC_OK;
}

occ_status occ_get_unique_id(uint8_t id[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId u;
  ncclResult_t nr = ncclGetUniqueId(&u);
  if (nr != ncclSuccess) return nccl_fail(nr, "ncclGetUniqueId");
  memcpy(id, &u, 128);
  return OCC_OK;
}

occ_status occ_comm_init(occ_comm* comm, const uint8_t id[128], int nranks, int rank) {
  if (!comm || !id || nranks < 1 || rank < 0 || rank >= nranks) return fail(OCC_ERR_INVALID_ARG, "bad comm_init args");
  ncclUniqueId u;
  memcpy(&u, id, 128);
  occ_comm c = new occ_comm_s;
  ncclResult_t nr = ncclCommInitRank(&c->comm, nranks, u, rank);
  if (nr != ncclSuccess) { delete c; return nccl_fail(nr, "ncclCommInitRank"); }
  c->rank = rank;
  c->nranks = nranks;
  *comm = c;
  return OCC_OK;
}

occ_status occ_comm_split(occ_comm parent, int color, int key, occ_comm* out) {
  if (!parent || !out) return fail(OCC_ERR_INVALID_ARG, "bad comm_split args");
  occ_comm c = new occ_comm_s;
  ncclResult_t nr = ncclCommSplit(parent->comm, color, key, &c->comm, nullptr);
  if (nr != ncclSuccess) { delete c; return nccl_fail(nr, "ncclCommSplit"); }
  if (!c->comm) { delete c; *out = nullptr; return OCC_OK; }  // color == NCCL_SPLIT_NOCOLOR
  ncclCommUserRank(c->comm, &c->rank);
  ncclCommCount(c->comm, &c->nranks);
  *out = c;
  return OCC_OK;
}

occ_status occ_comm_rank(occ_comm comm, int* rank, int* nranks) {
  if (!comm) return fail(OCC_ERR_INVALID_ARG, "null comm");
  if (rank) *rank = comm->rank;
  if (nranks) *nranks = comm->nranks;
  return OCC_OK;
}

occ_status occ_comm_wrap(occ_comm* comm, void* nccl_comm) {
  if (!comm || !nccl_comm) return fail(OCC_ERR_INVALID_ARG, "bad comm_wrap args");
  occ_comm c = new occ_comm_s;
  c->comm = static_cast<ncclComm_t>(nccl_comm);
  c->owned = false;
  ncclResult_t nr = ncclCommUserRank(c->comm, &c->rank);
  if (nr == ncclSuccess) nr = ncclCommCount(c->comm, &c->nranks);
  if (nr != ncclSuccess) { delete c; return nccl_fail(nr, "occ_comm_wrap"); }
  *comm = c;
  return OCC_OK;
}

occ_status occ_comm_destroy(occ_comm comm) {
  if (!comm) return OCC_OK;
  if (comm->has_premul) ncclRedOpDestroy(comm->premul_op, comm->comm);
  ncclResult_t nr = comm->owned ? ncclCommDestroy(comm->comm) : ncclSuccess;
  delete comm;
  return nr == ncclSuccess ? OCC_OK : nccl_fail(nr, "ncclCommDestroy");
}

occ_status occ_check_status(cudaStream_t stream, occ_comm comm) {
  cudaError_t e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) return cuda_fail(e, "stream");
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "last error");
  if (comm) {
    ncclResult_t ar;
    ncclResult_t nr = ncclCommGetAsyncError(comm->comm, &ar);
    if (nr != ncclSuccess) return nccl_fail(nr, "ncclCommGetAsyncError");
    if (ar != ncclSuccess) return nccl_fail(ar, "nccl async");
  }
  if (take_link_timeout()) return fail(OCC_ERR_NCCL, "occ_link: a wait for the peer timed out (peer gone?)");
  const unsigned nf = take_nonfinite_v1() | take_nonfinite_v2();
  if (nf) return fail(OCC_ERR_NONFINITE, "non-finite M or err in a call made with OCC_CHECK_FINITE");
  return OCC_OK;
}

occ_status occ_read_stats(const void* ws, occ_stats* out, cudaStream_t stream) {
  if (!ws || !out) return fail(OCC_ERR_INVALID_ARG, "null ws/out");
  DevStats d;
  cudaError_t e = cudaMemcpyAsync(&d, static_cast<const char*>(ws) + 64, sizeof d, cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) return cuda_fail(e, "occ_read_stats");
  out->fallback_columns = d.fallback_columns;
  out->second_pass = d.second_pass;
  out->kappa_est = d.kappa_est;
  out->path = d.path;
  out->grid = d.grid;
  for (int k = 0; k < 12; k++) out->t_ns[k] = d.t_ns[k];
  out->q_amp = d.q_amp;
  out->q_fused = d.q_fused;
  return OCC_OK;
}

}  // extern "C"

extern "C" occ_status occ_read_trace(const void* ws, uint64_t* out, int count, cudaStream_t stream) {
  if (!ws || !out || count < 0) return fail(OCC_ERR_INVALID_ARG, "null ws/out");
  const size_t words = std::min<size_t>((size_t)count, kTraceBytes / 8);
  cudaError_t e = cudaMemcpyAsync(out, static_cast<const char*>(ws) + kTraceOffset, words * 8, cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  return e == cudaSuccess ? OCC_OK : cuda_fail(e, "occ_read_trace");
}

// ------------------------------------------------------------------ occ_link (f1)
// Mailbox of one rank: two slots of (max_rows + max_cols) x r fp32, then the
// words at words_off: +0 flag (released by the rank that sends to us), +64 ack
// (released by the rank we send to), +128 / +192 our push / receive CTA-exit
// counters.  The neighbours' mailboxes are mapped with CUDA IPC.
struct occ_link_s {
  occ_comm pp = nullptr;
  int send_peer = -1, recv_peer = -1, r = 0;
  int64_t cap_rows = 0;        // max_rows + max_cols: P rows + Q rows of one message
  size_t slot_bytes = 0, words_off = 0;
  char* local = nullptr;
  char* send_base = nullptr;   // send_peer's mailbox
  char* recv_base = nullptr;   // recv_peer's mailbox
  bool send_ipc = false, recv_ipc = false;
  unsigned send_seq = 0, recv_seq = 0;
};

namespace {
constexpr size_t kLinkFlag = 0, kLinkAck = 64, kLinkPushCtr = 128, kLinkRecvCtr = 192;
unsigned* link_word(char* base, const occ_link_s* L, size_t off) {
  return reinterpret_cast<unsigned*>(base + L->words_off + off);
}
}  // namespace

extern "C" occ_status occ_link_open(occ_comm pp, int send_peer, int recv_peer, int64_t max_rows, int64_t max_cols,
                                    int r, occ_link* out) {
  NvtxRange nvtx_("occ_link_open");
  if (!pp || !out) return fail(OCC_ERR_INVALID_ARG, "null communicator or output");
  if (send_peer >= pp->nranks || recv_peer >= pp->nranks || send_peer < -1 || recv_peer < -1)
    return fail(OCC_ERR_INVALID_ARG, "bad peer (send %d, recv %d, nranks %d)", send_peer, recv_peer, pp->nranks);
  if (max_rows < 1 || max_cols < 1 || r < 1) return fail(OCC_ERR_SHAPE, "bad link capacity");
  occ_link L = new occ_link_s;
  L->pp = pp;
  L->send_peer = send_peer;
  L->recv_peer = recv_peer;
  L->r = r;
  L->cap_rows = max_rows + max_cols;
  L->slot_bytes = ((size_t)L->cap_rows * r * 4 + 255) / 256 * 256;
  L->words_off = 2 * L->slot_bytes;
  const size_t bytes = L->words_off + 256;
  auto bail = [&](occ_status st) {
    if (L->send_ipc) cudaIpcCloseMemHandle(L->send_base);
    if (L->recv_ipc && L->recv_base != L->send_base) cudaIpcCloseMemHandle(L->recv_base);
    if (L->local) cudaFree(L->local);
    delete L;
    return st;
  };
  cudaError_t e = cudaMalloc(&L->local, bytes);
  if (e == cudaSuccess) e = cudaMemset(L->local, 0, bytes);
  if (e != cudaSuccess) return bail(cuda_fail(e, "link mailbox"));
  // all-gather the IPC handles over the communicator
  cudaIpcMemHandle_t h;
  e = cudaIpcGetMemHandle(&h, L->local);
  if (e != cudaSuccess) return bail(cuda_fail(e, "cudaIpcGetMemHandle"));
  const int n = pp->nranks;
  char* dbuf = nullptr;
  e = cudaMalloc(&dbuf, (size_t)(n + 1) * sizeof h);
  if (e == cudaSuccess) e = cudaMemcpy(dbuf + (size_t)n * sizeof h, &h, sizeof h, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    if (dbuf) cudaFree(dbuf);
    return bail(cuda_fail(e, "link handle exchange"));
  }
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  ncclResult_t nr = ncclAllGather(dbuf + (size_t)n * sizeof h, dbuf, sizeof h, ncclUint8, pp->comm, st);
  e = cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  std::string hb((size_t)n * sizeof h, '\0');
  if (nr == ncclSuccess && e == cudaSuccess) e = cudaMemcpy(&hb[0], dbuf, hb.size(), cudaMemcpyDeviceToHost);
  cudaFree(dbuf);
  if (nr != ncclSuccess) return bail(nccl_fail(nr, "ncclAllGather(link handles)"));
  if (e != cudaSuccess) return bail(cuda_fail(e, "link handle exchange"));
  auto open_peer = [&](int peer, char** base, bool* ipc) -> occ_status {
    if (peer < 0) return OCC_OK;
    if (peer == pp->rank) { *base = L->local; return OCC_OK; }
    cudaIpcMemHandle_t ph;
    memcpy(&ph, hb.data() + (size_t)peer * sizeof ph, sizeof ph);
    cudaError_t e2 = cudaIpcOpenMemHandle(reinterpret_cast<void**>(base), ph, cudaIpcMemLazyEnablePeerAccess);
    if (e2 != cudaSuccess) return cuda_fail(e2, "cudaIpcOpenMemHandle");
    *ipc = true;
    return OCC_OK;
  };
  occ_status s = open_peer(send_peer, &L->send_base, &L->send_ipc);
  if (s) return bail(s);
  if (recv_peer >= 0 && recv_peer == send_peer) {
    L->recv_base = L->send_base;   // one mapping serves both directions
  } else if ((s = open_peer(recv_peer, &L->recv_base, &L->recv_ipc))) {
    return bail(s);
  }
  *out = L;
  return OCC_OK;
}

extern "C" occ_status occ_link_close(occ_link L) {
  if (!L) return OCC_OK;
  cudaError_t e = cudaDeviceSynchronize();
  if (L->send_ipc) cudaIpcCloseMemHandle(L->send_base);
  if (L->recv_ipc && L->recv_base != L->send_base) cudaIpcCloseMemHandle(L->recv_base);
  cudaFree(L->local);
  delete L;
  return e == cudaSuccess ? OCC_OK : cuda_fail(e, "occ_link_close");
}

extern "C" occ_status occ_dplink_open(occ_comm dp, int64_t max_floats, occ_dplink* out) {
  NvtxRange nvtx_("occ_dplink_open");
  if (!dp || !out) return fail(OCC_ERR_INVALID_ARG, "null communicator or output");
  if (dp->nranks > kDplinkMax) return fail(OCC_ERR_UNSUPPORTED, "dplink: at most %d ranks", kDplinkMax);
  if (max_floats < 1) return fail(OCC_ERR_SHAPE, "bad dplink capacity");
  occ_dplink L = new occ_dplink_s;
  L->dp = dp;
  L->D = dp->nranks;
  L->rank = dp->rank;
  L->cap = ((size_t)max_floats + 63) / 64 * 64;
  L->words_off = 2 * (size_t)L->D * L->cap * 4;
  const size_t bytes = L->words_off + 2048;
  auto bail = [&](occ_status st) {
    for (int q = 0; q < L->D; q++)
      if (L->ipc[q]) cudaIpcCloseMemHandle(L->base[q]);
    if (L->local) cudaFree(L->local);
    delete L;
    return st;
  };
  cudaError_t e = cudaMalloc(&L->local, bytes);
  if (e == cudaSuccess) e = cudaMemset(L->local, 0, bytes);
  if (e != cudaSuccess) return bail(cuda_fail(e, "dplink mailbox"));
  cudaIpcMemHandle_t h;
  e = cudaIpcGetMemHandle(&h, L->local);
  if (e != cudaSuccess) return bail(cuda_fail(e, "cudaIpcGetMemHandle"));
  const int n = L->D;
  char* dbuf = nullptr;
  e = cudaMalloc(&dbuf, (size_t)(n + 1) * sizeof h);
  if (e == cudaSuccess) e = cudaMemcpy(dbuf + (size_t)n * sizeof h, &h, sizeof h, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    if (dbuf) cudaFree(dbuf);
    return bail(cuda_fail(e, "dplink handle exchange"));
  }
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  ncclResult_t nr = ncclAllGather(dbuf + (size_t)n * sizeof h, dbuf, sizeof h, ncclUint8, dp->comm, st);
  e = cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  std::string hb((size_t)n * sizeof h, '\0');
  if (nr == ncclSuccess && e == cudaSuccess) e = cudaMemcpy(&hb[0], dbuf, hb.size(), cudaMemcpyDeviceToHost);
  cudaFree(dbuf);
  if (nr != ncclSuccess) return bail(nccl_fail(nr, "ncclAllGather(dplink handles)"));
  if (e != cudaSuccess) return bail(cuda_fail(e, "dplink handle exchange"));
  for (int q = 0; q < n; q++) {
    if (q == L->rank) { L->base[q] = L->local; continue; }
    cudaIpcMemHandle_t ph;
    memcpy(&ph, hb.data() + (size_t)q * sizeof ph, sizeof ph);
    cudaError_t e2 = cudaIpcOpenMemHandle(reinterpret_cast<void**>(&L->base[q]), ph, cudaIpcMemLazyEnablePeerAccess);
    if (e2 != cudaSuccess) return bail(cuda_fail(e2, "cudaIpcOpenMemHandle (dplink)"));
    L->ipc[q] = true;
  }
  *out = L;
  return OCC_OK;
}

extern "C" occ_status occ_dplink_close(occ_dplink L) {
  if (!L) return OCC_OK;
  cudaError_t e = cudaDeviceSynchronize();
  for (int q = 0; q < L->D; q++)
    if (L->ipc[q]) cudaIpcCloseMemHandle(L->base[q]);
  cudaFree(L->local);
  delete L;
  return e == cudaSuccess ? OCC_OK : cuda_fail(e, "occ_dplink_close");
}

extern "C" occ_status occ_dplink_allreduce(occ_dplink link, const float* src, float* dst, int64_t count,
                                           cudaStream_t stream) {
  NvtxRange nvtx_("occ_dplink_allreduce");
  if (!link || !src || !dst) return fail(OCC_ERR_INVALID_ARG, "null dplink or buffer");
  if (count < 0 || (size_t)count > link->cap) return fail(OCC_ERR_WORKSPACE, "count %lld outside the dplink capacity %zu",
                                                         (long long)count, link->cap);
  if ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15)
    return fail(OCC_ERR_ALIGN, "src / dst not 16-byte aligned");
  const cudaError_t e = run_dplink_allreduce(link, src, dst, (size_t)count, stream);
  return e == cudaSuccess ? OCC_OK : cuda_fail(e, "occ_dplink_allreduce");
}

extern "C" occ_status occ_allreduce_factors_link(int nmat, const occ_mat* G, const occ_mat* err, const occ_mat* Q,
                                                 const occ_mat* P, const int* r, float scale, uint32_t flags,
                                                 occ_dplink link, void* ws, size_t ws_bytes, cudaStream_t stream) {
  NvtxRange nvtx_("occ_allreduce_factors_link");
  if (!link) return fail(OCC_ERR_INVALID_ARG, "null dplink");
  return allreduce_factors_impl(nmat, G, err, Q, P, r, scale, flags, nullptr, link, ws, ws_bytes, stream);
}

extern "C" occ_status occ_sendrecv_factors_link(occ_mat M, occ_mat err, occ_mat Q, occ_mat P, int r, occ_mat out,
                                                occ_mat Prcv, occ_mat Qrcv, uint32_t flags, occ_link L, void* ws,
                                                size_t ws_bytes, cudaStream_t stream) {
  NvtxRange nvtx_("occ_sendrecv_factors_link");
  if (!L) return fail(OCC_ERR_INVALID_ARG, "link is null");
  if (r != L->r) return fail(OCC_ERR_RANK, "rank %d differs from the link's %d", r, L->r);
  // a side whose arguments are all null is skipped this call (e.g. a pipeline
  // stage whose send is compressed but whose receive is dense this micro-batch)
  const bool snd = L->send_peer >= 0 && (M.ptr || P.ptr);
  const bool rcv = L->recv_peer >= 0 && (out.ptr || Prcv.ptr);
  const bool compress = snd && M.ptr != nullptr, decompress = rcv && out.ptr != nullptr;
  const bool ot = (flags & OCC_ORIENT_T) != 0;
  occ_status s;
  // every argument check before anything is enqueued
  if (compress) {
    if ((s = check_step(M, err, Q, P, nullptr, r, flags))) return s;
  } else if (snd) {
    if ((s = check_rank(r, P.rows, Q.rows))) return s;
    if ((s = check_view(P, "P", P.rows, r, true, true))) return s;
    if ((s = check_view(Q, "Q", Q.rows, r, true, true))) return s;
  }
  if (snd && P.rows + Q.rows > L->cap_rows)
    return fail(OCC_ERR_SHAPE, "factors of %lld + %lld rows exceed the link's %lld", (long long)P.rows,
                (long long)Q.rows, (long long)L->cap_rows);
  if (decompress) {
    const occ_mat sb[4] = {M, err, Q, P};
    if ((s = check_recv_side(out, Prcv, Qrcv, r, flags & ~(uint32_t)OCC_WIRE_BF16, sb, snd ? 4 : 0))) return s;
  } else if (rcv) {
    if ((s = check_view(Prcv, "Prcv", Prcv.rows, r, true, true))) return s;
    if ((s = check_view(Qrcv, "Qrcv", Qrcv.rows, r, true, true))) return s;
    if (overlap(Prcv, Qrcv)) return fail(OCC_ERR_ALIAS, "Prcv and Qrcv overlap");
  }
  if (rcv && Prcv.rows + Qrcv.rows > L->cap_rows) return fail(OCC_ERR_SHAPE, "received factors exceed the link");
  cudaError_t e = cudaSuccess;
  if (snd && rcv && !compress && !decompress) {   // exchange only, both directions: one launch
    const unsigned sseq = ++L->send_seq, rseq = ++L->recv_seq;
    float* pP = reinterpret_cast<float*>(L->send_base + (sseq & 1u) * L->slot_bytes);
    float* mP = reinterpret_cast<float*>(L->local + (rseq & 1u) * L->slot_bytes);
    e = run_link_exchange(static_cast<const float*>(P.ptr), static_cast<const float*>(Q.ptr), pP, pP + (size_t)P.rows * r,
                          (long long)P.rows * r, (long long)Q.rows * r, link_word(L->local, L, kLinkAck),
                          link_word(L->local, L, kLinkPushCtr), link_word(L->send_base, L, kLinkFlag), sseq, mP,
                          mP + (size_t)Prcv.rows * r, static_cast<float*>(Prcv.ptr), static_cast<float*>(Qrcv.ptr),
                          (long long)Prcv.rows * r, (long long)Qrcv.rows * r, link_word(L->local, L, kLinkFlag),
                          link_word(L->local, L, kLinkRecvCtr), link_word(L->recv_base, L, kLinkAck), rseq, stream);
    return e == cudaSuccess ? OCC_OK : cuda_fail(e, "link exchange");
  }
  if (snd) {
    const unsigned seq = ++L->send_seq;
    LinkPush push;
    push.P = reinterpret_cast<float*>(L->send_base + (seq & 1u) * L->slot_bytes);
    push.Q = push.P + (size_t)P.rows * r;
    push.flag = link_word(L->send_base, L, kLinkFlag);
    push.ack = link_word(L->local, L, kLinkAck);
    push.ctr = link_word(L->local, L, kLinkPushCtr);
    push.seq = seq;
    bool pushed = false;
    if (compress) {
      occ_mat none = {nullptr, 0, 0, 0, M.dtype};
      if ((s = compress_impl(M, err, Q, P, none, r, flags, ws, ws_bytes, stream, &push, &pushed))) return s;
    }
    if (!pushed)
      e = run_link_copy(static_cast<const float*>(P.ptr), static_cast<const float*>(Q.ptr), push.P, push.Q,
                        (long long)P.rows * r, (long long)Q.rows * r, seq > 2 ? push.ack : nullptr, seq - 2,
                        push.ctr, push.flag, seq, stream);
    if (e != cudaSuccess) return cuda_fail(e, "link push");
  }
  if (rcv) {
    const unsigned seq = ++L->recv_seq;
    float* Pm = reinterpret_cast<float*>(L->local + (seq & 1u) * L->slot_bytes);
    float* Qm = Pm + (size_t)Prcv.rows * r;
    LinkRecv lr;
    lr.wait_flag = link_word(L->local, L, kLinkFlag);
    lr.seq = seq;
    lr.ack = link_word(L->recv_base, L, kLinkAck);
    lr.ctr = link_word(L->local, L, kLinkRecvCtr);
    if (decompress) {
      // the kernel's P operand is the row-side factor: P_hat, or Q with OCC_ORIENT_T (out = Q P^T)
      const float* kP = ot ? Qm : Pm;
      const float* kQ = ot ? Pm : Qm;
      lr.copyP = static_cast<float*>(ot ? Qrcv.ptr : Prcv.ptr);
      lr.copyQ = static_cast<float*>(ot ? Prcv.ptr : Qrcv.ptr);
      lr.nP = (long long)(ot ? Qrcv.rows : Prcv.rows) * r;
      lr.nQ = (long long)(ot ? Prcv.rows : Qrcv.rows) * r;
      e = run_v2_decompress_link(kP, kQ, out.ptr, out.ld, (int)out.rows, (int)out.cols, r, out.dtype == OCC_BF16, lr,
                                 stream);
    } else {
      e = run_link_copy(Pm, Qm, static_cast<float*>(Prcv.ptr), static_cast<float*>(Qrcv.ptr),
                        (long long)Prcv.rows * r, (long long)Qrcv.rows * r, lr.wait_flag, seq, lr.ctr, lr.ack, seq,
                        stream);
    }
    if (e != cudaSuccess) return cuda_fail(e, "link receive");
  }
  return OCC_OK;
}
