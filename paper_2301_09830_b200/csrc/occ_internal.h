// occ_internal.h -- declarations shared by the C-ABI layer and the launch glue.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace occ {

struct Params;

struct Geometry {
  int64_t n = 0, m = 0;
  int r = 0;
  int cs1 = 0, s1 = 0;   // sweep-1 column split width / count
  int rs2 = 0, s2 = 0;   // sweep-2 row split height / count
  int ngp = 0;           // Gram partial count (units of 128 rows)
};

constexpr size_t kTraceOffset = 256;
constexpr int kTraceSlots = 48;                           // per CTA: 24 clock64 stamps, then the matching globaltimer stamps (v2::kTrStamps)
constexpr size_t kTraceBytes = 160 * kTraceSlots * 8;     // up to 160 CTAs
constexpr size_t kBarLinesOffset = kTraceOffset + kTraceBytes;   // v2 grid barrier: spread arrival counters
constexpr size_t kBarLinesBytes = 8 * 128;                        // (v2::kBarLines lines of 128 B)

struct WsLayout {
  size_t bar = 0, p_part = 0, q_part = 0, g_part = 0, g2_part = 0, xy_part = 0;
  size_t p_bucket = 0, qw_bucket = 0, qs_bucket = 0, qt = 0, li = 0, gred = 0, v2_tail = 0, v2_tail_bytes = 0, total = 0;
};

Geometry make_geometry(int64_t n, int64_t m, int r, int sms);
WsLayout make_layout(const Geometry& g, int nmat);
void fill_ws(Params& p, const Geometry& g, const WsLayout& L, void* ws);

cudaError_t run_phases(const Params& p, const Geometry& g, int ph0, int ph1, bool multi, bool dpl,
                       cudaStream_t st);
cudaError_t run_decompress(const Params& p, int r, cudaStream_t st);
// one rank's step kernels (occ_step_r{4..64}.cu)
#define OCC_DECL_STEP(RR)                                                                               \
  cudaError_t run_phases_r##RR(const Params& p, const Geometry& g, int ph0, int ph1, bool multi, bool dpl, \
                               cudaStream_t st);                                                        \
  unsigned take_nonfinite_v1_r##RR();
OCC_DECL_STEP(4)
OCC_DECL_STEP(8)
OCC_DECL_STEP(16)
OCC_DECL_STEP(32)
OCC_DECL_STEP(64)
#undef OCC_DECL_STEP
size_t v2_tail_bytes(int64_t n, int64_t m, int r, int sms);
cudaError_t run_v2(const Params& p, int r, void* ws_tail, size_t tail_avail, int sms, cudaStream_t st);
// OCC_CHECK_FINITE: read and clear the device status words (occ_check_status)
unsigned take_nonfinite_v1();
// OCC_WIRE_BF16 helpers (occ_step.cu)
cudaError_t run_round_bf16(float* x, long long count, cudaStream_t st);
cudaError_t run_pack_bf16(const float* x, void* y, long long count, cudaStream_t st);
cudaError_t run_unpack_bf16(const void* y, float* x, long long count, cudaStream_t st);
unsigned take_nonfinite_v2();
// out = round(P Q^T) with the fused kernel's phase-5 arithmetic (bit-identical
// to the sender's reconstruction, reading C8); every supported rank (4..64),
// cudaErrorNotSupported for any other.
cudaError_t run_v2_decompress(const float* P, const float* Q, void* out, long long ldo, int n, int m, int r, bool bf16,
                              cudaStream_t st);
// sender-side M' and e_new = (M + e_old) - M' of the per-phase paths, in the
// decompress kernel's arithmetic (reading C8), every supported rank (4..64).
// A = M + e_old is loaded before M' is stored, so recon may alias M.
cudaError_t run_v2_reconstruct(const Params& p, int r, cudaStream_t st);
cudaError_t run_init_q(float* q, int64_t rows, int r, int64_t ld, uint64_t seed, cudaStream_t st);
// occ_link receiver side of one step (occ_v2.cu)
struct LinkRecv {
  const unsigned* wait_flag;   // local flag word
  unsigned seq;
  unsigned* ack;               // the sender's ack word (peer memory)
  unsigned* ctr;               // local CTA-exit counter
  float* copyP;                // caller's Prcv / Qrcv (or nullptr)
  float* copyQ;
  long long nP, nQ;            // floats
};
cudaError_t run_v2_decompress_link(const float* P, const float* Q, void* out, long long ldo, int n, int m, int r,
                                   bool bf16, const LinkRecv& lr, cudaStream_t st);
cudaError_t run_link_copy(const float* sP, const float* sQ, float* dP, float* dQ, long long nP, long long nQ,
                          const unsigned* wait_word, unsigned wait_target, unsigned* ctr, unsigned* done_word,
                          unsigned done_seq, cudaStream_t st);
cudaError_t run_link_exchange(const float* sP, const float* sQ, float* pP, float* pQ, long long nP, long long nQ,
                              const unsigned* ack_in, unsigned* push_ctr, unsigned* peer_flag, unsigned sseq,
                              const float* mP, const float* mQ, float* dP, float* dQ, long long mnP, long long mnQ,
                              const unsigned* flag_in, unsigned* recv_ctr, unsigned* peer_ack, unsigned rseq,
                              cudaStream_t st);
unsigned take_link_timeout();
// occ_dplink: the in-kernel allreduce-sum of a DP group over NVLink peer memory (occ_v2.cu)
constexpr int kDplinkMax = 8;
struct DplinkArgs {
  int D, rank;
  unsigned seq;
  long long cap, words_off;   // floats per slot; byte offset of the words
  char* base[kDplinkMax];     // every member's mailbox (this rank's own included)
  const float* src;
  float* dst;
  long long count;
};
cudaError_t run_dplink_kernel(const DplinkArgs& a, cudaStream_t st);
// tcgen05 sweeps (occ_umma.cu): workspace of the split, transposed small factor
size_t umma_qt_bytes(int64_t n, int64_t m, int r);
bool umma_applies(const Params& p, int r);
// dst = sum of S partials of count floats, stride floats apart (fixed order)
cudaError_t run_reduce_partials(const float* src, long long stride, int S, float* dst, long long count,
                                cudaStream_t st);
// sweep 1 (transposed = false: P_part) or sweep 2 (true: Q_part) on tcgen05
cudaError_t run_umma_sweep(const Params& p, int r, bool transposed, int max_splits, int* G_out, cudaStream_t st);
// the DP reconstruction (phase F with f_tc) on tcgen05, r in {32, 64}
cudaError_t run_umma_recon(const Params& p, int r, cudaStream_t st);

}  // namespace occ
