// occ_umma.cu -- the per-phase path's streaming kernels on the 5th-generation
// tensor cores (tcgen05, TMEM, TMA tensor maps), for the shapes the fused
// kernel does not hold on chip (BASELINE configs[2], configs[3], the G^T
// embedding: r = 16 .. 64, fp32 M):
//   umma_sweep_kernel<R, false>  sweep 1, P_part = (M + e) Q_prev        (a1, a2)
//   umma_sweep_kernel<R, true>   sweep 2, Q_part = (M + e)^T P_hat       (a1, a5)
//   occ_reduce_partials_kernel   P / Q = the sum of the sweeps' partials
//   umma_recon_kernel<R, MODE>   the DP reconstruction, M' and e_new      (a7, a8)
// (north_star steps; PAPER.md:269-270 the PowerSGD power iteration, 383-389
// lazy error propagation, 676-677 the DP allreduce of P and Q.)
//
// Sweeps: one persistent CTA per SM, warp-specialised:
//   warp 0      TMA producer: 2-D tensor-map loads (cp.async.bulk.tensor, 128-B
//               swizzle) of a 128-row x 32-column box of M and of e (sweep 2:
//               four 32 x 32 boxes, 128-B swizzle with 32-B atoms), and of the
//               32-wide slices of the small factor's transpose split into hi / lo
//               (pre-split once per step by occ_split_t_kernel), into an
//               mbarrier ring of stages.
//   warps 2..5  converters: A = M + e and the 3-term TF32 split A = A_hi + A_lo
//               (hi: the low 13 mantissa bits masked off, lo = A - hi exact in
//               fp32), in place (A_hi over the M box, A_lo over the e box) --
//               elementwise, so the swizzled layout TMA wrote is kept as is.
//   warp 1      MMA issuer (one thread): per stage and per 8-wide K step,
//               tcgen05.mma.kind::tf32 A_lo.F_hi + A_hi.F_lo + A_hi.F_hi
//               (fp32-level accuracy) into a 128 x R fp32 accumulator in TENSOR
//               MEMORY; tcgen05.commit frees the stage back to the producer.
//   epilogue    the converter warps drain the accumulator (tcgen05.ld, lane =
//               output row) into fp32 registers every 256 terms and store the
//               band's partial rows.
// Work split: a band of 128 output rows is shared by G CTAs, each owning a
// contiguous range of 32-wide K chunks (G = the smallest count that keeps the
// persistent grid busy), so the reduce that follows reads G partials.
#include "occ_internal.h"
#include "occ_kernels.cuh"
#include "occ_v2.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

namespace occ {
namespace umma {

using v2::mbar_arrive;
using v2::mbar_expect_tx;
using v2::mbar_init;
using v2::mbar_wait;
using v2::smem_u32;

constexpr int BM = 128;    // tile rows = TMEM lanes = MMA M
constexpr int KC = 32;     // columns per stage: one 128-byte swizzle row of fp32
constexpr int NTH = 192;   // warp 0 producer, warp 1 MMA, warps 2..5 converters / epilogue
constexpr int NCV = 128;   // converter threads
// K chunks per TMEM accumulator: the tensor core's fp32 accumulation loses
// precision linearly in the chain length (measured: element error vs the fp64
// oracle 3.9e-6 at 256 terms, 1.8e-5 at 2048, relative to max|A|), so each
// 256-term partial is drained into fp32 registers (tools/umma_acc.py)
constexpr int KSUB = 8;
constexpr int kSmemCap = 227 * 1024;

template <int R>
struct Cfg1 {
  static constexpr int N = R;                                // MMA N
  static constexpr int BOX_A = BM * KC * 4;                  // one M (or e) box, bytes
  static constexpr int BOX_Q = N * KC * 4;                   // one Q^T hi (or lo) box
  static constexpr int STAGE = 2 * BOX_A + 2 * BOX_Q;        // multiple of 1024
  static constexpr int NS = std::min(6, (kSmemCap - 2048) / STAGE);
  static constexpr int SMEM = NS * STAGE + 1024 /* align */ + 512 /* barriers */;
  static constexpr int TCOLS = (2 * N <= 32) ? 32 : (2 * N <= 64) ? 64 : (2 * N <= 128) ? 128 : 256;
};

struct S1Args {
  int n, m;
  int nrb, G, nkc;   // bands (128 rows; sweep 2: 128 columns), CTAs per band, 32-wide K chunks
  int has_e;
  float* P_part;     // sweep 1: [G][n][R]; sweep 2: Q_part [G][m][R]
};

// K-major operand, 128-byte swizzle, 8-row groups 1024 B apart (sm_100 descriptor version 1)
__device__ __forceinline__ uint64_t desc_k_sw128(unsigned saddr) {
  uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;              // leading byte offset (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;    // stride byte offset
  d |= (uint64_t)1 << 46;              // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;              // SWIZZLE_128B
  return d;
}
// MN-major tf32 operand: the only layout the hardware takes for it is the
// 128-byte swizzle with 32-byte atoms (SWIZZLE_128B_BASE32B, descriptor layout
// type 1; TMA CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B): a K row is 128 B of 32
// consecutive M elements, 4-row K groups 512 B apart (SBO), 32-element M
// atoms LBO apart
__device__ __forceinline__ uint64_t desc_mn_sw128_32b(unsigned saddr, unsigned lbo) {
  uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)1 << 61;
  return d;
}
// instruction descriptor: D f32, A / B tf32, B K-major, A K-major (a_mn = 0) or
// MN-major (a_mn = 1, sweep 2: A^T read from A's row-major tile), M = 128, N
__host__ __device__ constexpr uint32_t idesc_tf32(int N, int a_mn = 0) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(BM >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32(unsigned tmem_d, uint64_t a, uint64_t b, uint32_t idesc, unsigned acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* tm, int x, int y, uint64_t* bar,
                                       unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ uint4 split_hi(float4 a, uint4& lo) {
  uint4 h;
  h.x = __float_as_uint(a.x) & 0xffffe000u;
  h.y = __float_as_uint(a.y) & 0xffffe000u;
  h.z = __float_as_uint(a.z) & 0xffffe000u;
  h.w = __float_as_uint(a.w) & 0xffffe000u;
  lo.x = __float_as_uint(a.x - __uint_as_float(h.x));
  lo.y = __float_as_uint(a.y - __uint_as_float(h.y));
  lo.z = __float_as_uint(a.z - __uint_as_float(h.z));
  lo.w = __float_as_uint(a.w - __uint_as_float(h.w));
  return h;
}

// T = false: sweep 1, D[128 rows][R] = A[rows][K = 32-column chunks] . Q_prev
//   (A K-major: one 32-column x 128-row TMA box per operand and stage).
// T = true: sweep 2, D[128 columns][R] = A^T[columns][K = 32-row chunks] . F
//   (F = P_hat, or the row-side factor of OCC_ORIENT_T): the same row-major
//   tile read as an MN-major operand -- four 32-column x 32-row boxes per
//   stage (128-B swizzle with 32-B atoms), 4096 B apart (LBO), each K row
//   128 B, 4-row groups 512 B (SBO).
// The small factor arrives pre-split and transposed (K-major) either way.
template <int R, bool T>
__global__ void __launch_bounds__(NTH, 1)
    umma_sweep_kernel(const __grid_constant__ CUtensorMap tmM, const __grid_constant__ CUtensorMap tmE,
                      const __grid_constant__ CUtensorMap tmQh, const __grid_constant__ CUtensorMap tmQl,
                      const S1Args a) {
  using C = Cfg1<R>;
  constexpr int NS = C::NS, N = C::N;
  extern __shared__ unsigned char smraw[];
  unsigned char* sm = smraw + ((1024 - (smem_u32(smraw) & 1023)) & 1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + NS * C::STAGE);
  uint64_t* conv = full + NS;
  uint64_t* empty = conv + NS;
  uint64_t* accf = empty + NS;    // [2] accumulator ready (MMA -> epilogue)
  uint64_t* acce = accf + 2;      // [2] accumulator drained (epilogue -> MMA)
  unsigned* tmem_hold = reinterpret_cast<unsigned*>(acce + 2);
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  auto stM = [&](int s) { return sm + s * C::STAGE; };
  auto stE = [&](int s) { return sm + s * C::STAGE + C::BOX_A; };
  auto stQh = [&](int s) { return sm + s * C::STAGE + 2 * C::BOX_A; };
  auto stQl = [&](int s) { return sm + s * C::STAGE + 2 * C::BOX_A + C::BOX_Q; };

  if (w == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_hold)),
                 "n"(C::TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < NS; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], NCV / 32);   // one arrival per converter warp
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; b++) {
      mbar_init(&accf[b], 1);
      mbar_init(&acce[b], NCV / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tbase = *tmem_hold;
  const int items = a.nrb * a.G;
  auto range = [&](int it, int& band, int& gi, int& c_lo, int& c_hi) {
    band = it / a.G;
    gi = it % a.G;
    c_lo = (int)((long long)gi * a.nkc / a.G);
    c_hi = (int)((long long)(gi + 1) * a.nkc / a.G);
  };

  if (w == 0) {
    if (lane == 0) {   // ------------------------------------------------ TMA producer
      const unsigned long long pol_stream = v2::l2_evict_first(), pol_keep = v2::l2_evict_normal();
      const unsigned bytes = (a.has_e ? 2 : 1) * C::BOX_A + 2 * C::BOX_Q;
      int s = 0;
      unsigned ph = 0;
      for (int it = blockIdx.x; it < items; it += gridDim.x) {
        int band, gi, c_lo, c_hi;
        range(it, band, gi, c_lo, c_hi);
        for (int c = c_lo; c < c_hi; c++) {
          mbar_wait(&empty[s], ph ^ 1u);
          mbar_expect_tx(&full[s], bytes);
          if constexpr (T) {
#pragma unroll
            for (int q = 0; q < BM / KC; q++) {
              tma_2d(stM(s) + q * (C::BOX_A / 4), &tmM, band * BM + q * KC, c * KC, &full[s], pol_stream);
              if (a.has_e) tma_2d(stE(s) + q * (C::BOX_A / 4), &tmE, band * BM + q * KC, c * KC, &full[s], pol_stream);
            }
          } else {
            tma_2d(stM(s), &tmM, c * KC, band * BM, &full[s], pol_stream);
            if (a.has_e) tma_2d(stE(s), &tmE, c * KC, band * BM, &full[s], pol_stream);
          }
          tma_2d(stQh(s), &tmQh, c * KC, 0, &full[s], pol_keep);
          tma_2d(stQl(s), &tmQl, c * KC, 0, &full[s], pol_keep);
          if (++s == NS) { s = 0; ph ^= 1u; }
        }
      }
    }
  } else if (w == 1) {
    if (lane == 0) {   // ------------------------------------------------ MMA issuer
      constexpr uint32_t idesc = idesc_tf32(N, T ? 1 : 0);
      int s = 0;
      unsigned ph = 0, aph[2] = {0u, 0u};
      int k = 0;
      for (int it = blockIdx.x; it < items; it += gridDim.x) {
        int band, gi, c_lo, c_hi;
        range(it, band, gi, c_lo, c_hi);
        for (int sb = c_lo; sb < c_hi; sb += KSUB, k++) {   // one accumulator per KSUB chunks
          const int se = min(c_hi, sb + KSUB);
          const int ab = k & 1;
          mbar_wait(&acce[ab], aph[ab] ^ 1u);   // the epilogue has drained this accumulator
          aph[ab] ^= 1u;
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const unsigned td = tbase + (unsigned)(ab * N);
          for (int c = sb; c < se; c++) {
            mbar_wait(&conv[s], ph);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            uint64_t dh, dl;
            if constexpr (T) {
              dh = desc_mn_sw128_32b(smem_u32(stM(s)), C::BOX_A / 4);
              dl = desc_mn_sw128_32b(smem_u32(stE(s)), C::BOX_A / 4);
            } else {
              dh = desc_k_sw128(smem_u32(stM(s)));
              dl = desc_k_sw128(smem_u32(stE(s)));
            }
            const uint64_t qh = desc_k_sw128(smem_u32(stQh(s))), ql = desc_k_sw128(smem_u32(stQl(s)));
#pragma unroll
            for (int kk = 0; kk < KC / 8; kk++) {
              // K step of 8: K-major +32 B inside the swizzle row; MN-major +8 K rows = 1024 B
              const uint64_t oa = T ? (uint64_t)(64 * kk) : (uint64_t)(2 * kk);
              const uint64_t ob = (uint64_t)(2 * kk);
              mma_tf32(td, dl + oa, qh + ob, idesc, (c > sb || kk > 0) ? 1u : 0u);
              mma_tf32(td, dh + oa, ql + ob, idesc, 1u);
              mma_tf32(td, dh + oa, qh + ob, idesc, 1u);
            }
            mma_commit(&empty[s]);
            if (++s == NS) { s = 0; ph ^= 1u; }
          }
          mma_commit(&accf[ab]);
        }
      }
    }
  } else {   // ------------------------------------------------------------ converters + epilogue
    const int ct = tid - 64;
    int s = 0;
    unsigned ph = 0, aph[2] = {0u, 0u};
    int k = 0;
    const int q = w & 3;   // TMEM lane quadrant of this warp
    const int nout = T ? a.m : a.n;
    float acc[R];          // the item's sum of its KSUB-chunk accumulators (row 32 q + lane)
    // drain accumulator kk: tcgen05.ld (lane = output row, sweep 2: column) into acc
    auto drain = [&](int kk) {
      const int ab = kk & 1;
      mbar_wait(&accf[ab], aph[ab]);
      aph[ab] ^= 1u;
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const unsigned ta = tbase + ((unsigned)(32 * q) << 16) + (unsigned)(ab * N);
#pragma unroll
      for (int j = 0; j < R / 16; j++) {
        float v[16];
        v2::tmem_ld16(ta + 16 * j, v);
#pragma unroll
        for (int u = 0; u < 16; u++) acc[16 * j + u] += v[u];
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&acce[ab]);
    };
    for (int it = blockIdx.x; it < items; it += gridDim.x) {
      int band, gi, c_lo, c_hi;
      range(it, band, gi, c_lo, c_hi);
#pragma unroll
      for (int j = 0; j < R; j++) acc[j] = 0.f;
      int pend = -1;
      for (int sb = c_lo; sb < c_hi; sb += KSUB, k++) {
        const int se = min(c_hi, sb + KSUB);
        for (int c = sb; c < se; c++) {
          mbar_wait(&full[s], ph);
          uint4* pm = reinterpret_cast<uint4*>(stM(s));
          uint4* pe = reinterpret_cast<uint4*>(stE(s));
#pragma unroll
          for (int j = 0; j < C::BOX_A / 16 / NCV; j++) {
            const int x = ct + NCV * j;
            const uint4 mv = pm[x];
            float4 av = make_float4(__uint_as_float(mv.x), __uint_as_float(mv.y), __uint_as_float(mv.z),
                                    __uint_as_float(mv.w));
            if (a.has_e) {
              const uint4 ev = pe[x];
              const float2 s0 = v2::add2(make_float2(av.x, av.y), make_float2(__uint_as_float(ev.x), __uint_as_float(ev.y)));
              const float2 s1 = v2::add2(make_float2(av.z, av.w), make_float2(__uint_as_float(ev.z), __uint_as_float(ev.w)));
              av = make_float4(s0.x, s0.y, s1.x, s1.y);
            }
            uint4 lo;
            pm[x] = split_hi(av, lo);
            pe[x] = lo;
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(&conv[s]);
          if (++s == NS) { s = 0; ph ^= 1u; }
        }
        if (pend >= 0) drain(pend);   // the previous accumulator, while this one's MMAs run
        pend = k;
      }
      if (pend >= 0) drain(pend);
      // epilogue: output row (sweep 2: column) 32 q + lane of the band, R columns
      const int row = band * BM + 32 * q + lane;
      if (row < nout) {
        float* dst = a.P_part + ((size_t)gi * nout + row) * R;
#pragma unroll
        for (int j = 0; j < R / 4; j++)
          reinterpret_cast<float4*>(dst)[j] = make_float4(acc[4 * j], acc[4 * j + 1], acc[4 * j + 2], acc[4 * j + 3]);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (w == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(C::TCOLS));
}

// ------------------------------------------------------------------ DP reconstruction
// The data-parallel reconstruction (north_star a7, a8; reading C1/C2/C15/C6)
// on tcgen05: two products per tile, out of TMEM accumulators
//   D1[c][i] = sum_k C1[c][k] R1[i][k]   -> M' = round(D1)
//   D2[c][i] = sum_k C2[c][k] R2[i][k]   -> e_new = A - D2 (DPL)   (else A - M')
// with plain DP: C1 = scale Q_sum, C2 = Q_w, R1 = R2 = P_hat; OCC_ORIENT_T:
// C1 = C2 = U_hat, R1 = scale V_sum, R2 = V_w (the occ_tc.cuh phase_F_tc
// definitions).  The MMA's M index (TMEM lane) is the COLUMN of the output,
// so the epilogue thread of lane c reads and writes column c of consecutive
// rows: a warp's accesses are 32 consecutive floats of one row (coalesced)
// without any staging.  A CTA owns a 128-column band (its column factors hi /
// lo resident in shared memory) and a range of 64-row tiles, whose row
// factors stream through a two-stage TMA ring.  Warp 0 TMA, warp 1 MMA,
// warps 2..9 epilogue (warp w serves TMEM lane quadrant w % 4 and rows
// 32 ((w - 2) / 4) .. + 31 of the tile).
namespace rc {
constexpr int BC = 128;     // columns per band (MMA M)
constexpr int TR = 64;      // rows per tile (MMA N)
constexpr int NTH = 320;    // warp 0 TMA, warp 1 MMA, warps 2..9 epilogue
constexpr int NEP = 256;    // epilogue threads
constexpr int NSMAX = 3;    // row-factor stages (as many as shared memory holds, at most 3)
template <int R>
struct Cfg {
  static constexpr int CBOX = BC * R * 4;       // one column-factor operand (hi or lo), all K blocks
  static constexpr int RBOX = TR * R * 4;       // one row-factor operand
  static constexpr int stages(bool two_c, bool two_r) {
    const int left = kSmemCap - (two_c ? 4 : 2) * CBOX - 1024 - 512;
    const int ns = left / ((two_r ? 4 : 2) * RBOX);
    return ns < NSMAX ? ns : NSMAX;
  }
  static constexpr int smem(bool two_c, bool two_r) {
    return (two_c ? 4 : 2) * CBOX + stages(two_c, two_r) * (two_r ? 4 : 2) * RBOX + 1024 + 512;
  }
};
}  // namespace rc

struct RcArgs {
  int n, m, nb, G, ntile;       // column bands, row splits per band, 64-row tiles
  int dpl;                      // e_new = A - D2 (else A - round(D1))
  int has_e, r_bf16;
  int ns;                       // row-factor stages
  const float* M; long long ldm;
  const float* E; long long lde;
  void* out; long long ldo;     // M' (nullptr: not written)
  float* Eo; long long ldeo;    // e_new (nullptr: not written)
};

// MODE: 0 e_new = A - M' (global EF, one product); 1 plain DP, local EF (a
// second column factor Q_w); 2 OCC_ORIENT_T, local EF (a second row factor V_w)
template <int R, int MODE>
__global__ void __launch_bounds__(rc::NTH, 1)
    umma_recon_kernel(const __grid_constant__ CUtensorMap tC1h, const __grid_constant__ CUtensorMap tC1l,
                      const __grid_constant__ CUtensorMap tC2h, const __grid_constant__ CUtensorMap tC2l,
                      const __grid_constant__ CUtensorMap tR1h, const __grid_constant__ CUtensorMap tR1l,
                      const __grid_constant__ CUtensorMap tR2h, const __grid_constant__ CUtensorMap tR2l,
                      const RcArgs a) {
  using C = rc::Cfg<R>;
  constexpr int KB = R / 32;                 // 32-wide K blocks (128-B swizzle rows)
  constexpr int CB1 = rc::BC * 32 * 4;       // one K block of a column operand
  constexpr int RB1 = rc::TR * 32 * 4;       // one K block of a row operand
  extern __shared__ unsigned char smraw[];
  unsigned char* sm = smraw + ((1024 - (smem_u32(smraw) & 1023)) & 1023);
  constexpr bool TWO_C = MODE == 1, TWO_R = MODE == 2, DPL2 = MODE != 0;
  constexpr int ncop = TWO_C ? 4 : 2, nrop = TWO_R ? 4 : 2;
  unsigned char* cbase = sm;                                   // [ncop][KB][128 rows][128 B]
  unsigned char* rbase = sm + ncop * C::CBOX;                  // [NS][nrop][KB][64 rows][128 B]
  const int NS = a.ns;
  uint64_t* bars = reinterpret_cast<uint64_t*>(rbase + NS * nrop * C::RBOX);
  uint64_t* cfull = bars;
  uint64_t* cempty = bars + 1;
  uint64_t* rfull = bars + 2;                 // [NS]
  uint64_t* rempty = rfull + NS;              // [NS]
  uint64_t* accf = rempty + NS;               // [2]
  uint64_t* acce = accf + 2;                  // [2]
  unsigned* tmem_hold = reinterpret_cast<unsigned*>(acce + 2);
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  auto cop = [&](int o) { return cbase + o * C::CBOX; };
  auto rop = [&](int s, int o) { return rbase + (s * nrop + o) * C::RBOX; };

  if (w == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_hold)),
                 "n"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(cfull, 1);
    mbar_init(cempty, 1);
    for (int s = 0; s < NS; s++) {
      mbar_init(&rfull[s], 1);
      mbar_init(&rempty[s], 1);
    }
    for (int b = 0; b < 2; b++) {
      mbar_init(&accf[b], 1);
      mbar_init(&acce[b], rc::NEP / 32);   // one arrival per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tbase = *tmem_hold;
  const int items = a.nb * a.G;
  auto range = [&](int it, int& band, int& t_lo, int& t_hi) {
    band = it / a.G;
    const int gi = it % a.G;
    t_lo = (int)((long long)gi * a.ntile / a.G);
    t_hi = (int)((long long)(gi + 1) * a.ntile / a.G);
  };

  if (w == 0) {   // ------------------------------------------------ TMA producer (lane 0)
    const unsigned long long pol = v2::l2_evict_normal();
    int s = 0;
    unsigned ph = 0, cph = 0;
    for (int it = blockIdx.x; it < items; it += gridDim.x) {
      int band, t_lo, t_hi;
      range(it, band, t_lo, t_hi);
      if (lane == 0) {
        mbar_wait(cempty, cph ^ 1u);
        mbar_expect_tx(cfull, ncop * C::CBOX);
#pragma unroll
        for (int kb = 0; kb < KB; kb++) {
          tma_2d(cop(0) + kb * CB1, &tC1h, 32 * kb, band * rc::BC, cfull, pol);
          tma_2d(cop(1) + kb * CB1, &tC1l, 32 * kb, band * rc::BC, cfull, pol);
          if (TWO_C) {
            tma_2d(cop(2) + kb * CB1, &tC2h, 32 * kb, band * rc::BC, cfull, pol);
            tma_2d(cop(3) + kb * CB1, &tC2l, 32 * kb, band * rc::BC, cfull, pol);
          }
        }
      }
      cph ^= 1u;
      for (int t = t_lo; t < t_hi; t++) {
        if (lane == 0) {
          mbar_wait(&rempty[s], ph ^ 1u);
          mbar_expect_tx(&rfull[s], nrop * C::RBOX);
#pragma unroll
          for (int kb = 0; kb < KB; kb++) {
            tma_2d(rop(s, 0) + kb * RB1, &tR1h, 32 * kb, t * rc::TR, &rfull[s], pol);
            tma_2d(rop(s, 1) + kb * RB1, &tR1l, 32 * kb, t * rc::TR, &rfull[s], pol);
            if (TWO_R) {
              tma_2d(rop(s, 2) + kb * RB1, &tR2h, 32 * kb, t * rc::TR, &rfull[s], pol);
              tma_2d(rop(s, 3) + kb * RB1, &tR2l, 32 * kb, t * rc::TR, &rfull[s], pol);
            }
          }
        }
        if (++s == NS) { s = 0; ph ^= 1u; }
      }
    }
  } else if (w == 1) {
    if (lane == 0) {   // ------------------------------------------------ MMA issuer
      constexpr uint32_t idesc = idesc_tf32(rc::TR);
      int s = 0, k = 0;
      unsigned ph = 0, cph = 0, aph[2] = {0u, 0u};
      for (int it = blockIdx.x; it < items; it += gridDim.x) {
        int band, t_lo, t_hi;
        range(it, band, t_lo, t_hi);
        mbar_wait(cfull, cph);
        cph ^= 1u;
        for (int t = t_lo; t < t_hi; t++, k++) {
          const int ab = k & 1;
          mbar_wait(&acce[ab], aph[ab] ^ 1u);
          aph[ab] ^= 1u;
          mbar_wait(&rfull[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const unsigned d1 = tbase + (unsigned)(ab * 2 * rc::TR), d2 = d1 + rc::TR;
          // descriptors of the stage's operands; the K steps add constant offsets
          // (16-byte units) to the start-address field: a straight-line block of
          // 3 R / 8 (x 2 with the second product) MMAs
          const uint64_t c1h = desc_k_sw128(smem_u32(cop(0))), c1l = desc_k_sw128(smem_u32(cop(1)));
          const uint64_t r1h = desc_k_sw128(smem_u32(rop(s, 0))), r1l = desc_k_sw128(smem_u32(rop(s, 1)));
          const uint64_t c2h = TWO_C ? desc_k_sw128(smem_u32(cop(2))) : c1h;
          const uint64_t c2l = TWO_C ? desc_k_sw128(smem_u32(cop(3))) : c1l;
          const uint64_t r2h = TWO_R ? desc_k_sw128(smem_u32(rop(s, 2))) : r1h;
          const uint64_t r2l = TWO_R ? desc_k_sw128(smem_u32(rop(s, 3))) : r1l;
#pragma unroll
          for (int kk = 0; kk < R / 8; kk++) {
            const uint64_t co = (uint64_t)(((kk >> 2) * CB1 + (kk & 3) * 32) >> 4);
            const uint64_t ro = (uint64_t)(((kk >> 2) * RB1 + (kk & 3) * 32) >> 4);
            const unsigned acc = kk > 0 ? 1u : 0u;
            mma_tf32(d1, c1l + co, r1h + ro, idesc, acc);
            mma_tf32(d1, c1h + co, r1l + ro, idesc, 1u);
            mma_tf32(d1, c1h + co, r1h + ro, idesc, 1u);
            if (DPL2) {
              mma_tf32(d2, c2l + co, r2h + ro, idesc, acc);
              mma_tf32(d2, c2h + co, r2l + ro, idesc, 1u);
              mma_tf32(d2, c2h + co, r2h + ro, idesc, 1u);
            }
          }
          mma_commit(&rempty[s]);
          mma_commit(&accf[ab]);
          if (++s == NS) { s = 0; ph ^= 1u; }
        }
        mma_commit(cempty);
      }
    }
  } else {   // ------------------------------------------------------------ epilogue
    const int q = w & 3, h = (w - 2) >> 2;
    unsigned aph[2] = {0u, 0u};
    int k = 0;
    // One tile of this warp: M and e of the thread's column for the warp's 32
    // rows (all 64 loads in flight before the accumulator wait), then M' and
    // e_new.  (An L2 bulk prefetch of the next tiles' rows by the producer warp
    // measured slower: 194 vs 160 us for the MLP matrix.)  The flags
    // are compile-time in the element loop (DPL: e_new against the second
    // product; EF: e read and written; RBF: M' in bf16; FULL: all 32 rows exist).
    auto tile = [&](auto dpl_, auto ef_, auto full_, auto gen_, int c, bool cok, int i0, int ab, int inext) {
      // GEN: every flag read at run time (bf16 output, no error feedback, ...)
      constexpr bool GEN = decltype(gen_)::value, FULL = decltype(full_)::value;
      const bool DPL = GEN ? a.dpl != 0 : decltype(dpl_)::value;
      const bool HE = GEN ? a.has_e != 0 : decltype(ef_)::value;
      const bool WE = GEN ? a.Eo != nullptr : decltype(ef_)::value;
      const bool RBF = GEN ? a.r_bf16 != 0 : false;
      const bool WO = GEN ? a.out != nullptr : true;
      float mv[32], ev[32];
      const size_t ldm = (size_t)a.ldm, lde = (size_t)a.lde, ldo = (size_t)a.ldo, ldeo = (size_t)a.ldeo;
      const float* pm = a.M + (size_t)i0 * ldm + c;
      const float* pe = HE ? a.E + (size_t)i0 * lde + c : nullptr;
#pragma unroll
      for (int j = 0; j < 32; j++) {
        const bool ok = cok && (FULL || i0 + j < a.n);
        mv[j] = ok ? __ldcs(pm + j * ldm) : 0.f;
        ev[j] = (ok && HE) ? __ldcs(pe + j * lde) : 0.f;
      }
      // the warp's next tile into L2 while this one waits and stores: lane j
      // prefetches the 128-byte line of row inext + j (the warp's 32 columns)
      if (inext >= 0 && inext + lane < a.n && c - lane < a.m) {
        const size_t o = (size_t)(inext + lane);
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.M + o * ldm + (c - lane)));
        if (HE) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.E + o * lde + (c - lane)));
      }
      mbar_wait(&accf[ab], aph[ab]);
      aph[ab] ^= 1u;
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const unsigned ta = tbase + ((unsigned)(32 * q) << 16) + (unsigned)(ab * 2 * rc::TR + 32 * h);
      float* po = reinterpret_cast<float*>(a.out) + (size_t)i0 * ldo + c;
      __nv_bfloat16* pob = reinterpret_cast<__nv_bfloat16*>(a.out) + (size_t)i0 * ldo + c;
      float* peo = a.Eo + (size_t)i0 * ldeo + c;
#pragma unroll
      for (int hh = 0; hh < 2; hh++) {
        float d1[16], d2[16];
        v2::tmem_ld16(ta + 16 * hh, d1);
        if (DPL) v2::tmem_ld16(ta + rc::TR + 16 * hh, d2);
#pragma unroll
        for (int jj = 0; jj < 16; jj++) {
          const int j = 16 * hh + jj;
          if (!cok || !(FULL || i0 + j < a.n)) continue;
          float mr = d1[jj];
          if (RBF) {
            const __nv_bfloat16 b = __float2bfloat16_rn(mr);
            if (WO) pob[j * ldo] = b;
            mr = __bfloat162float(b);
          } else if (WO) {
            __stcs(po + j * ldo, mr);
          }
          if (WE) __stcs(peo + j * ldeo, (mv[j] + ev[j]) - (DPL ? d2[jj] : mr));
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&acce[ab]);
    };
    using T1 = std::true_type;
    using F0 = std::false_type;
    const bool fast = !a.r_bf16 && a.has_e && a.Eo && a.out;   // fp32 M' and error feedback (the DP step)
    for (int it = blockIdx.x; it < items; it += gridDim.x) {
      int band, t_lo, t_hi;
      range(it, band, t_lo, t_hi);
      const int c = band * rc::BC + 32 * q + lane;
      const bool cok = c < a.m;
      for (int t = t_lo; t < t_hi; t++, k++) {
        const int ab = k & 1;
        const int i0 = t * rc::TR + 32 * h;   // this warp's first row
        const bool full = i0 + 32 <= a.n;
        const int inext = t + 1 < t_hi ? i0 + rc::TR : -1;
        if (fast && a.dpl) {
          if (full) tile(T1{}, T1{}, T1{}, F0{}, c, cok, i0, ab, inext);
          else tile(T1{}, T1{}, F0{}, F0{}, c, cok, i0, ab, inext);
        } else if (fast) {
          if (full) tile(F0{}, T1{}, T1{}, F0{}, c, cok, i0, ab, inext);
          else tile(F0{}, T1{}, F0{}, F0{}, c, cok, i0, ab, inext);
        } else {
          tile(F0{}, F0{}, F0{}, T1{}, c, cok, i0, ab, inext);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (w == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(256));
}

// The reconstruction's factor operands, all in one launch: for each of up to
// four factors x (rows x R, row stride R), x scaled by `scale`, split hi / lo
// (K-major, row stride R); `state` (optional) receives the scaled factor (the
// warm start, reading C15).
struct SplitJob {
  const float* x;
  long long count;
  float scale;
  unsigned* hi;
  unsigned* lo;
  float* state;
};
struct SplitJobs {
  SplitJob j[4];
  int n;
};
__global__ void occ_split_rows_kernel(const __grid_constant__ SplitJobs jobs) {
  for (int q = 0; q < jobs.n; q++) {
    const SplitJob& J = jobs.j[q];
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < J.count;
         i += (long long)gridDim.x * blockDim.x) {
      const float v = J.scale * J.x[i];
      if (J.state) J.state[i] = v;
      const unsigned hb = __float_as_uint(v) & 0xffffe000u;
      J.hi[i] = hb;
      J.lo[i] = __float_as_uint(v - __uint_as_float(hb));
    }
  }
}

// dst = sum of S partials (src + s * stride, s = 0 .. S-1, fixed order) of
// `count` floats: the sweeps' P / Q reduce as a plain launch (16-byte vectors,
// 4 partials per step in flight) instead of a cooperative step-kernel phase.
__global__ void __launch_bounds__(256) occ_reduce_partials_kernel(const float* __restrict__ src, long long stride,
                                                                  int S, float* __restrict__ dst, long long count) {
  const long long nv = count / 4, sv = stride / 4;
  const float4* s4 = reinterpret_cast<const float4*>(src);
  for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < nv; x += (long long)gridDim.x * blockDim.x) {
    float4 v = __ldcg(s4 + x);
    int k = 1;
    for (; k + 3 < S; k += 4) {
      const float4 a = __ldcg(s4 + x + k * sv), b = __ldcg(s4 + x + (k + 1) * sv);
      const float4 c = __ldcg(s4 + x + (k + 2) * sv), d = __ldcg(s4 + x + (k + 3) * sv);
      v.x += a.x; v.y += a.y; v.z += a.z; v.w += a.w;
      v.x += b.x; v.y += b.y; v.z += b.z; v.w += b.w;
      v.x += c.x; v.y += c.y; v.z += c.z; v.w += c.w;
      v.x += d.x; v.y += d.y; v.z += d.z; v.w += d.w;
    }
    for (; k < S; k++) {
      const float4 a = __ldcg(s4 + x + k * sv);
      v.x += a.x; v.y += a.y; v.z += a.z; v.w += a.w;
    }
    reinterpret_cast<float4*>(dst)[x] = v;
  }
}

// Q^T split into hi / lo (tf32 split as above), K-major for the B operand:
// th[k][c] = hi(Q[c][k]), tl[k][c] = lo(Q[c][k]), row stride ldt.
__global__ void occ_split_t_kernel(const float* __restrict__ Q, int m, int R, unsigned* th, unsigned* tl, int ldt) {
  __shared__ float tile[32][33];
  const int c0 = blockIdx.x * 32;
  for (int k0 = 0; k0 < R; k0 += 32) {
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
      const int c = c0 + i, k = k0 + threadIdx.x;
      tile[i][threadIdx.x] = (c < m && k < R) ? Q[(size_t)c * R + k] : 0.f;
    }
    __syncthreads();
    for (int kk = threadIdx.y; kk < 32; kk += blockDim.y) {
      const int k = k0 + kk, c = c0 + threadIdx.x;
      if (k < R && c < ldt) {
        const float x = tile[threadIdx.x][kk];
        const unsigned h = __float_as_uint(x) & 0xffffe000u;
        th[(size_t)k * ldt + c] = h;
        tl[(size_t)k * ldt + c] = __float_as_uint(x - __uint_as_float(h));
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ host
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// fp32 rows x cols (row stride ld elements), box box_cols x box_rows, 128-B swizzle, OOB zero fill
static bool tmap_f32(CUtensorMap* tm, const void* ptr, uint64_t rows, uint64_t cols, uint64_t ld, uint32_t box_cols,
                     uint32_t box_rows, CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 4};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t es[2] = {1, 1};
  return fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static int sm_count() {
  static int c = 0;
  if (!c) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev);
    if (c <= 0) c = 148;
  }
  return c;
}

bool umma_enabled() {
  const char* e = getenv("OCC_UMMA");
  return !(e && e[0] == '0');
}

// Splits per band: the smallest G in [1, max_splits] (at most one 32-wide K
// chunk each) whose bands * G items keep the persistent grid >= 90 % busy in
// its last round (fewer partials for the reduction that follows), else the
// best-filling G.
static int choose_splits(int bands, int nk, int max_splits, int sms) {
  int best = 1;
  double best_eff = 0.0;
  const int gmax = std::max(1, std::min({max_splits, nk, 4 * sms}));
  for (int G = 1; G <= gmax; G++) {
    const long long items = (long long)bands * G;
    const long long rounds = (items + sms - 1) / sms;
    const double eff = (double)items / (double)(rounds * sms);
    if (eff >= 0.9) return G;
    if (eff > best_eff) { best_eff = eff; best = G; }
  }
  return best;
}

// T = false: sweep 1 over M (n x m): P_part[G][n][R] = (M + e) Q_prev.
// T = true: sweep 2: Q_part[G][m][R] = (M + e)^T F with F = p.P (n x R).
template <int R, bool T>
static cudaError_t launch_sweep(const Params& p, int max_splits, int* G_out, cudaStream_t st) {
  using C = Cfg1<R>;
  const int n = p.n, m = p.m;
  const int klen = T ? n : m;                         // contraction length
  const int ldt = (klen + 31) / 32 * 32;
  unsigned* th = reinterpret_cast<unsigned*>(p.Qt);
  unsigned* tl = th + (size_t)R * ldt;
  const float* F = T ? p.P : p.Qprev;                  // klen x R
  occ_split_t_kernel<<<ldt / 32, dim3(32, 8), 0, st>>>(F, klen, R, th, tl, ldt);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  CUtensorMap tmM, tmE, tmQh, tmQl;
  const uint32_t box_rows = T ? KC : BM;
  const CUtensorMapSwizzle sw = T ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B;
  if (!tmap_f32(&tmM, p.M, n, m, p.ldm, KC, box_rows, sw)) return cudaErrorNotSupported;
  if (p.err_in) {
    if (!tmap_f32(&tmE, p.err_in, n, m, p.lde_in, KC, box_rows, sw)) return cudaErrorNotSupported;
  } else {
    tmE = tmM;
  }
  if (!tmap_f32(&tmQh, th, R, klen, ldt, KC, R) || !tmap_f32(&tmQl, tl, R, klen, ldt, KC, R))
    return cudaErrorNotSupported;
  S1Args a;
  a.n = n;
  a.m = m;
  a.nrb = ((T ? m : n) + BM - 1) / BM;
  a.nkc = (klen + KC - 1) / KC;
  const int sms = sm_count();
  a.G = choose_splits(a.nrb, a.nkc, max_splits, sms);
  if (const char* km = getenv("OCC_UMMA_KMAX")) {   // experiment knob: at most KMAX contraction terms per split
    const int kmax = std::max(32, atoi(km));
    a.G = std::min(std::max(a.G, (klen + kmax - 1) / kmax), std::max(1, std::min(max_splits, a.nkc)));
  }
  a.has_e = p.err_in != nullptr;
  a.P_part = T ? p.Q_part : p.P_part;
  const int grid = std::min(a.nrb * a.G, sms);
  auto kern = umma_sweep_kernel<R, T>;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  if (e != cudaSuccess) return e;
  kern<<<grid, NTH, C::SMEM, st>>>(tmM, tmE, tmQh, tmQl, a);
  e = cudaGetLastError();
  if (e == cudaSuccess) *G_out = a.G;
  return e;
}

// The DP reconstruction (phase F of occ_allreduce_factors, plain or
// OCC_ORIENT_T) on tcgen05: the factor operands split into the Qt workspace,
// then one persistent launch.
template <int R>
static cudaError_t launch_recon(const Params& p, cudaStream_t st) {
  const int n = p.n, m = p.m;
  const bool rowloc = p.Pstate_out != nullptr;   // OCC_ORIENT_T (phase_F_tc's convention)
  const bool dpl = p.dp_local_err != 0;
  if (dpl && rowloc && !p.Ploc) return cudaErrorNotSupported;
  const float* c1 = p.Qrec;
  const float* r1 = p.P;
  const float* c2 = (dpl && !rowloc) ? p.Qloc : nullptr;
  const float* r2 = (dpl && rowloc) ? p.Ploc : nullptr;
  unsigned* c1h = reinterpret_cast<unsigned*>(p.Qt);
  unsigned* c1l = c1h + (size_t)m * R;
  unsigned* c2h = c1l + (size_t)m * R;
  unsigned* c2l = c2h + (size_t)m * R;
  unsigned* r1h = c2l + (size_t)m * R;
  unsigned* r1l = r1h + (size_t)n * R;
  unsigned* r2h = r1l + (size_t)n * R;
  unsigned* r2l = r2h + (size_t)n * R;
  SplitJobs jobs;
  jobs.n = 0;
  long long most = 0;
  auto add = [&](const float* x, long long rows, float scale, unsigned* hi, unsigned* lo, float* state) {
    jobs.j[jobs.n++] = SplitJob{x, rows * R, scale, hi, lo, state};
    most = std::max(most, rows * R);
  };
  add(c1, m, rowloc ? 1.f : p.scale, c1h, c1l, rowloc ? nullptr : p.Qstate_out);
  add(r1, n, rowloc ? p.scale : 1.f, r1h, r1l, rowloc ? p.Pstate_out : nullptr);
  if (c2) add(c2, m, 1.f, c2h, c2l, nullptr);
  if (r2) add(r2, n, 1.f, r2h, r2l, nullptr);
  occ_split_rows_kernel<<<(int)std::max<long long>(1, std::min<long long>((most + 255) / 256, 1184)), 256, 0, st>>>(jobs);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  CUtensorMap t[8];
  bool ok = tmap_f32(&t[0], c1h, m, R, R, 32, rc::BC) && tmap_f32(&t[1], c1l, m, R, R, 32, rc::BC) &&
            tmap_f32(&t[4], r1h, n, R, R, 32, rc::TR) && tmap_f32(&t[5], r1l, n, R, R, 32, rc::TR);
  t[2] = t[0]; t[3] = t[1]; t[6] = t[4]; t[7] = t[5];
  if (ok && c2) ok = tmap_f32(&t[2], c2h, m, R, R, 32, rc::BC) && tmap_f32(&t[3], c2l, m, R, R, 32, rc::BC);
  if (ok && r2) ok = tmap_f32(&t[6], r2h, n, R, R, 32, rc::TR) && tmap_f32(&t[7], r2l, n, R, R, 32, rc::TR);
  if (!ok) return cudaErrorNotSupported;
  RcArgs a;
  a.n = n;
  a.m = m;
  a.nb = (m + rc::BC - 1) / rc::BC;
  a.ntile = (n + rc::TR - 1) / rc::TR;
  const int sms = sm_count();
  a.G = choose_splits(a.nb, a.ntile, a.ntile, sms);
  a.dpl = dpl;
  a.has_e = p.err_in != nullptr;
  a.r_bf16 = p.r_bf16;
  a.M = static_cast<const float*>(p.M);
  a.ldm = p.ldm;
  a.E = p.err_in;
  a.lde = p.lde_in;
  a.out = p.recon;
  a.ldo = p.ldr;
  a.Eo = p.err_out;
  a.ldeo = p.lde_out;
  const bool two_c = c2 != nullptr, two_r = r2 != nullptr;
  const int smem = rc::Cfg<R>::smem(two_c, two_r);
  a.ns = rc::Cfg<R>::stages(two_c, two_r);
  if (a.ns < 2) return cudaErrorNotSupported;
  auto kern = two_c ? umma_recon_kernel<R, 1> : two_r ? umma_recon_kernel<R, 2> : umma_recon_kernel<R, 0>;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  kern<<<std::min(a.nb * a.G, sms), rc::NTH, smem, st>>>(t[0], t[1], t[2], t[3], t[4], t[5], t[6], t[7], a);
  return cudaGetLastError();
}

}  // namespace umma

// the sweeps: the small factor transposed, hi / lo (2 r x round32(max(n, m)));
// the DP reconstruction: up to two column and two row factors, hi / lo (4 r (n + m))
size_t umma_qt_bytes(int64_t n, int64_t m, int r) {
  return (4 * (size_t)(n + m) + 64) * (size_t)r * 4;
}

// count and stride are multiples of 4 (R >= 4 columns of fp32)
cudaError_t run_reduce_partials(const float* src, long long stride, int S, float* dst, long long count,
                                cudaStream_t st) {
  const long long nv = count / 4;
  const int grid = (int)std::max<long long>(1, std::min<long long>((nv + 255) / 256, 148 * 8));
  umma::occ_reduce_partials_kernel<<<grid, 256, 0, st>>>(src, stride, S, dst, count);
  return cudaGetLastError();
}

bool umma_applies(const Params& p, int r) {
  return umma::umma_enabled() && !p.m_bf16 && p.Qt && p.n >= 1 && p.m >= 1 && (r == 16 || r == 32 || r == 64);
}

// Sweep 1 (transposed = false) or sweep 2 (true) on the tcgen05 path when it
// applies (fp32 M, r in {16, 32, 64}, OCC_UMMA != 0); *G_out = the number of
// partials written (at most max_splits).  cudaErrorNotSupported: use the
// mma.sync sweep.
cudaError_t run_umma_sweep(const Params& p, int r, bool transposed, int max_splits, int* G_out, cudaStream_t st) {
  if (!umma_applies(p, r)) return cudaErrorNotSupported;
  switch (r) {
    case 16: return transposed ? umma::launch_sweep<16, true>(p, max_splits, G_out, st)
                               : umma::launch_sweep<16, false>(p, max_splits, G_out, st);
    case 32: return transposed ? umma::launch_sweep<32, true>(p, max_splits, G_out, st)
                               : umma::launch_sweep<32, false>(p, max_splits, G_out, st);
    case 64: return transposed ? umma::launch_sweep<64, true>(p, max_splits, G_out, st)
                               : umma::launch_sweep<64, false>(p, max_splits, G_out, st);
  }
  return cudaErrorNotSupported;
}

// Phase F of the DP paths (the occ_tc.cuh phase_F_tc definitions) on tcgen05
// when it applies (fp32 M, r in {32, 64}, OCC_UMMA != 0).
cudaError_t run_umma_recon(const Params& p, int r, cudaStream_t st) {
  if (!umma_applies(p, r)) return cudaErrorNotSupported;
  switch (r) {
    case 32: return umma::launch_recon<32>(p, st);
    case 64: return umma::launch_recon<64>(p, st);
  }
  return cudaErrorNotSupported;
}

}  // namespace occ
