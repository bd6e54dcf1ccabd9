// occ_umma.cu -- 5th-generation tensor-core (tcgen05) sweep of the per-phase
// path: sweep 1, P_part = (M + e) Q_prev (north_star a1, a2; PAPER.md:269-270,
// the PowerSGD power iteration P = M Q), for the shapes the fused kernel does
// not hold on chip (BASELINE configs[2], configs[3]: r = 32, 64).
//
// One persistent CTA per SM, warp-specialised:
//   warp 0      TMA producer: 2-D tensor-map loads (cp.async.bulk.tensor, 128-B
//               swizzle) of a 128-row x 32-column box of M and of e, and of the
//               32-column slices of Q_prev^T split into hi / lo (the small
//               factor, pre-split and transposed once per step by
//               occ_split_t_kernel), into an mbarrier ring of stages.
//   warps 2..5  converters: A = M + e and the 3-term TF32 split A = A_hi + A_lo
//               (hi: the low 13 mantissa bits masked off, lo = A - hi exact in
//               fp32), in place (A_hi over the M box, A_lo over the e box) --
//               elementwise, so the swizzled layout TMA wrote is kept as is.
//   warp 1      MMA issuer (one thread): per stage and per 8-column K step,
//               tcgen05.mma.kind::tf32 A_lo.Q_hi + A_hi.Q_lo + A_hi.Q_hi
//               (fp32-level accuracy, as the mma.sync sweeps) into a 128 x R
//               fp32 accumulator in TENSOR MEMORY; tcgen05.commit frees the
//               stage back to the producer.
//   epilogue    the converter warps read the accumulator (tcgen05.ld, lane =
//               row) and store the band's partial P rows.
//
// Work split: a row band of 128 rows is shared by G CTAs, each owning a
// contiguous range of 32-column chunks, so the partial count is G (about
// 148 / bands), not m / 256 -- the P reduce that follows reads G partials.
// Both operands are K-major with the 128-B swizzle: 8-row core groups 1024 B
// apart (SBO), the K step of 8 tf32 = 32 B inside the swizzle row.
#include "occ_internal.h"
#include "occ_kernels.cuh"
#include "occ_v2.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

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
  int nrb, G, nkc;   // row bands, CTAs per band, 32-column chunks
  int has_e;
  float* P_part;     // [G][n][R]
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
// instruction descriptor: D f32, A / B tf32, both K-major, M = 128, N
__host__ __device__ constexpr uint32_t idesc_tf32(int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
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

template <int R>
__global__ void __launch_bounds__(NTH, 1)
    umma_sweep1_kernel(const __grid_constant__ CUtensorMap tmM, const __grid_constant__ CUtensorMap tmE,
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
      mbar_init(&conv[s], NCV);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; b++) {
      mbar_init(&accf[b], 1);
      mbar_init(&acce[b], NCV);
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
          tma_2d(stM(s), &tmM, c * KC, band * BM, &full[s], pol_stream);
          if (a.has_e) tma_2d(stE(s), &tmE, c * KC, band * BM, &full[s], pol_stream);
          tma_2d(stQh(s), &tmQh, c * KC, 0, &full[s], pol_keep);
          tma_2d(stQl(s), &tmQl, c * KC, 0, &full[s], pol_keep);
          if (++s == NS) { s = 0; ph ^= 1u; }
        }
      }
    }
  } else if (w == 1) {
    if (lane == 0) {   // ------------------------------------------------ MMA issuer
      constexpr uint32_t idesc = idesc_tf32(N);
      int s = 0;
      unsigned ph = 0, aph[2] = {0u, 0u};
      int k = 0;
      for (int it = blockIdx.x; it < items; it += gridDim.x, k++) {
        int band, gi, c_lo, c_hi;
        range(it, band, gi, c_lo, c_hi);
        const int ab = k & 1;
        mbar_wait(&acce[ab], aph[ab] ^ 1u);   // the epilogue has drained this accumulator
        aph[ab] ^= 1u;
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const unsigned td = tbase + (unsigned)(ab * N);
        for (int c = c_lo; c < c_hi; c++) {
          mbar_wait(&conv[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t dh = desc_k_sw128(smem_u32(stM(s))), dl = desc_k_sw128(smem_u32(stE(s)));
          const uint64_t qh = desc_k_sw128(smem_u32(stQh(s))), ql = desc_k_sw128(smem_u32(stQl(s)));
#pragma unroll
          for (int kk = 0; kk < KC / 8; kk++) {
            const uint64_t o = (uint64_t)(2 * kk);   // 32 B per K step, in 16-B units
            mma_tf32(td, dl + o, qh + o, idesc, (c > c_lo || kk > 0) ? 1u : 0u);
            mma_tf32(td, dh + o, ql + o, idesc, 1u);
            mma_tf32(td, dh + o, qh + o, idesc, 1u);
          }
          mma_commit(&empty[s]);
          if (++s == NS) { s = 0; ph ^= 1u; }
        }
        mma_commit(&accf[ab]);
      }
    }
  } else {   // ------------------------------------------------------------ converters + epilogue
    const int ct = tid - 64;
    int s = 0;
    unsigned ph = 0, aph[2] = {0u, 0u};
    int k = 0;
    const int q = w & 3;   // TMEM lane quadrant of this warp
    for (int it = blockIdx.x; it < items; it += gridDim.x, k++) {
      int band, gi, c_lo, c_hi;
      range(it, band, gi, c_lo, c_hi);
      for (int c = c_lo; c < c_hi; c++) {
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
        mbar_arrive(&conv[s]);
        if (++s == NS) { s = 0; ph ^= 1u; }
      }
      // epilogue: row 32 q + lane of the band, R accumulator columns
      const int ab = k & 1;
      mbar_wait(&accf[ab], aph[ab]);
      aph[ab] ^= 1u;
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int row = band * BM + 32 * q + lane;
      const unsigned ta = tbase + ((unsigned)(32 * q) << 16) + (unsigned)(ab * N);
      float* dst = a.P_part + ((size_t)gi * a.n + row) * R;
#pragma unroll
      for (int j = 0; j < R / 16; j++) {
        float v[16];
        v2::tmem_ld16(ta + 16 * j, v);
        if (row < a.n) {
#pragma unroll
          for (int u = 0; u < 4; u++)
            reinterpret_cast<float4*>(dst + 16 * j)[u] = make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(&acce[ab]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (w == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(C::TCOLS));
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
                     uint32_t box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 4};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t es[2] = {1, 1};
  return fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
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

template <int R>
static cudaError_t launch_sweep1(const Params& p, int max_splits, int* G_out, cudaStream_t st) {
  using C = Cfg1<R>;
  const int n = p.n, m = p.m;
  const int ldt = (m + 31) / 32 * 32;
  unsigned* th = reinterpret_cast<unsigned*>(p.Qt);
  unsigned* tl = th + (size_t)R * ldt;
  occ_split_t_kernel<<<ldt / 32, dim3(32, 8), 0, st>>>(p.Qprev, m, R, th, tl, ldt);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  CUtensorMap tmM, tmE, tmQh, tmQl;
  if (!tmap_f32(&tmM, p.M, n, m, p.ldm, KC, BM)) return cudaErrorNotSupported;
  if (p.err_in) {
    if (!tmap_f32(&tmE, p.err_in, n, m, p.lde_in, KC, BM)) return cudaErrorNotSupported;
  } else {
    tmE = tmM;
  }
  if (!tmap_f32(&tmQh, th, R, m, ldt, KC, R) || !tmap_f32(&tmQl, tl, R, m, ldt, KC, R)) return cudaErrorNotSupported;
  S1Args a;
  a.n = n;
  a.m = m;
  a.nrb = (n + BM - 1) / BM;
  a.nkc = (m + KC - 1) / KC;
  const int sms = sm_count();
  a.G = (a.nrb >= sms) ? 1 : std::max(1, std::min({sms / a.nrb, a.nkc, max_splits}));
  a.has_e = p.err_in != nullptr;
  a.P_part = p.P_part;
  const int grid = std::min(a.nrb * a.G, sms);
  auto kern = umma_sweep1_kernel<R>;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  if (e != cudaSuccess) return e;
  kern<<<grid, NTH, C::SMEM, st>>>(tmM, tmE, tmQh, tmQl, a);
  e = cudaGetLastError();
  if (e == cudaSuccess) *G_out = a.G;
  return e;
}

}  // namespace umma

size_t umma_qt_bytes(int64_t n, int64_t m, int r) {
  const int64_t len = (std::max(n, m) + 31) / 32 * 32;
  return 2 * (size_t)r * (size_t)len * 4;
}

// Sweep 1 on the tcgen05 path when it applies (fp32 M, r in {16, 32, 64},
// OCC_UMMA != 0); *G_out = the number of partials written per row.
// cudaErrorNotSupported: use the mma.sync sweep.
cudaError_t run_umma_sweep1(const Params& p, int r, int max_splits, int* G_out, cudaStream_t st) {
  if (!umma::umma_enabled() || p.m_bf16 || !p.Qt) return cudaErrorNotSupported;
  if (p.n < 1 || p.m < 1) return cudaErrorNotSupported;
  switch (r) {
    case 16: return umma::launch_sweep1<16>(p, max_splits, G_out, st);
    case 32: return umma::launch_sweep1<32>(p, max_splits, G_out, st);
    case 64: return umma::launch_sweep1<64>(p, max_splits, G_out, st);
  }
  return cudaErrorNotSupported;
}

}  // namespace occ
