// occ_step.cu -- geometry, workspace layout and launch glue of one compression
// step; the per-phase step kernels are in occ_step_impl.cuh (one translation
// unit per rank: occ_step_r{4..64}.cu), the phase bodies in occ_kernels.cuh.
#include "occ_kernels.cuh"
#include "occ_internal.h"
#include "occ_tc.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>

namespace occ {

static int num_sms() {
  static int cached = 0;
  if (!cached) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
    if (cached <= 0) cached = 148;
  }
  return cached;
}

Geometry make_geometry(int64_t n, int64_t m, int r, int sms) {
  Geometry g;
  g.n = n; g.m = m; g.r = r;
  const int ur = (r <= 32) ? 64 : 32;
  const int64_t nrb = (n + ur - 1) / ur;
  int64_t cs1 = (m * nrb) / (2 * (int64_t)sms);
  cs1 = cs1 / 8 * 8;
  const int64_t cmax = (r <= 16) ? 512 : 256;
  cs1 = std::max<int64_t>(64, std::min<int64_t>(cmax, cs1));
  cs1 = std::min<int64_t>(cs1, (m + 7) / 8 * 8);
  g.cs1 = (int)cs1;
  g.s1 = (int)((m + cs1 - 1) / cs1);
  g.rs2 = 256;   // rows per sweep-2 split: Q_part holds s2 = n / 256 partials
  g.s2 = (int)((n + g.rs2 - 1) / g.rs2);
  g.ngp = (int)((n + B_ROWS - 1) / B_ROWS);
  return g;
}

static size_t al(size_t x) { return (x + 255) / 256 * 256; }

// max over n' <= n, m' <= m (m' % 8 == 0) of s1(n', m') * n' (see make_layout)
static size_t max_sweep1_rows(int64_t n, int64_t m, int r) {
  const int ur = (r <= 32) ? 64 : 32;
  size_t best = 0;
  for (int64_t nb = 1; (nb - 1) * ur < n; nb++) {
    const int64_t nn = std::min<int64_t>(nb * ur, n);
    for (int64_t mm = 8; mm <= m; mm += 8) {
      const Geometry g = make_geometry(nn, mm, r, 148);
      best = std::max(best, (size_t)g.s1 * (size_t)nn);
    }
  }
  return best;
}

WsLayout make_layout(const Geometry& g, int nmat) {
  WsLayout L;
  const int R = g.r;
  const size_t np = (size_t)R * (R + 1) / 2;
  size_t off = 0;
  L.bar = off; off += 256;                                 // bar[2], ctl[4], stats
  off += kTraceBytes;                                      // per-CTA phase trace (occ_read_trace)
  off += kBarLinesBytes;                                   // v2 grid-barrier arrival lines
  // A bucket (nmat > 1) holds matrices of at most n x m; each one's sweep-1
  // partials need s1_i * n_i rows, which can exceed s1 * n of the largest
  // shape (s1 grows as a matrix gets shorter), so take the maximum over every
  // shape the bucket may hold (s1 depends on the rows only through the row
  // block count, and cols are multiples of 8).
  size_t prows = (size_t)g.s1 * g.n;
  if (nmat > 1) prows = std::max(prows, max_sweep1_rows(g.n, g.m, R));
  L.p_part = off; off = al(off + prows * R * 4);
  L.q_part = off; off = al(off + (size_t)g.s2 * g.m * R * 4);
  // Gram partials: per 128 rows of the orthonormalised factor, which is the
  // row side (n) or, with OCC_ORIENT_T, the column side (m)
  const size_t ngp = std::max<size_t>(g.ngp, (size_t)((g.m + B_ROWS - 1) / B_ROWS));
  L.g_part = off; off = al(off + ngp * np * 8);
  L.g2_part = off; off = al(off + ngp * np * 8);
  L.xy_part = off; off = al(off + ngp * 2 * R * R * 8);
  L.p_bucket = off; off = al(off + (size_t)nmat * g.n * R * 4);
  L.qw_bucket = off; off = al(off + (size_t)nmat * g.m * R * 4);
  L.qs_bucket = off; off = al(off + (size_t)nmat * std::max(g.n, g.m) * R * 4);   // reduced Q (or V, OCC_ORIENT_T)
  L.qt = off; off = al(off + umma_qt_bytes(g.n, g.m, R));      // tcgen05 kernels: split, transposed factors
  L.li = off; off = al(off + (size_t)R * R * 8);               // Li of the one-CTA factorisation
  L.gred = off; off = al(off + np * 8);                        // its reduced Gram
  L.v2_tail_bytes = v2_tail_bytes(g.n, g.m, R, 148);   // reused by every matrix of a multi-matrix call
  L.v2_tail = off; off = al(off + L.v2_tail_bytes);
  L.total = off;
  return L;
}

void fill_ws(Params& p, const Geometry& g, const WsLayout& L, void* ws) {
  char* base = static_cast<char*>(ws);
  p.bar = reinterpret_cast<unsigned*>(base + L.bar);
  p.ctl = reinterpret_cast<int*>(base + L.bar + 16);
  p.stats = reinterpret_cast<DevStats*>(base + L.bar + 64);
  p.P_part = reinterpret_cast<float*>(base + L.p_part);
  p.Q_part = reinterpret_cast<float*>(base + L.q_part);
  p.G_part = reinterpret_cast<double*>(base + L.g_part);
  p.G2_part = reinterpret_cast<double*>(base + L.g2_part);
  p.XY_part = reinterpret_cast<double*>(base + L.xy_part);
  p.Qt = reinterpret_cast<float*>(base + L.qt);
  p.Li_g = reinterpret_cast<double*>(base + L.li);
  p.G_red = reinterpret_cast<double*>(base + L.gred);
  static const bool fast = [] {
    const char* e = getenv("OCC_FAST_ORTH");
    return !(e && e[0] == '0');
  }();
  p.fast_orth = fast ? 1 : 0;
  p.s1 = g.s1; p.cs1 = g.cs1; p.s2 = g.s2; p.rs2 = g.rs2; p.ngp = g.ngp;
}

cudaError_t run_phases(const Params& p, const Geometry& g, int ph0, int ph1, bool multi, bool dpl,
                       cudaStream_t st) {
  switch (g.r) {
    case 4: return run_phases_r4(p, g, ph0, ph1, multi, dpl, st);
    case 8: return run_phases_r8(p, g, ph0, ph1, multi, dpl, st);
    case 16: return run_phases_r16(p, g, ph0, ph1, multi, dpl, st);
    case 32: return run_phases_r32(p, g, ph0, ph1, multi, dpl, st);
    case 64: return run_phases_r64(p, g, ph0, ph1, multi, dpl, st);
  }
  return cudaErrorInvalidValue;
}

// ------------------------------------------------------------------ decompress
// out = round(P Q^T): a standalone phase F with no residual (receiver side).
template <int R>
__global__ void __launch_bounds__(NT) occ_decompress_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(16) unsigned char smraw[];
  phase_F<R, false>(p, reinterpret_cast<float*>(smraw));
}

cudaError_t run_decompress(const Params& p, int r, cudaStream_t st) {
  const int sms = num_sms();
  switch (r) {
#define OCC_DCASE(RR)                                                                       \
  case RR: {                                                                                \
    const size_t smem = (size_t)F_ROWS * RR * 4;                                            \
    const int units = (int)(((p.m + CfgF<RR, false>::CB - 1) / CfgF<RR, false>::CB) *       \
                            ((p.n + F_ROWS - 1) / F_ROWS));                                 \
    occ_decompress_kernel<RR><<<std::max(1, std::min(units, sms * 8)), NT, smem, st>>>(p); \
    return cudaGetLastError();                                                              \
  }
    OCC_DCASE(4) OCC_DCASE(8) OCC_DCASE(16) OCC_DCASE(32) OCC_DCASE(64)
#undef OCC_DCASE
  }
  return cudaErrorInvalidValue;
}

// OCC_CHECK_FINITE: read and clear this device's v1 status words (one per
// translation unit holding step kernels)
unsigned take_nonfinite_v1() {
  return take_nonfinite_v1_r4() | take_nonfinite_v1_r8() | take_nonfinite_v1_r16() | take_nonfinite_v1_r32() |
         take_nonfinite_v1_r64();
}

// ------------------------------------------------------------------ bf16 wire (OCC_WIRE_BF16)
__global__ void occ_round_bf16_kernel(float* x, long long count) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count; i += (long long)gridDim.x * blockDim.x)
    x[i] = __bfloat162float(__float2bfloat16_rn(x[i]));
}
__global__ void occ_pack_bf16_kernel(const float* x, __nv_bfloat16* y, long long count) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count; i += (long long)gridDim.x * blockDim.x)
    y[i] = __float2bfloat16_rn(x[i]);
}
__global__ void occ_unpack_bf16_kernel(const __nv_bfloat16* y, float* x, long long count) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count; i += (long long)gridDim.x * blockDim.x)
    x[i] = __bfloat162float(y[i]);
}
static int grid_for(long long count) { return (int)std::max<long long>(1, std::min<long long>((count + 255) / 256, 4096)); }
cudaError_t run_round_bf16(float* x, long long count, cudaStream_t st) {
  occ_round_bf16_kernel<<<grid_for(count), 256, 0, st>>>(x, count);
  return cudaGetLastError();
}
cudaError_t run_pack_bf16(const float* x, void* y, long long count, cudaStream_t st) {
  occ_pack_bf16_kernel<<<grid_for(count), 256, 0, st>>>(x, static_cast<__nv_bfloat16*>(y), count);
  return cudaGetLastError();
}
cudaError_t run_unpack_bf16(const void* y, float* x, long long count, cudaStream_t st) {
  occ_unpack_bf16_kernel<<<grid_for(count), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(y), x, count);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ init_q
__global__ void occ_init_q_kernel(float* q, long long rows, int r, long long ld, unsigned long long seed) {
  const long long total = rows * r;
  for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < total;
       x += (long long)gridDim.x * blockDim.x) {
    const long long i = x / r, k = x % r;
    // Box-Muller on two splitmix64 uniforms keyed by (seed, element).
    auto mix = [](unsigned long long z) {
      z += 0x9E3779B97F4A7C15ull;
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
      return z ^ (z >> 31);
    };
    const unsigned long long h1 = mix(seed ^ (2ull * (unsigned long long)x));
    const unsigned long long h2 = mix(seed ^ (2ull * (unsigned long long)x + 1ull));
    const double u1 = ((double)(h1 >> 11) + 0.5) * (1.0 / 9007199254740992.0);
    const double u2 = (double)(h2 >> 11) * (1.0 / 9007199254740992.0);
    q[i * ld + k] = (float)(sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2));
  }
}

cudaError_t run_init_q(float* q, int64_t rows, int r, int64_t ld, uint64_t seed, cudaStream_t st) {
  const long long total = rows * r;
  const int grid = (int)std::min<long long>((total + 255) / 256, 4096);
  occ_init_q_kernel<<<std::max(grid, 1), 256, 0, st>>>(q, rows, r, ld, seed);
  return cudaGetLastError();
}

}  // namespace occ
