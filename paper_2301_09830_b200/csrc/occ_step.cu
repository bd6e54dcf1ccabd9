// occ_step.cu -- kernel entry points and launch glue for one compression step.
// The phase bodies live in occ_kernels.cuh (see its header comment).
#include "occ_kernels.cuh"
#include "occ_internal.h"
#include "occ_tc.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>

namespace occ {

enum PhaseId { P_A = 0, P_B1 = 1, P_B2 = 2, P_C1 = 3, P_C2 = 4, P_C3 = 5, P_D = 6, P_E = 7, P_F = 8, P_END = 9 };

template <int R>
__host__ __device__ constexpr size_t orth_bytes() { return (sizeof(OrthSmem<R>) + 15) / 16 * 16; }

template <int R, bool DPL>
__global__ void __launch_bounds__(NT, 1) occ_step_kernel(const __grid_constant__ Params p, int ph0, int ph1, int coop) {
  extern __shared__ __align__(16) unsigned char smraw[];
  float* sm = reinterpret_cast<float*>(smraw);
  unsigned nb = 0;
  auto bar = [&]() { nb++; grid_barrier(p.bar, nb * gridDim.x); };
  const bool stamp = coop && blockIdx.x == 0 && threadIdx.x == 0;
  if (stamp) p.stats->t_ns[0] = gtimer();
  // a4 with the one-CTA factorisation (occ_kernels.cuh, fast orthonormalisation);
  // a degenerate column takes phases C1 / C2 / C3
  auto orth_fast = [&](bool do_reduce) {
    const int units = (p.n + B_ROWS - 1) / B_ROWS;
    phase_B_fast<R>(p, p.P, p.G_part, do_reduce, smraw);
    bar();
    OCC_STAMP(p, 9);
    if (blockIdx.x == 0) {
      const int plan = factor_fast<R>(p, p.G_part, true, true, smraw);
      if (threadIdx.x == 0) p.ctl[1] = plan;
    }
    bar();
    OCC_STAMP(p, 10);
    const int plan = __ldcg(p.ctl + 1);
    if (plan == 2) {
      OrthSmem<R>& o = *reinterpret_cast<OrthSmem<R>*>(smraw);
      float* ps = reinterpret_cast<float*>(smraw + orth_bytes<R>());
      int pl = phase_C1<R>(p, o, ps);
      if (pl == 2) { bar(); pl = phase_C2<R>(p, o, ps); }
      if (pl == 3) { bar(); phase_C3<R>(p, o, ps); }
      return;
    }
    if (plan == 3) {   // CholQR2: P_hat of the first pass and its Gram, a second factorisation
      for (int u = blockIdx.x; u < units; u += gridDim.x)
        apply_fast<R>(p, u * B_ROWS, min(p.n, (u + 1) * B_ROWS), smraw, p.G2_part);
      bar();
      if (blockIdx.x == 0) factor_fast<R>(p, p.G2_part, false, false, smraw);
      bar();
    }
    const int r0 = (int)((long long)blockIdx.x * p.n / gridDim.x);
    const int r1 = (int)((long long)(blockIdx.x + 1) * p.n / gridDim.x);
    apply_fast<R>(p, r0, r1, smraw, nullptr);
    OCC_STAMP(p, 11);
  };
  for (int ph = ph0; ph < ph1; ph++) {
    switch (ph) {
      case P_A:   // tensor-core sweep 1 (occ_tc.cuh)
        if (p.m_bf16) tc::phase_A_tc<R, true>(p, smraw);
        else tc::phase_A_tc<R, false>(p, smraw);
        break;
      case P_B1: {
        if (coop && p.fast_orth && ph1 > P_C3) {   // P reduce + Gram + orthonormalisation (orth_fast)
          orth_fast(true);
          ph = P_C3;
          break;
        }
        if (p.fast_orth && ph1 <= P_B2) {           // the P reduce alone, over every CTA
          reduce_p_all<R>(p);
          break;
        }
        const bool g = ph1 > P_B2;
        phase_B<R>(p, sm, true, g);
        if (g) ph = P_B2;
        break;
      }
      case P_B2:
        if (coop && p.fast_orth && ph1 > P_C3) {
          orth_fast(false);
          ph = P_C3;
          break;
        }
        phase_B<R>(p, sm, false, true);
        break;
      case P_C1: {
        OrthSmem<R>& o = *reinterpret_cast<OrthSmem<R>*>(smraw);
        float* ps = reinterpret_cast<float*>(smraw + orth_bytes<R>());
        int plan = phase_C1<R>(p, o, ps);
        if (coop) {
          if (plan == 2) { bar(); plan = phase_C2<R>(p, o, ps); }
          if (plan == 3) { bar(); phase_C3<R>(p, o, ps); }
          ph = P_C3;
        }
        break;
      }
      case P_C2: {
        OrthSmem<R>& o = *reinterpret_cast<OrthSmem<R>*>(smraw);
        float* ps = reinterpret_cast<float*>(smraw + orth_bytes<R>());
        if (__ldcg(p.ctl) == 2) phase_C2<R>(p, o, ps);
        break;
      }
      case P_C3: {
        OrthSmem<R>& o = *reinterpret_cast<OrthSmem<R>*>(smraw);
        float* ps = reinterpret_cast<float*>(smraw + orth_bytes<R>());
        if (__ldcg(p.ctl) == 3) phase_C3<R>(p, o, ps);
        break;
      }
      case P_D:   // tensor-core sweep 2 (occ_tc.cuh)
        if (p.m_bf16) tc::phase_D_tc<R, true>(p, smraw);
        else tc::phase_D_tc<R, false>(p, smraw);
        break;
      case P_E: phase_E<R>(p); break;
      case P_F:
        if (p.f_tc) {   // the DP reconstruction (occ_tc.cuh), plain or OCC_ORIENT_T
          if (p.m_bf16) tc::phase_F_tc<R, DPL, true>(p, smraw);
          else tc::phase_F_tc<R, DPL, false>(p, smraw);
        } else {
          phase_F<R, DPL>(p, sm);
        }
        break;
      default: break;
    }
    if (ph + 1 < ph1) bar();
    if (stamp && ph + 1 < 12) p.stats->t_ns[ph + 1] = gtimer();
  }
  if (coop) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned old = atomicAdd(p.bar + 1, 1u);
      if (old == gridDim.x - 1) {
        atomicExch(p.bar, 0u);
        atomicExch(p.bar + 1, 0u);
      }
    }
  }
  // stamped by the launch that ends the step's v1 part: phase F, or phase E when
  // F runs in the v2 reconstruct kernel (occ_api.cu reconstruct)
  if (blockIdx.x == 0 && threadIdx.x == 0 && ph0 <= P_F && P_E < ph1) {
    p.stats->path = p.path;
    p.stats->grid = gridDim.x;
    p.stats->q_amp = -1.0;
    p.stats->q_fused = 0;
  }
}

// ------------------------------------------------------------------ sizes
template <int R>
static size_t smem_bytes_for(const Geometry& g) {
  size_t a = tc::smem_A_tc<R>(g.cs1);
  size_t b = (size_t)B_ROWS * R * 4;
  size_t c = orth_bytes<R>() + 2 * (size_t)B_ROWS * R * 4;
  size_t d = tc::smem_D_tc<R>(g.rs2);
  size_t f = std::max(2 * (size_t)F_ROWS * R * 4,   // P rows + Ploc rows (DP, OCC_ORIENT_T)
                      tc::smem_F_tc<R>());
  return std::max({a, b, c, d, f, smem_fast_orth<R>()});
}

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
  L.qt = off; off = al(off + umma_qt_bytes(g.n, g.m, R));
  L.li = off; off = al(off + (size_t)R * R * 8);               // Li of the one-CTA factorisation   // tcgen05 sweeps: Q^T / P_hat^T split hi / lo
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
  static const bool fast = [] {
    const char* e = getenv("OCC_FAST_ORTH");
    return !(e && e[0] == '0');
  }();
  p.fast_orth = fast ? 1 : 0;
  p.s1 = g.s1; p.cs1 = g.cs1; p.s2 = g.s2; p.rs2 = g.rs2; p.ngp = g.ngp;
}

// Launch phases [ph0, ph1) of one step.  coop: one cooperative persistent
// launch (grid = co-resident CTAs); otherwise one launch per phase group.
template <int R, bool DPL>
static cudaError_t run_t(Params p, const Geometry& g, int ph0, int ph1, bool multi, cudaStream_t st) {
  if (ph0 == P_A && ph1 > P_A && umma_applies(p, R)) {   // sweep 1 on the tcgen05 path (occ_umma.cu)
    int G = 0;
    const cudaError_t eu = run_umma_sweep(p, R, false, g.s1, &G, st);
    if (eu == cudaSuccess) {
      p.s1 = G;
      ph0 = P_B1;
      if (ph0 >= ph1) return cudaSuccess;
    } else if (eu != cudaErrorNotSupported) {
      return eu;
    }
  }
  if (ph0 <= P_D && P_D < ph1 && umma_applies(p, R)) {   // sweep 2 on the tcgen05 path
    if (ph0 < P_D) {
      const cudaError_t e0 = run_t<R, DPL>(p, g, ph0, P_D, multi, st);
      if (e0 != cudaSuccess) return e0;
      ph0 = P_D;
    }
    int G = 0;
    const cudaError_t eu = run_umma_sweep(p, R, true, g.s2, &G, st);
    if (eu == cudaSuccess) {
      p.s2 = G;
      ph0 = P_E;
      if (ph0 >= ph1) return cudaSuccess;
    } else if (eu != cudaErrorNotSupported) {
      return eu;
    }
  }
  if (ph0 == P_F && ph1 == P_END && p.f_tc && umma_applies(p, R)) {   // the DP reconstruction on tcgen05
    const cudaError_t eu = run_umma_recon(p, R, st);
    if (eu != cudaErrorNotSupported) return eu;
  }
  auto kern = occ_step_kernel<R, DPL>;
  const size_t smem = smem_bytes_for<R>(g);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int sms = num_sms();
  if (!multi) {
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    per_sm = std::min(per_sm, 2);
    const int grid = sms * per_sm;
    p.path = 1;
    int coop = 1;
    void* args[] = {&p, &ph0, &ph1, &coop};
    return cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(NT), args, smem, st);
  }
  p.path = 2;
  // per-phase launches; grid = units of the phase (bounded)
  auto units = [&](int ph) -> int {
    const int64_t n = g.n, m = g.m;
    switch (ph) {
      case P_A: return (int)(((n + tc::TcCfg<R>::A_ROWS - 1) / tc::TcCfg<R>::A_ROWS) * g.s1);
      case P_B1: case P_B2: case P_C1: case P_C2: case P_C3: return g.ngp;
      case P_D: return (int)(((m + tc::TcCfg<R>::D_COLS - 1) / tc::TcCfg<R>::D_COLS) * g.s2);
      case P_E: return (int)((m + 31) / 32);
      case P_F:
        if (p.f_tc) return (int)(((m + tc::F_TC_COLS - 1) / tc::F_TC_COLS) * ((n + tc::F_TC_ROWS - 1) / tc::F_TC_ROWS));
        return (int)(((m + CfgF<R, DPL>::CB - 1) / CfgF<R, DPL>::CB) * ((n + F_ROWS - 1) / F_ROWS));
    }
    return 1;
  };
  for (int ph = ph0; ph < ph1; ph++) {
    int hi = ph + 1;
    if (ph == P_B1 && ph1 > P_B2) hi = P_B2 + 1;
    const int grid = std::max(1, std::min(units(ph), sms * 16));
    kern<<<grid, NT, smem, st>>>(p, ph, hi, 0);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    ph = hi - 1;
  }
  return cudaSuccess;
}

cudaError_t run_phases(const Params& p, const Geometry& g, int ph0, int ph1, bool multi, bool dpl,
                       cudaStream_t st) {
  switch (g.r) {
#define OCC_CASE(RR)                                                              \
  case RR:                                                                        \
    return dpl ? run_t<RR, true>(p, g, ph0, ph1, multi, st)                       \
               : run_t<RR, false>(p, g, ph0, ph1, multi, st);
    OCC_CASE(4) OCC_CASE(8) OCC_CASE(16) OCC_CASE(32) OCC_CASE(64)
#undef OCC_CASE
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

// OCC_CHECK_FINITE: read and clear this device's v1 status word.
unsigned take_nonfinite_v1() {
  unsigned v = 0, z = 0;
  if (cudaMemcpyFromSymbol(&v, g_nonfinite_v1, sizeof v) != cudaSuccess) return 0;
  if (v) cudaMemcpyToSymbol(g_nonfinite_v1, &z, sizeof z);
  return v;
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
