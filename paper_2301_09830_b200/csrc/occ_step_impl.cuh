// occ_step_impl.cuh -- the per-phase step kernel (occ_step_kernel<R, DPL>) and
// its launch glue (run_t), compiled once per rank R by occ_step_r{4..64}.cu so
// that the instantiations build in parallel.  The phase bodies live in
// occ_kernels.cuh (see its header comment).
#pragma once
#include "occ_kernels.cuh"
#include "occ_internal.h"
#include "occ_tc.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>

namespace occ {
namespace {

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
    if (do_reduce) {   // P = sum of the sweep-1 partials over every CTA, then the Gram per unit
      reduce_p_all<R>(p);
      bar();
    }
    phase_B_fast<R>(p, p.P, p.G_part, smraw);
    bar();
    reduce_gram_all<R>(p.G_part, units, p.G_red);
    bar();
    OCC_STAMP(p, 9);
    if (blockIdx.x == 0) {
      const int plan = factor_fast<R>(p, p.G_red, 1, true, true, smraw);
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
    const int r0 = (int)((long long)blockIdx.x * p.n / gridDim.x);
    const int r1 = (int)((long long)(blockIdx.x + 1) * p.n / gridDim.x);
    if (plan == 3) {   // CholQR2: P_hat of the first pass (every CTA), its Gram per unit, a second factorisation
      apply_fast<R>(p, r0, r1, smraw, nullptr);
      bar();
      phase_B_fast<R>(p, p.P, p.G2_part, smraw);
      bar();
      reduce_gram_all<R>(p.G2_part, units, p.G_red);
      bar();
      if (blockIdx.x == 0) factor_fast<R>(p, p.G_red, 1, false, false, smraw);
      bar();
    }
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
  // (P_D == ph1: the orthonormalisation launch before a tcgen05 sweep 2, whose
  // Q reduce is a plain launch)
  if (blockIdx.x == 0 && threadIdx.x == 0 && ph0 <= P_F && (P_E < ph1 || ph1 == P_D)) {
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

int num_sms() {
  static int cached = 0;
  if (!cached) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
    if (cached <= 0) cached = 148;
  }
  return cached;
}

// Launch phases [ph0, ph1) of one step.  coop: one cooperative persistent
// launch (grid = co-resident CTAs); otherwise one launch per phase group.
template <int R, bool DPL>
cudaError_t run_t(Params p, const Geometry& g, int ph0, int ph1, bool multi, cudaStream_t st) {
  if (ph0 == P_A && ph1 > P_A && umma_applies(p, R)) {   // sweep 1 on the tcgen05 path (occ_umma.cu)
    int G = 0;
    const cudaError_t eu = run_umma_sweep(p, R, false, g.s1, &G, st);
    if (eu == cudaSuccess) {
      p.s1 = G;
      ph0 = P_B1;
      if (ph0 >= ph1) return cudaSuccess;
      if (ph1 <= P_B2)   // the P reduce alone (the DP path): a plain launch
        return run_reduce_partials(p.P_part, (long long)p.n * R, G, p.P, (long long)p.n * R, st);
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
      // the Q reduce (phase E) as a plain launch
      const cudaError_t er = run_reduce_partials(p.Q_part, (long long)p.m * R, G, p.Qloc, (long long)p.m * R, st);
      if (er != cudaSuccess) return er;
      ph0 = P_F;
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

}  // namespace

// entry points of one rank's translation unit (declared in occ_internal.h)
#define OCC_STEP_INSTANCE(RR)                                                                          \
  cudaError_t run_phases_r##RR(const Params& p, const Geometry& g, int ph0, int ph1, bool multi,       \
                               bool dpl, cudaStream_t st) {                                            \
    return dpl ? run_t<RR, true>(p, g, ph0, ph1, multi, st) : run_t<RR, false>(p, g, ph0, ph1, multi, st); \
  }                                                                                                    \
  unsigned take_nonfinite_v1_r##RR() {                                                                 \
    unsigned v = 0, z = 0;                                                                             \
    if (cudaMemcpyFromSymbol(&v, g_nonfinite_v1, sizeof v) != cudaSuccess) return 0;                   \
    if (v) cudaMemcpyToSymbol(g_nonfinite_v1, &z, sizeof z);                                           \
    return v;                                                                                          \
  }

}  // namespace occ
