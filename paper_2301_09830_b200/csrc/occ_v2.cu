// occ_v2.cu -- kernel body and launcher of the TMEM-resident fused step
// (design in occ_v2.cuh).
#include "occ_v2.cuh"
#include "occ_internal.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>

namespace occ {
namespace v2 {

template <int R>
struct K {
  static constexpr int RP = R < 8 ? 8 : R;   // padded rank
  static constexpr int MT = (RP + 15) / 16;  // m-tiles of 16 over the rank
  static constexpr int KS5 = RP / 8;         // phase-5 k-steps
  static constexpr int NP = npairs(R);
};

struct OrthW {  // small fp64 linear algebra in shared memory
  double L[32 * 32];
  double Li[32 * 32];
  double X[32 * 32];
  double Y[32 * 32];
  double gdiag[32];
  int rep[32];
  int deg;
  double kappa;
};

__device__ __forceinline__ double shfl_d(double v, int src) {
  int lo = __double2loint(v), hi = __double2hiint(v);
  lo = __shfl_sync(0xffffffffu, lo, src);
  hi = __shfl_sync(0xffffffffu, hi, src);
  return __hiloint2double(hi, lo);
}

// G (packed upper triangle, nparts partials) -> o.L (full symmetric), o.gdiag.  All threads.
template <int R>
__device__ void reduce_partials(const double* __restrict__ part, int nparts, OrthW& o) {
  constexpr int NP = K<R>::NP;
  for (int q = threadIdx.x; q < NP; q += blockDim.x) {
    int a = 0, rem = q;
    while (rem >= R - a) { rem -= R - a; a++; }
    const int b = a + rem;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int u = 0;
    for (; u + 4 <= nparts; u += 4) {
      s0 += __ldcg(part + (size_t)u * NP + q);
      s1 += __ldcg(part + (size_t)(u + 1) * NP + q);
      s2 += __ldcg(part + (size_t)(u + 2) * NP + q);
      s3 += __ldcg(part + (size_t)(u + 3) * NP + q);
    }
    for (; u < nparts; u++) s0 += __ldcg(part + (size_t)u * NP + q);
    const double gsum = (s0 + s1) + (s2 + s3);
    o.L[a * 32 + b] = gsum;
    o.L[b * 32 + a] = gsum;
    if (a == b) o.gdiag[a] = gsum;
  }
}

// Warp-level right-looking Cholesky of o.L (R <= 32): lane i holds row i in
// registers.  detect: stop at the first column whose squared residual is below
// tau2 * its own squared norm (reading C3) and return 1.  Called by warp 0.
template <int R>
__device__ int chol_warp(OrthW& o, double tau2, bool detect) {
  const int i = threadIdx.x & 31;
  double row[R];
#pragma unroll
  for (int k = 0; k < R; k++) row[k] = (i < R) ? o.L[i * 32 + k] : 0.0;
  const double g0 = (i < R) ? o.gdiag[i] : 0.0;
  int deg = 0;
#pragma unroll
  for (int j = 0; j < R; j++) {
    const double d = shfl_d(row[j], j);
    const double gj = shfl_d(g0, j);
    if (detect && (gj == 0.0 || !(d >= tau2 * gj))) { deg = 1; break; }
    const double ljj = sqrt(d > 0.0 ? d : 1e-300);
    const double inv = 1.0 / ljj;
    const double lij = (i > j) ? row[j] * inv : (i == j ? ljj : 0.0);
    row[j] = lij;
#pragma unroll
    for (int k = j + 1; k < R; k++) {
      const double lk = shfl_d(lij, k);
      if (i >= k) row[k] = fma(-lij, lk, row[k]);
    }
  }
  if (!deg && i < R) {
#pragma unroll
    for (int k = 0; k < R; k++) o.L[i * 32 + k] = (k <= i) ? row[k] : 0.0;
  }
  return deg;
}

// o.Li = o.L^-1 (lower), kappa = ||L||_F ||L^-1||_F.  Warp 0; lane c owns column c.
template <int R>
__device__ void inverse_warp(OrthW& o) {
  const int c = threadIdx.x & 31;
  double col[R];
  double nl = 0.0, ni = 0.0;
#pragma unroll
  for (int i = 0; i < R; i++) {
    double v = (i == c) ? 1.0 : 0.0;
#pragma unroll
    for (int k = 0; k < i; k++) v = fma(-o.L[i * 32 + k], col[k], v);
    col[i] = (i >= c && c < R) ? v / o.L[i * 32 + i] : 0.0;
    if (c < R && i >= c) { ni = fma(col[i], col[i], ni); }
  }
  if (c < R) {
#pragma unroll
    for (int i = 0; i < R; i++) {
      o.Li[i * 32 + c] = col[i];
      if (i >= c) nl = fma(o.L[i * 32 + c], o.L[i * 32 + c], nl);
    }
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    nl += __shfl_xor_sync(0xffffffffu, nl, off);
    ni += __shfl_xor_sync(0xffffffffu, ni, off);
  }
  if (c == 0) o.kappa = sqrt(nl) * sqrt(ni);
}

// Up-looking Cholesky with column substitution (slow path, thread 0).
template <int R>
__device__ void chol_subst(OrthW& o, double tau2) {
  if (threadIdx.x != 0) return;
  double* L = o.Li;  // scratch; o.L keeps P^T P
  for (int x = 0; x < 32 * 32; x++) L[x] = 0.0;
  for (int j = 0; j < R; j++) o.rep[j] = 0;
  auto gram = [&](int a, int b) -> double {
    const bool ra = o.rep[a], rb = o.rep[b];
    if (!ra && !rb) return o.L[a * 32 + b];
    if (!ra && rb) return o.X[a * 32 + b];
    if (ra && !rb) return o.X[b * 32 + a];
    return o.Y[a * 32 + b];
  };
  for (int i = 0; i < R; i++) {
    for (int attempt = 0; attempt < 2; attempt++) {
      for (int k = 0; k < i; k++) {
        double v = gram(i, k);
        for (int l = 0; l < k; l++) v -= L[i * 32 + l] * L[k * 32 + l];
        L[i * 32 + k] = v / L[k * 32 + k];
      }
      double d = gram(i, i);
      const double g = d;
      for (int k = 0; k < i; k++) d -= L[i * 32 + k] * L[i * 32 + k];
      if (attempt == 0 && (g == 0.0 || !(d >= tau2 * g))) { o.rep[i] = 1; continue; }
      L[i * 32 + i] = sqrt(d > 0.0 ? d : 1e-300);
      break;
    }
  }
  for (int x = 0; x < 32 * 32; x++) o.L[x] = L[x];
}

// out[i][a] = sum_{b<=a} Pm[i][b] Li[a][b]  (fp64, rounded to fp32); Pm[i][b] = rep[b] ? f_b : ps[i][b]
template <int R>
__device__ void band_apply(const float* ps, float* out, int nr, const OrthW& o, bool use_rep,
                           unsigned long long seed, int row0) {
  constexpr int RP = K<R>::RP;
  for (int x = threadIdx.x; x < nr * R; x += blockDim.x) {
    const int i = x / R, a = x % R;
    double v = 0.0;
#pragma unroll 4
    for (int b = 0; b <= a; b++) {
      const double pv = (use_rep && o.rep[b]) ? (double)fallback_entry(seed, b, row0 + i) : (double)ps[i * RP + b];
      v = fma(pv, o.Li[a * 32 + b], v);
    }
    out[i * RP + a] = (float)v;
  }
}

// Gram partial (packed) of rows [0,nr) of an fp32 [.][RP] array, fp64.
template <int R>
__device__ void band_gram(const float* ps, int nr, double* part, double* scratch) {
  constexpr int RP = K<R>::RP, NP = K<R>::NP;
  const int gsz = max(1, (int)blockDim.x / NP);
  for (int x = threadIdx.x; x < NP * gsz; x += blockDim.x) {
    const int q = x % NP, grp = x / NP;
    int a = 0, rem = q;
    while (rem >= R - a) { rem -= R - a; a++; }
    const int b = a + rem;
    double gg = 0.0;
    for (int i = grp; i < nr; i += gsz) gg = fma((double)ps[i * RP + a], (double)ps[i * RP + b], gg);
    scratch[x] = gg;
  }
  __syncthreads();
  for (int q = threadIdx.x; q < NP; q += blockDim.x) {
    double gg = 0.0;
    for (int grp = 0; grp < gsz; grp++) gg += scratch[grp * NP + q];
    part[q] = gg;
  }
}

template <int R, bool MBF>
__global__ void __launch_bounds__(NT, 1) occ_v2_kernel(Params2 p) {
  constexpr int RP = K<R>::RP, MT = K<R>::MT, KS5 = K<R>::KS5, NP = K<R>::NP;
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint64_t mbar[MAX_STAGES];
  __shared__ unsigned tmem_base_sh;

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, g = lane >> 2, t = lane & 3;
  const Tile T = tile_of(p);
  const bool active = T.rb < p.nr && T.th > 0 && T.tw > 0;
  const int CGW = (T.ncg + NW - 1) / NW;     // column groups per warp
  unsigned nb = 0;
  auto gbar = [&]() { nb++; grid_barrier(p.bar, nb * gridDim.x); };
  const bool stamp = blockIdx.x == 0 && tid == 0;
  if (stamp) p.stats->t_ns[0] = gtimer();

  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base_sh)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < MAX_STAGES; s++) mbar_init(&mbar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tbase = tmem_base_sh;
  const unsigned taddr_w = tbase + ((unsigned)((w & 3) * 32) << 16) + (unsigned)((w >> 2) * 128);
  auto cell_slot = [&](int rblk, int cg) { return rblk * CGW + cg / NW; };

  // ============================================================== phase 1
  unsigned char* stM = sm + p.off_stm;
  float* stE = reinterpret_cast<float*>(sm + p.off_ste);
  float* qs = reinterpret_cast<float*>(sm + p.off_qs);    // [W][RP] Q_prev slice
  float* red = reinterpret_cast<float*>(sm + p.off_red);  // [NW][8][RP]
  const int nst = active ? T.nrblk : 0;
  const size_t esz = MBF ? 2 : 4;
  auto issue = [&](int s) {
    const int slot = s % p.ns;
    const int r0 = s * SR, nrow = min(SR, T.th - r0);
    const unsigned rbM = (unsigned)(T.tw * esz), rbE = (unsigned)(T.tw * 4);
    mbar_expect_tx(&mbar[slot], (unsigned)nrow * (rbM + (p.err_in ? rbE : 0u)));
    for (int i = 0; i < nrow; i++) {
      const size_t gi = (size_t)(T.row0 + r0 + i);
      bulk_g2s(stM + ((size_t)(slot * SR + i) * p.sw) * 4,
               reinterpret_cast<const char*>(p.M) + (gi * p.ldm + T.col0) * esz, rbM, &mbar[slot]);
      if (p.err_in)
        bulk_g2s(stE + (size_t)(slot * SR + i) * p.sw, p.err_in + gi * p.lde_in + T.col0, rbE, &mbar[slot]);
    }
  };
  if (active) {
    if (tid == 0)
      for (int s = 0; s < min(p.ns, nst); s++) issue(s);
    for (int x = tid; x < T.tw * RP; x += NT) {
      const int c = x / RP, k = x % RP;
      qs[x] = (k < R) ? __ldcg(p.Qprev + (size_t)(T.col0 + c) * R + k) : 0.f;
    }
  }
  __syncthreads();
  for (int s = 0; s < nst; s++) {
    const int slot = s % p.ns;
    mbar_wait(&mbar[slot], (unsigned)((s / p.ns) & 1));
    const int nrow = min(SR, T.th - s * SR);
    const unsigned char* sMb = stM + (size_t)slot * SR * p.sw * 4;
    const float* sE = stE + (size_t)slot * SR * p.sw;
    auto Av = [&](int i, int j) -> float {
      if (i >= nrow || j >= T.tw) return 0.f;
      float v = MBF ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(sMb)[(size_t)i * 2 * p.sw + j])
                    : reinterpret_cast<const float*>(sMb)[(size_t)i * p.sw + j];
      if (p.err_in) v += sE[(size_t)i * p.sw + j];
      return v;
    };
    // (a) P^T[k][rows] = Q_prev^T[k][cols] A^T[cols][rows]; warps split the column k-steps
    float acc[MT][4];
#pragma unroll
    for (int mt = 0; mt < MT; mt++) acc[mt][0] = acc[mt][1] = acc[mt][2] = acc[mt][3] = 0.f;
    for (int kk = w; kk < T.tw / 8; kk += NW) {
      const int c = 8 * kk;
      unsigned bh0, bl0, bh1, bl1;
      split3(Av(g, c + t), bh0, bl0);
      split3(Av(g, c + t + 4), bh1, bl1);
#pragma unroll
      for (int mt = 0; mt < MT; mt++) {
        const int k0 = 16 * mt + g;
        unsigned ah[4], al[4];
        split3(qs[(c + t) * RP + k0], ah[0], al[0]);
        split3((k0 + 8 < RP) ? qs[(c + t) * RP + k0 + 8] : 0.f, ah[1], al[1]);
        split3(qs[(c + t + 4) * RP + k0], ah[2], al[2]);
        split3((k0 + 8 < RP) ? qs[(c + t + 4) * RP + k0 + 8] : 0.f, ah[3], al[3]);
        mma3(acc[mt], ah, al, bh0, bh1, bl0, bl1);
      }
    }
    {  // D[k][row]: c0 = (k=16mt+g, row=2t), c1 = (g, 2t+1), c2 = (g+8, 2t), c3 = (g+8, 2t+1)
      float* rw = red + (size_t)w * SR * RP;
#pragma unroll
      for (int mt = 0; mt < MT; mt++) {
        const int k0 = 16 * mt + g;
        rw[(2 * t) * RP + k0] = acc[mt][0];
        rw[(2 * t + 1) * RP + k0] = acc[mt][1];
        if (k0 + 8 < RP) {
          rw[(2 * t) * RP + k0 + 8] = acc[mt][2];
          rw[(2 * t + 1) * RP + k0 + 8] = acc[mt][3];
        }
      }
    }
    // (b) TMEM: cells of row block s in this warp's column groups
    for (int cg = w; cg < T.ncg; cg += NW) {
      const int cs = cell_slot(s, cg);
      if (cs >= TMEM_CELLS) break;
      const int c0 = 16 * cg + g;
      tmem_st4(taddr_w + (unsigned)(cs * 4), Av(2 * t, c0), Av(2 * t + 1, c0), Av(2 * t, c0 + 8), Av(2 * t + 1, c0 + 8));
    }
    __syncthreads();
    for (int x = tid; x < SR * R; x += NT) {
      const int i = x / R, k = x % R;
      float v = 0.f;
#pragma unroll
      for (int ww = 0; ww < NW; ww++) v += red[(size_t)(ww * SR + i) * RP + k];
      if (i < nrow) p.P_part[((size_t)T.cb * p.n + T.row0 + s * SR + i) * R + k] = v;
    }
    __syncthreads();
    if (tid == 0 && s + p.ns < nst) issue(s + p.ns);
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  gbar();
  if (stamp) p.stats->t_ns[1] = gtimer();

  // ============================================================== phase 2
  const int H8 = T.nrblk * 8;
  float* ps = reinterpret_cast<float*>(sm + p.off_ps);   // [H8][RP] P_band, later P_hat
  float* ps2 = ps + (size_t)((p.H + 7) / 8 * 8) * RP;   // [H8][RP]
  double* gscr = reinterpret_cast<double*>(sm + p.off_gs);
  OrthW& o = *reinterpret_cast<OrthW*>(sm + p.off_orth);
  if (active) {
    for (int x = tid; x < H8 * RP; x += NT) {
      const int i = x / RP, k = x % RP;
      float v = 0.f;
      if (i < T.th && k < R) {
        const float* src = p.P_part + ((size_t)T.row0 + i) * R + k;
        for (int c = 0; c < p.nc; c++) v += __ldcg(src + (size_t)c * p.n * R);
      }
      ps[x] = v;
    }
    __syncthreads();
    if (T.cb == 0) band_gram<R>(ps, T.th, p.G_band + (size_t)T.rb * NP, gscr);
  }
  gbar();
  if (stamp) p.stats->t_ns[2] = gtimer();

  // ============================================================== phase 3
  const double tau2 = p.tau * p.tau;
  reduce_partials<R>(p.G_band, p.nr, o);
  __syncthreads();
  if (w == 0) {
    const int d = chol_warp<R>(o, tau2, true);
    if (lane == 0) o.deg = d;
  }
  __syncthreads();
  const bool deg = o.deg != 0;
  if (deg) {  // slow path: augmented Gram with the fallback vector of every column
    if (active && T.cb == 0) {
      float* fs = ps2;
      for (int x = tid; x < T.th * RP; x += NT) fs[x] = fallback_entry(p.fb_seed, x % RP, T.row0 + x / RP);
      __syncthreads();
      for (int q = tid; q < 2 * R * R; q += NT) {
        const int which = q / (R * R), a = (q / R) % R, b = q % R;
        const float* lhs = which ? fs : ps;
        double gg = 0.0;
        for (int i = 0; i < T.th; i++) gg = fma((double)lhs[i * RP + a], (double)fs[i * RP + b], gg);
        p.XY_band[(size_t)T.rb * 2 * R * R + q] = gg;
      }
    }
    gbar();
    reduce_partials<R>(p.G_band, p.nr, o);
    for (int q = tid; q < 2 * R * R; q += NT) {
      double gg = 0.0;
      for (int u = 0; u < p.nr; u++) gg += __ldcg(p.XY_band + (size_t)u * 2 * R * R + q);
      const int a = (q / R) % R, b = q % R;
      if (q < R * R) o.X[a * 32 + b] = gg; else o.Y[a * 32 + b] = gg;
    }
    __syncthreads();
    chol_subst<R>(o, tau2);
  } else if (tid < 32) {
    o.rep[tid] = 0;
  }
  __syncthreads();
  if (w == 0) inverse_warp<R>(o);
  __syncthreads();
  const bool need2 = p.force_two_pass || o.kappa > p.kappa_thr;
  if (active) {
    band_apply<R>(ps, ps2, T.th, o, deg, p.fb_seed, T.row0);
    __syncthreads();
    for (int x = tid; x < H8 * RP; x += NT) ps[x] = (x / RP < T.th) ? ps2[x] : 0.f;
    __syncthreads();
  }
  if (blockIdx.x == 0 && tid == 0) {
    int cnt = 0;
    for (int j = 0; j < R; j++) cnt += deg ? o.rep[j] : 0;
    p.stats->fallback_columns = cnt;
    p.stats->second_pass = need2 ? 1 : 0;
    p.stats->kappa_est = o.kappa;
  }
  if (need2) {  // CholQR2: orthonormalise the fp32-rounded P_hat once more
    if (active && T.cb == 0) band_gram<R>(ps, T.th, p.G2_band + (size_t)T.rb * NP, gscr);
    gbar();
    reduce_partials<R>(p.G2_band, p.nr, o);
    __syncthreads();
    if (w == 0) chol_warp<R>(o, 0.0, false);
    __syncthreads();
    if (w == 0) inverse_warp<R>(o);
    __syncthreads();
    if (active) {
      band_apply<R>(ps, ps2, T.th, o, false, p.fb_seed, T.row0);
      __syncthreads();
      for (int x = tid; x < H8 * RP; x += NT) ps[x] = (x / RP < T.th) ? ps2[x] : 0.f;
      __syncthreads();
    }
  }
  if (stamp) p.stats->t_ns[3] = gtimer();
  uint4* pa = reinterpret_cast<uint4*>(sm + p.off_pa);   // [nrblk][MT][32][2] (hi, lo)
  uint4* pb = reinterpret_cast<uint4*>(sm + p.off_pb);   // [nrblk][KS5][32]   (h0, h1, l0, l1)
  if (active) {
    if (T.cb == 0)
      for (int x = tid; x < T.th * R; x += NT) p.Pout[((size_t)T.row0 + x / R) * R + x % R] = ps[(x / R) * RP + x % R];
    for (int x = tid; x < T.nrblk * MT * 32; x += NT) {
      const int ln = x % 32, mt = (x / 32) % MT, rblk = x / (32 * MT);
      const int gg = ln >> 2, tt = ln & 3;
      const int r0 = 8 * rblk + 2 * tt, k0 = 16 * mt + gg;
      float v[4];
      v[0] = (k0 < R) ? ps[r0 * RP + k0] : 0.f;
      v[1] = (k0 + 8 < R) ? ps[r0 * RP + k0 + 8] : 0.f;
      v[2] = (k0 < R) ? ps[(r0 + 1) * RP + k0] : 0.f;
      v[3] = (k0 + 8 < R) ? ps[(r0 + 1) * RP + k0 + 8] : 0.f;
      uint4 hi, lo;
      split3(v[0], hi.x, lo.x); split3(v[1], hi.y, lo.y); split3(v[2], hi.z, lo.z); split3(v[3], hi.w, lo.w);
      pa[2 * x] = hi;
      pa[2 * x + 1] = lo;
    }
    for (int x = tid; x < T.nrblk * KS5 * 32; x += NT) {
      const int ln = x % 32, ks = (x / 32) % KS5, rblk = x / (32 * KS5);
      const int gg = ln >> 2, tt = ln & 3;
      const int r = 8 * rblk + gg, k = 8 * ks + tt;
      uint4 v;
      unsigned h0, l0, h1, l1;
      split3((k < R) ? ps[r * RP + k] : 0.f, h0, l0);
      split3((k + 4 < R) ? ps[r * RP + k + 4] : 0.f, h1, l1);
      v.x = h0; v.y = h1; v.z = l0; v.w = l1;
      pb[x] = v;
    }
  }
  __syncthreads();
  // phase 3a: Q_part[rb][cols] = A_tile^T P_hat_band, complete per column group in one warp
  if (active) {
    for (int cg = w; cg < T.ncg; cg += NW) {
      float qa[MT][2][4];
#pragma unroll
      for (int mt = 0; mt < MT; mt++)
#pragma unroll
        for (int nt = 0; nt < 2; nt++) qa[mt][nt][0] = qa[mt][nt][1] = qa[mt][nt][2] = qa[mt][nt][3] = 0.f;
      for (int rblk = 0; rblk < T.nrblk; rblk++) {
        float v[4];
        const int cs = cell_slot(rblk, cg);
        if (cs < TMEM_CELLS) tmem_ld4(taddr_w + (unsigned)(cs * 4), v);
        else cell_from_global<MBF>(p, T, rblk, cg, g, t, v);
        unsigned vh[4], vl[4];
#pragma unroll
        for (int q = 0; q < 4; q++) split3(v[q], vh[q], vl[q]);
#pragma unroll
        for (int mt = 0; mt < MT; mt++) {
          const uint4 h = pa[2 * ((rblk * MT + mt) * 32 + lane)], l = pa[2 * ((rblk * MT + mt) * 32 + lane) + 1];
          const unsigned ah[4] = {h.x, h.y, h.z, h.w}, al[4] = {l.x, l.y, l.z, l.w};
          mma3(qa[mt][0], ah, al, vh[0], vh[1], vl[0], vl[1]);
          mma3(qa[mt][1], ah, al, vh[2], vh[3], vl[2], vl[3]);
        }
      }
      // D[k][col]: c0 = (k=16mt+g, col=8nt+2t), c1 = (g, 2t+1), c2 = (g+8, 2t), c3 = (g+8, 2t+1)
      float* dst = p.Q_part + ((size_t)T.rb * p.m + T.col0 + 16 * cg) * R;
#pragma unroll
      for (int mt = 0; mt < MT; mt++)
#pragma unroll
        for (int nt = 0; nt < 2; nt++) {
          const int col = 8 * nt + 2 * t, k = 16 * mt + g;
          if (16 * cg + col < T.tw) {
            if (k < R) dst[col * R + k] = qa[mt][nt][0];
            if (k + 8 < R) dst[col * R + k + 8] = qa[mt][nt][2];
          }
          if (16 * cg + col + 1 < T.tw) {
            if (k < R) dst[(col + 1) * R + k] = qa[mt][nt][1];
            if (k + 8 < R) dst[(col + 1) * R + k + 8] = qa[mt][nt][3];
          }
        }
    }
  }
  gbar();
  if (stamp) p.stats->t_ns[4] = gtimer();

  // ============================================================== phase 4
  if (active) {
    const int tot = T.tw * R;
    const int per = (tot + p.nr - 1) / p.nr;
    const int x0 = T.rb * per, x1 = min(tot, x0 + per);
    for (int x = x0 + tid; x < x1; x += NT) {
      const float* src = p.Q_part + (size_t)T.col0 * R + x;
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
      int u = 0;
      for (; u + 4 <= p.nr; u += 4) {
        s0 += __ldcg(src + (size_t)u * p.m * R);
        s1 += __ldcg(src + (size_t)(u + 1) * p.m * R);
        s2 += __ldcg(src + (size_t)(u + 2) * p.m * R);
        s3 += __ldcg(src + (size_t)(u + 3) * p.m * R);
      }
      for (; u < p.nr; u++) s0 += __ldcg(src + (size_t)u * p.m * R);
      p.Qout[(size_t)T.col0 * R + x] = (s0 + s1) + (s2 + s3);
    }
  }
  gbar();
  if (stamp) p.stats->t_ns[5] = gtimer();

  // ============================================================== phase 5
  if (active) {
    for (int cg = w; cg < T.ncg; cg += NW) {
      unsigned qh[KS5][4], ql[KS5][4];
      {
        const int cA = T.col0 + 16 * cg + g;
        const bool okA = 16 * cg + g < T.tw, okB = 16 * cg + g + 8 < T.tw;
#pragma unroll
        for (int ks = 0; ks < KS5; ks++) {
          const int k0 = 8 * ks + t;
          const float a0 = (okA && k0 < R) ? __ldcg(p.Qout + (size_t)cA * R + k0) : 0.f;
          const float a1 = (okB && k0 < R) ? __ldcg(p.Qout + (size_t)(cA + 8) * R + k0) : 0.f;
          const float a2 = (okA && k0 + 4 < R) ? __ldcg(p.Qout + (size_t)cA * R + k0 + 4) : 0.f;
          const float a3 = (okB && k0 + 4 < R) ? __ldcg(p.Qout + (size_t)(cA + 8) * R + k0 + 4) : 0.f;
          split3(a0, qh[ks][0], ql[ks][0]);
          split3(a1, qh[ks][1], ql[ks][1]);
          split3(a2, qh[ks][2], ql[ks][2]);
          split3(a3, qh[ks][3], ql[ks][3]);
        }
      }
      for (int rblk = 0; rblk < T.nrblk; rblk++) {
        float mr[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int ks = 0; ks < KS5; ks++) {
          const uint4 b = pb[(rblk * KS5 + ks) * 32 + lane];
          mma3(mr, qh[ks], ql[ks], b.x, b.y, b.z, b.w);
        }
        float v[4];
        const int cs = cell_slot(rblk, cg);
        if (cs < TMEM_CELLS) tmem_ld4(taddr_w + (unsigned)(cs * 4), v);
        else cell_from_global<MBF>(p, T, rblk, cg, g, t, v);
        if (MBF) {
#pragma unroll
          for (int q = 0; q < 4; q++) mr[q] = __bfloat162float(__float2bfloat16_rn(mr[q]));
        }
        const int r = 8 * rblk + 2 * t, c = 16 * cg + g;
        const int rows[4] = {r, r + 1, r, r + 1}, cols[4] = {c, c, c + 8, c + 8};
#pragma unroll
        for (int q = 0; q < 4; q++) {
          if (rows[q] < T.th && cols[q] < T.tw) {
            const size_t gi = (size_t)T.row0 + rows[q], gj = (size_t)T.col0 + cols[q];
            if (p.recon) {
              if (MBF) reinterpret_cast<__nv_bfloat16*>(p.recon)[gi * p.ldr + gj] = __float2bfloat16_rn(mr[q]);
              else reinterpret_cast<float*>(p.recon)[gi * p.ldr + gj] = mr[q];
            }
            if (p.err_out) p.err_out[gi * p.lde_out + gj] = v[q] - mr[q];
          }
        }
      }
    }
  }
  if (stamp) p.stats->t_ns[6] = gtimer();

  // ============================================================== teardown
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
  if (tid == 0) {
    const unsigned old = atomicAdd(p.bar + 1, 1u);
    if (old == gridDim.x - 1) {
      atomicExch(p.bar, 0u);
      atomicExch(p.bar + 1, 0u);
    }
  }
  if (blockIdx.x == 0 && tid == 0) {
    p.stats->path = 3;
    p.stats->grid = gridDim.x;
  }
}

// ------------------------------------------------------------------ host side
struct Plan2 {
  bool ok = false;
  int nr = 0, nc = 0, H = 0, W = 0, ns = 0, sw = 0;
  int off_stm = 0, off_ste = 0, off_qs = 0, off_red = 0, off_pa = 0, off_pb = 0, off_orth = 0, off_ps = 0, off_gs = 0;
  int total = 0, cells_per_warp = 0;
  double cost = 0;
};

static int al128(int x) { return (x + 127) / 128 * 128; }

// streaming efficiency of one cp.async.bulk per tile row (measured: 1 KB -> 0.6, 2 KB -> 0.92, >= 4 KB -> 1.0)
static double row_eff(int bytes) {
  if (bytes >= 4096) return 1.0;
  if (bytes >= 2048) return 0.92 + 0.08 * (bytes - 2048) / 2048.0;
  if (bytes >= 1024) return 0.6 + 0.32 * (bytes - 1024) / 1024.0;
  return 0.35 + 0.25 * bytes / 1024.0;
}

template <int R>
static Plan2 plan_for(int64_t n, int64_t m, int sms, bool mbf) {
  constexpr int RP = K<R>::RP, MT = K<R>::MT, KS5 = K<R>::KS5, NP = K<R>::NP;
  Plan2 best;
  const int smem_cap = 227 * 1024 - 2048;
  for (int nc = 1; nc <= sms; nc++) {
    const int nr_max = sms / nc;
    if (nr_max < 1) break;
    const int W = (int)(((m + nc - 1) / nc + 15) / 16 * 16);
    const int H = (int)(((n + nr_max - 1) / nr_max + 7) / 8 * 8);
    Plan2 pl;
    pl.nr = (int)((n + H - 1) / H);
    pl.nc = (int)((m + W - 1) / W);
    if (pl.nr * pl.nc > sms) continue;
    pl.H = H;
    pl.W = W;
    pl.sw = W + 4;   // = 4 (mod 8) floats: conflict-free fragment reads
    const int stage_bytes = SR * pl.sw * 4;
    const int qs_bytes = al128(W * RP * 4);
    const int red_bytes = al128(NW * SR * RP * 4);
    int ns = 0;
    for (int k = MAX_STAGES; k >= 2; k--)
      if (2 * k * stage_bytes + qs_bytes + red_bytes <= smem_cap) { ns = k; break; }
    if (!ns) continue;
    pl.ns = ns;
    int off = 0;
    pl.off_stm = off; off += ns * stage_bytes;
    pl.off_ste = off; off += ns * stage_bytes;
    pl.off_qs = off; off += qs_bytes;
    pl.off_red = off; off += red_bytes;
    const int p1 = off;
    const int H8 = (H + 7) / 8 * 8, nrblk = H8 / 8, ncg = W / 16;
    off = 0;
    pl.off_ps = off; off += al128(2 * H8 * RP * 4);
    pl.off_gs = off; off += al128((std::max(NT, NP) + NP) * 8);
    pl.off_orth = off; off += al128((int)sizeof(OrthW));
    pl.off_pa = off; off += al128(nrblk * MT * 32 * 32);
    pl.off_pb = off; off += al128(nrblk * KS5 * 32 * 16);
    pl.total = std::max(p1, off);
    if (pl.total > smem_cap) continue;
    const int cgw = (ncg + NW - 1) / NW;
    pl.cells_per_warp = cgw * nrblk;
    pl.ok = true;
    // modelled time (arbitrary units = bytes at HBM speed): streaming the tile,
    // re-reading non-resident cells from L2, and the partial-sum traffic
    const double tile_bytes = (double)H * W * ((mbf ? 2 : 4) + 4 + 4 + (mbf ? 2 : 4));
    const int row_bytes = W * 4;
    const double spill = std::max(0, pl.cells_per_warp - TMEM_CELLS) / (double)pl.cells_per_warp;
    const double partial = ((double)pl.nc * n + (double)pl.nr * m) * R * 4 * 2 / sms;
    pl.cost = tile_bytes / row_eff(row_bytes) + spill * (double)H * W * 16 + partial;
    if (!best.ok || pl.cost < best.cost) best = pl;
  }
  return best;
}

template <int R, bool MBF>
static cudaError_t launch2(const Params& p1, const Plan2& pl, void* ws_tail, cudaStream_t st) {
  Params2 p;
  memset(&p, 0, sizeof p);
  p.M = p1.M; p.ldm = p1.ldm;
  p.err_in = p1.err_in; p.lde_in = p1.lde_in;
  p.err_out = p1.err_out; p.lde_out = p1.lde_out;
  p.recon = p1.recon; p.ldr = p1.ldr;
  p.n = p1.n; p.m = p1.m;
  p.Qprev = p1.Qprev; p.Pout = p1.P; p.Qout = p1.Qloc;
  p.nr = pl.nr; p.nc = pl.nc; p.H = pl.H; p.W = pl.W; p.ns = pl.ns; p.sw = pl.sw;
  p.off_stm = pl.off_stm; p.off_ste = pl.off_ste; p.off_qs = pl.off_qs; p.off_red = pl.off_red;
  p.off_pa = pl.off_pa; p.off_pb = pl.off_pb; p.off_orth = pl.off_orth; p.off_ps = pl.off_ps; p.off_gs = pl.off_gs;
  p.smem_total = pl.total;
  char* tail = static_cast<char*>(ws_tail);
  constexpr int NP = K<R>::NP;
  size_t off = 0;
  auto take = [&](size_t bytes) { char* q = tail + off; off += (bytes + 255) / 256 * 256; return q; };
  p.P_part = reinterpret_cast<float*>(take((size_t)pl.nc * p.n * R * 4));
  p.Q_part = reinterpret_cast<float*>(take((size_t)pl.nr * p.m * R * 4));
  p.G_band = reinterpret_cast<double*>(take((size_t)pl.nr * NP * 8));
  p.G2_band = reinterpret_cast<double*>(take((size_t)pl.nr * NP * 8));
  p.XY_band = reinterpret_cast<double*>(take((size_t)pl.nr * 2 * R * R * 8));
  p.bar = p1.bar;
  p.stats = p1.stats;
  p.fb_seed = p1.fb_seed;
  p.tau = p1.tau;
  p.kappa_thr = p1.kappa_thr;
  p.force_two_pass = p1.force_two_pass;
  auto kern = occ_v2_kernel<R, MBF>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, pl.total);
  if (e != cudaSuccess) return e;
  void* args[] = {&p};
  return cudaLaunchCooperativeKernel((const void*)kern, dim3(pl.nr * pl.nc), dim3(NT), args, pl.total, st);
}

template <int R>
static size_t tail_bytes(const Plan2& pl, int64_t n, int64_t m) {
  constexpr int NP = K<R>::NP;
  auto a = [](size_t b) { return (b + 255) / 256 * 256; };
  return a((size_t)pl.nc * n * R * 4) + a((size_t)pl.nr * m * R * 4) + 2 * a((size_t)pl.nr * NP * 8) +
         a((size_t)pl.nr * 2 * R * R * 8);
}

}  // namespace v2

// Workspace the fused v2 path needs (0 if no plan applies; the v1 phases run then).
// The plan is computed for fp32 M; a bf16 M picks a plan with the same or smaller tail.
size_t v2_tail_bytes(int64_t n, int64_t m, int r, int sms) {
  size_t b = 0;
  switch (r) {
#define V2T(RR)                                                                  \
  case RR: {                                                                     \
    auto p0 = v2::plan_for<RR>(n, m, sms, false);                                \
    auto p1 = v2::plan_for<RR>(n, m, sms, true);                                 \
    if (p0.ok) b = std::max(b, v2::tail_bytes<RR>(p0, n, m));                    \
    if (p1.ok) b = std::max(b, v2::tail_bytes<RR>(p1, n, m));                    \
    return b;                                                                    \
  }
    V2T(4) V2T(8) V2T(16) V2T(32)
#undef V2T
  }
  return 0;
}

cudaError_t run_v2(const Params& p, int r, void* ws_tail, size_t tail_avail, int sms, cudaStream_t st) {
  switch (r) {
#define V2C(RR)                                                                                   \
  case RR: {                                                                                      \
    auto pl = v2::plan_for<RR>(p.n, p.m, sms, p.m_bf16 != 0);                                     \
    if (!pl.ok || v2::tail_bytes<RR>(pl, p.n, p.m) > tail_avail) return cudaErrorNotSupported;     \
    return p.m_bf16 ? v2::launch2<RR, true>(p, pl, ws_tail, st) : v2::launch2<RR, false>(p, pl, ws_tail, st); \
  }
    V2C(4) V2C(8) V2C(16) V2C(32)
#undef V2C
  }
  return cudaErrorNotSupported;
}

}  // namespace occ
