// occ_v2.cu -- kernel body and launcher of the TMEM-resident fused step
// (design in occ_v2.cuh).
#include "occ_v2.cuh"
#include "occ_internal.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
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

constexpr int LD = 33;   // padded stride of the small fp64 matrices: conflict-free rows and columns

struct OrthW {  // small fp64 linear algebra in shared memory
  double L[32 * LD];    // Gram (full), then the unit lower factor of G = L D L^T
  double Li[32 * LD];   // D^-1/2 L^-1: P_hat = P Li^T
  double X[32 * LD];    // P^T F (slow path)
  double Y[32 * LD];    // F^T F (slow path)
  double gdiag[32];     // diag(G): each column's own squared norm (degeneracy test)
  double D[32];
  double col[32];       // per-step broadcast buffer
  double dinv[32];      // D^-1/2
  int rep[32];
  int deg;
  double kappa;
};

// out[e] = sum_{u < S} src[u * stride + e], e < E, in a fixed order (deterministic).
// Every thread keeps 16 independent loads in flight: the partial sums live in
// L2 and this is latency bound.  scratch: NT elements of shared memory.
template <typename Tv, typename Fout>
__device__ void strided_sum(const Tv* __restrict__ src, size_t stride, int S, int E, Tv* scratch, Fout&& out) {
  for (int e0 = 0; e0 < E; e0 += NT) {
    const int En = min(NT, E - e0);
    const int C = max(1, NT / En);
    const int x = threadIdx.x;
    Tv acc = Tv(0);
    if (x < En * C) {
      const int e = e0 + x % En, c = x / En;
      for (int u0 = c; u0 < S; u0 += 16 * C) {
        Tv v[16];
#pragma unroll
        for (int j = 0; j < 16; j++) {
          const int u = u0 + j * C;
          v[j] = (u < S) ? __ldcg(src + (size_t)u * stride + e) : Tv(0);
        }
#pragma unroll
        for (int j = 0; j < 16; j++) acc += v[j];
      }
    }
    __syncthreads();
    if (x < En * C) scratch[x] = acc;
    __syncthreads();
    if (x < En) {
      Tv r = Tv(0);
      for (int c = 0; c < C; c++) r += scratch[c * En + x];
      out(e0 + x, r);
    }
    __syncthreads();
  }
}

// G (packed upper triangle, nparts partials) -> o.L (full symmetric), o.gdiag.  All threads.
template <int R>
__device__ void reduce_partials(const double* __restrict__ part, int nparts, OrthW& o, double* scratch) {
  constexpr int NP = K<R>::NP;
  strided_sum<double>(part, NP, nparts, NP, scratch, [&](int q, double gsum) {
    int a = 0, rem = q;
    while (rem >= R - a) { rem -= R - a; a++; }
    const int b = a + rem;
    o.L[a * LD + b] = gsum;
    o.L[b * LD + a] = gsum;
    if (a == b) o.gdiag[a] = gsum;
  });
}

// 1/d for normal d > 0: MUFU reciprocal estimate + two Newton steps (full fp64
// accuracy; roughly half the latency of the IEEE division on the LDL chain).
__device__ __forceinline__ double rcp_fast(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  return fma(r, e, r);
}

// Warp-level right-looking LDL^T of the Gram in o.L (R <= 32), square-root free
// so the sequential chain per column is one fp64 reciprocal.  Lane i holds row
// i in registers; column j is broadcast through o.col.  detect: stop at the
// first column whose squared residual D_j is below tau2 * its own squared norm
// (reading C3: the MGS test ||v|| < tau ||p_j||) and return 1.  Warp 0 only.
template <int R>
__device__ int ldl_warp(OrthW& o, double tau2, bool detect) {
  const int i = threadIdx.x & 31;
  double row[R];
#pragma unroll
  for (int k = 0; k < R; k++) row[k] = (i < R) ? o.L[i * LD + k] : 0.0;
  int deg = 0;
#pragma unroll
  for (int j = 0; j < R; j++) {
    if (i >= j && i < R) o.col[i] = row[j];   // u_i = G_ij after the previous updates
    __syncwarp();
    const double d = o.col[j];
    const double gj = o.gdiag[j];
    if (detect && (gj == 0.0 || !(d >= tau2 * gj))) { deg = 1; break; }
    const double rinv = rcp_fast(d > 0.0 ? d : 1e-300);
    const double lij = row[j] * rinv;
#pragma unroll
    for (int k = j + 1; k < R; k++)
      if (i >= k && i < R) row[k] = fma(-lij, o.col[k], row[k]);
    if (i > j) row[j] = lij;
    if (i == j) { o.D[j] = d; row[j] = 1.0; }
    __syncwarp();
  }
  if (!deg && i < R) {
#pragma unroll
    for (int k = 0; k < R; k++) o.L[i * LD + k] = (k <= i) ? row[k] : 0.0;
    o.dinv[i] = 1.0 / sqrt(o.D[i]);
  }
  __syncwarp();
  return deg;
}

// o.Li = D^-1/2 L^-1 for the unit lower L; kappa = ||L D^1/2||_F ||D^-1/2 L^-1||_F
// (>= cond_2(P)).  Warp 0; lane c owns column c of L^-1.
template <int R>
__device__ void inverse_warp(OrthW& o) {
  const int c = threadIdx.x & 31;
  double col[R];
#pragma unroll
  for (int i = 0; i < R; i++) {
    double v0 = (i == c) ? 1.0 : 0.0, v1 = 0.0;   // two chains for ILP
#pragma unroll
    for (int k = 0; k < i; k++) {
      if (k & 1) v1 = fma(-o.L[i * LD + k], col[k], v1);
      else v0 = fma(-o.L[i * LD + k], col[k], v0);
    }
    col[i] = (i >= c && c < R) ? v0 + v1 : 0.0;
  }
  // D^-1/2 of every column, computed in parallel and broadcast through o.col
  if (c < R) o.col[c] = 1.0 / sqrt(o.D[c] > 0.0 ? o.D[c] : 1e-300);
  __syncwarp();
  const double sdc = (c < R) ? sqrt(o.D[c] > 0.0 ? o.D[c] : 0.0) : 0.0;
  double nl = 0.0, ni = 0.0;
  if (c < R) {
#pragma unroll
    for (int i = 0; i < R; i++) {
      const double v = col[i] * o.col[i];
      o.Li[i * LD + c] = v;
      ni = fma(v, v, ni);
      const double lc = o.L[i * LD + c] * sdc;   // (L D^1/2)[i][c]
      nl = fma(lc, lc, nl);
    }
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    nl += __shfl_xor_sync(0xffffffffu, nl, off);
    ni += __shfl_xor_sync(0xffffffffu, ni, off);
  }
  if (c == 0) o.kappa = sqrt(nl) * sqrt(ni);
  __syncwarp();
}

// Up-looking LDL^T with column substitution (slow path, thread 0): the Gram of
// the modified column set c_j = rep[j] ? f_j : p_j is read from o.L (P^T P),
// o.X (P^T F) and o.Y (F^T F); a column failing the test is replaced once.
template <int R>
__device__ __noinline__ void ldl_subst(OrthW& o, double tau2) {
  if (threadIdx.x != 0) return;
  double* Lt = o.Li;  // scratch; o.L keeps P^T P until the end
  for (int x = 0; x < 32 * LD; x++) Lt[x] = 0.0;
  for (int j = 0; j < R; j++) o.rep[j] = 0;
  auto gram = [&](int a, int b) -> double {
    const bool ra = o.rep[a], rb = o.rep[b];
    if (!ra && !rb) return o.L[a * LD + b];
    if (!ra && rb) return o.X[a * LD + b];
    if (ra && !rb) return o.X[b * LD + a];
    return o.Y[a * LD + b];
  };
  for (int i = 0; i < R; i++) {
    for (int attempt = 0; attempt < 2; attempt++) {
      for (int k = 0; k < i; k++) {
        double v = gram(i, k);
        for (int l = 0; l < k; l++) v -= Lt[i * LD + l] * o.D[l] * Lt[k * LD + l];
        Lt[i * LD + k] = v / o.D[k];
      }
      const double g = gram(i, i);
      double d = g;
      for (int k = 0; k < i; k++) d -= Lt[i * LD + k] * Lt[i * LD + k] * o.D[k];
      if (attempt == 0 && (g == 0.0 || !(d >= tau2 * g))) { o.rep[i] = 1; continue; }
      o.D[i] = d > 0.0 ? d : 1e-300;
      Lt[i * LD + i] = 1.0;
      break;
    }
  }
  for (int x = 0; x < 32 * LD; x++) o.L[x] = Lt[x];
  for (int j = 0; j < R; j++) o.dinv[j] = 1.0 / sqrt(o.D[j]);
}

// P_hat rows = D^-1/2 L^-1 P[i] by forward substitution with the unit lower
// L of G = L D L^T (no explicit inverse on the critical path).  One thread
// per row, threads [t0, blockDim) (warp 0 is busy with the kappa estimate).
// On the slow path ps already holds P_m (substituted columns replaced by their
// fallback vectors, orth_slow).  fp64, rounded to fp32.
template <int R>
__device__ void band_solve(const float* ps, float* out, int nr, const OrthW& o, int t0) {
  constexpr int RP = K<R>::RP;
  for (int i = (int)threadIdx.x - t0; i < nr && i >= 0; i += (int)blockDim.x - t0) {
    double x[R];
#pragma unroll
    for (int a = 0; a < R; a++) {
      double v0 = (double)ps[i * RP + a];
      double v1 = 0.0;
#pragma unroll
      for (int b = 0; b < a; b++) {
        if (b & 1) v1 = fma(-o.L[a * LD + b], x[b], v1);
        else v0 = fma(-o.L[a * LD + b], x[b], v0);
      }
      x[a] = v0 + v1;
    }
#pragma unroll
    for (int a = 0; a < R; a++) out[i * RP + a] = (float)(x[a] * o.dinv[a]);
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

// ------------------------------------------------------------------ cold paths
// Out of line (see the kernel's phase 3): taken only when a column is
// degenerate (reading C3) or the first pass is ill conditioned (reading C5).

// Slow path of the degenerate-column test: every column's fallback vector
// enters an augmented Gram (X = P^T F, Y = F^T F, one partial per row band,
// one extra grid barrier), the up-looking LDL^T with substitution decides
// which columns are replaced, and the band's P columns that are replaced are
// overwritten with their fallback vectors (P_m), so the solve is the common one.
template <int R>
__device__ __noinline__ void orth_slow(const Params2& p, Tile T, OrthW& o, float* ps, float* ps2, double* gscr,
                                       unsigned epoch, bool active) {
  constexpr int RP = K<R>::RP;
  const int tid = threadIdx.x;
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
  grid_barrier(p.bar, epoch * gridDim.x);
  reduce_partials<R>(p.G_band, p.nr, o, gscr);
  for (int q = tid; q < 2 * R * R; q += NT) {
    double gg = 0.0;
    for (int u = 0; u < p.nr; u++) gg += __ldcg(p.XY_band + (size_t)u * 2 * R * R + q);
    const int a = (q / R) % R, b = q % R;
    if (q < R * R) o.X[a * LD + b] = gg; else o.Y[a * LD + b] = gg;
  }
  __syncthreads();
  ldl_subst<R>(o, p.tau * p.tau);
  __syncthreads();
  if (active) {
    for (int x = tid; x < T.th * RP; x += NT) {
      const int a = x % RP;
      if (a < R && o.rep[a]) ps[x] = fallback_entry(p.fb_seed, a, T.row0 + x / RP);
    }
  }
}

// CholQR2 (reading C5): orthonormalise the fp32-rounded P_hat in ps once more.
template <int R>
__device__ __noinline__ void second_pass(const Params2& p, Tile T, OrthW& o, float* ps, float* ps2, double* gscr,
                                         unsigned epoch, bool active) {
  constexpr int RP = K<R>::RP, NP = K<R>::NP;
  if (active && T.cb == 0) band_gram<R>(ps, T.th, p.G2_band + (size_t)T.rb * NP, gscr);
  grid_barrier(p.bar, epoch * gridDim.x);
  reduce_partials<R>(p.G2_band, p.nr, o, gscr);
  __syncthreads();
  if (threadIdx.x < 32) ldl_warp<R>(o, 0.0, false);
  __syncthreads();
  if (active) {
    band_solve<R>(ps, ps2, T.th, o, 0);
    __syncthreads();
    for (int x = threadIdx.x; x < T.nrblk * 8 * RP; x += NT) ps[x] = (x / RP < T.th) ? ps2[x] : 0.f;
  }
  __syncthreads();
}

#include "occ_v2_kernel.cuh"

// ------------------------------------------------------------------ host side
struct Plan2 {
  bool ok = false;
  int nr = 0, nc = 0, H = 0, W = 0, ns = 0, sw = 0;
  int off_stm = 0, off_ste = 0, off_qs = 0, off_red = 0, off_pa = 0, off_pb = 0, off_orth = 0, off_ps = 0, off_gs = 0;
  int off_qsm = 0;
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
    pl.sw = W + ((8 - W % 32) + 32) % 32;   // = 8 (mod 32) floats: conflict-free 8-byte fragment reads
    const int stage_bytes = SR * pl.sw * 4;
    constexpr bool QREG = (R <= 16);
    constexpr int KREG = QREG ? (R <= 8 ? 8 : 4) : 1;
    if (QREG && (W / 8 + NCW - 1) / NCW > KREG) continue;   // Q_prev fragments must fit the registers
    const int qs_bytes = QREG ? 0 : al128(W * RP * 4);
    const int red_bytes = al128(NCW * ((H + 7) / 8 * 8) * RP * 4);   // per-warp P partials of every tile row
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
    pl.off_qsm = off; off += al128(W * R * 4);   // phase-5 Q slice
    pl.total = std::max(p1, off);
    if (pl.total > smem_cap) continue;
    const int cgw = (ncg + NCW - 1) / NCW;
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
  p.off_qsm = pl.off_qsm;
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
  p.trace = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(p1.bar) + kTraceOffset);
  p.stats = p1.stats;
  p.fb_seed = p1.fb_seed;
  p.tau = p1.tau;
  p.kappa_thr = p1.kappa_thr;
  p.force_two_pass = p1.force_two_pass;
  {
    const char* dbg = getenv("OCC_V2_DEBUG");
    p.debug = dbg ? atoi(dbg) : 0;
  }
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
  return a((size_t)pl.nc * n * R * 4) + a((size_t)pl.nr * m * R * 4) + a((size_t)pl.nr * NP * 8) + a((size_t)pl.nr * NP * 8) +
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
