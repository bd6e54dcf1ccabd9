// occ_v2_la.cuh -- small fp64 linear algebra of the fused step (reading C3-C5,
// C20): the Gram partials and their reduction, the warp-level LDL^T, the
// explicit D^-1/2 L^-1 with the conditioning estimates, the slow-path LDL with
// column substitution, and the row solves.  Included by occ_v2.cu and by the
// single-warp micro-benchmark tools/la_bench.cu.
#pragma once
#include "occ_v2.cuh"

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
  int prog;             // R + 2: Li, kappa, amp ready; -1: degenerate column (phase 3 protocol)
  double kappa;
  double amp;           // ||S Li^T||_F, S = diag(||p_j||): error amplification of Q = (A^T P) Li^T
};

struct SyncAll {
  __device__ __forceinline__ void operator()() const { __syncthreads(); }
};
struct SyncCompute {   // the NCW compute warps 0 .. NCW-1 (named barrier 1)
  __device__ __forceinline__ void operator()() const { asm volatile("bar.sync 1, %0;" ::"r"(NCW * 32) : "memory"); }
};
// Phase-3 warp groups: A = compute warps off warp NW-1's scheduler (w % 4 != 3),
// B = the compute warps that share it (w % 4 == 3).  Named barriers 2 and 4.
constexpr int NWA = NCW - NCW / 4, NWB = NCW / 4;
__device__ __forceinline__ bool in_group_a(int w) { return w < NCW && (w & 3) != 3; }
__device__ __forceinline__ int group_a_index() {   // dense 0 .. 32 NWA - 1
  const int w = threadIdx.x >> 5;
  return (w - (w >> 2)) * 32 + (threadIdx.x & 31);
}
__device__ __forceinline__ int group_b_index() { return (threadIdx.x >> 7) * 32 + (threadIdx.x & 31); }
struct SyncGroupA {
  __device__ __forceinline__ void operator()() const { asm volatile("bar.sync 2, %0;" ::"r"(NWA * 32) : "memory"); }
};
struct SyncGroupB {
  __device__ __forceinline__ void operator()() const { asm volatile("bar.sync 4, %0;" ::"r"(NWB * 32) : "memory"); }
};

// out[e] = sum_{u < S} src[u * stride + e], e < E, in a fixed order (deterministic),
// by the threads x in [0, nthr) of a group synchronised by sync().  Every thread
// keeps 8 independent loads in flight (the partial sums live in L2 and this is
// latency bound; 8 rather than 16 halves the code, which runs once per call
// from a cold instruction cache).  scratch: nthr elements of shared memory.
template <typename Tv, typename Fout, typename Sync = SyncAll>
__device__ void strided_sum(const Tv* __restrict__ src, size_t stride, int S, int E, Tv* scratch, Fout&& out,
                            int x = threadIdx.x, int nthr = NT, Sync sync = Sync()) {
  for (int e0 = 0; e0 < E; e0 += nthr) {
    const int En = min(nthr, E - e0);
    const int C = max(1, nthr / En);
    Tv acc = Tv(0);
    if (x < En * C) {
      const int e = e0 + x % En, c = x / En;
      for (int u0 = c; u0 < S; u0 += 8 * C) {
        Tv v[8];
#pragma unroll
        for (int j = 0; j < 8; j++) {
          const int u = u0 + j * C;
          v[j] = (u < S) ? __ldcg(src + (size_t)u * stride + e) : Tv(0);
        }
#pragma unroll
        for (int j = 0; j < 8; j++) acc += v[j];
      }
    }
    sync();
    if (x < En * C) scratch[x] = acc;
    sync();
    if (x < En) {
      Tv r = Tv(0);
      for (int c = 0; c < C; c++) r += scratch[c * En + x];
      out(e0 + x, r);
    }
    sync();
  }
}

// G (packed upper triangle, nparts partials) -> o.L (full symmetric), o.gdiag.  All threads.
template <int R, typename Sync = SyncAll>
__device__ void reduce_partials(const double* __restrict__ part, int nparts, OrthW& o, double* scratch,
                                int x = threadIdx.x, int nthr = NT, Sync sync = Sync()) {
  constexpr int NP = K<R>::NP;
  strided_sum<double>(
      part, NP, nparts, NP, scratch,
      [&](int q, double gsum) {
        int a = 0, rem = q;
        while (rem >= R - a) { rem -= R - a; a++; }
        const int b = a + rem;
        o.L[a * LD + b] = gsum;
        o.L[b * LD + a] = gsum;
        if (a == b) o.gdiag[a] = gsum;
      },
      x, nthr, sync);
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

// ldl_warp publish protocol: o.prog is written with st.release.cta after the
// step's shared stores (made visible to lane 0 by __syncwarp) and read with
// ld.acquire.cta by the solvers.
__device__ __forceinline__ void prog_release(OrthW& o, int v) {
  asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&o.prog)), "r"(v)
               : "memory");
}
__device__ __forceinline__ int prog_acquire(const OrthW& o) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(&o.prog))
               : "memory");
  return v;
}

// Warp-level right-looking LDL^T of the Gram in o.L (R <= 32), square-root free
// so the sequential chain per column is one fp64 reciprocal.  Lane i holds the
// active part of row i in registers, SHIFTED: at step j, rr[k] = a_{i, j+k}; the
// update writes rr[k-1] = rr[k] - l_ij a_{j+k, j}, so the pivot is always rr[0]
// and every register index is static while the step loop stays rolled (this
// code runs once per call, usually from a cold instruction cache: its size is
// part of its latency; tools/la_bench.cu).  Column j (unscaled) is broadcast
// through o.col; L (unit lower) is stored into o.L column by column.  detect:
// stop at the first column whose squared residual D_j is below tau2 * its own
// squared norm (reading C3: the MGS test ||v|| < tau ||p_j||) and return 1 (o.L
// is then partially overwritten; callers re-reduce it).  publish: advance o.prog
// after every column (kept for experiments; the hot path uses the unrolled form).
template <int R>
__device__ int ldl_warp(OrthW& o, double tau2, bool detect, bool publish = false) {
  const int i = threadIdx.x & 31;
  double rr[R];
#pragma unroll
  for (int k = 0; k < R; k++) rr[k] = (i < R) ? o.L[i * LD + k] : 0.0;
  if (publish && R <= 16) {   // rows R..31 of o.L read as zero by a row solver trailing the factorisation
    for (int x = i; x < (32 - R) * LD; x += 32) o.L[R * LD + x] = 0.0;
  }
  int deg = 0;
#pragma unroll 1
  for (int j = 0; j < R; j++) {
    if (i >= j && i < R) o.col[i] = rr[0];   // a_ij of the current Schur complement
    __syncwarp();
    const double d = o.col[j];
    const double gj = o.gdiag[j];
    double cv[R - 1];
    const double* cj = o.col + j;   // o.col has 32 entries: j + k <= 2R - 2 < 32 (R <= 16) or is past
#pragma unroll                      // the active part, whose rr entries are shifted out unused
    for (int k = 1; k < R; k++) cv[k - 1] = (R <= 16 || j + k < 32) ? cj[k] : 0.0;   // a_{j+k, j}
    if (detect && (gj == 0.0 || !(d >= tau2 * gj))) { deg = 1; break; }
    const double lij = (i > j && i < R) ? rr[0] * rcp_fast(d > 0.0 ? d : 1e-300) : 0.0;
#pragma unroll
    for (int k = 1; k < R; k++) rr[k - 1] = fma(-lij, cv[k - 1], rr[k]);
    rr[R - 1] = 0.0;
    if (i > j && i < R) o.L[i * LD + j] = lij;
    if (i == j) o.D[j] = d;
    __syncwarp();
    if (publish && i == 0) prog_release(o, j + 1);
  }
  if (!deg && i < R) {
#pragma unroll 1
    for (int k = i; k < R; k++) o.L[i * LD + k] = (k == i) ? 1.0 : 0.0;
    o.dinv[i] = 1.0 / sqrt(o.D[i]);
  }
  __syncwarp();
  if (publish && i == 0) prog_release(o, deg ? -1 : R + 1);
  return deg;
}

// o.Li = D^-1/2 L^-1 for the unit lower L; kappa = ||L D^1/2||_F ||D^-1/2 L^-1||_F
// (>= cond_2(P)), amp = ||S Li^T||_F with S = diag(sqrt(G_jj)).  One warp;
// lane c forms column c of L^-1 by forward substitution in place in o.Li
// (conflict-free: lanes touch consecutive words of a row).  Compact rolled
// loops: on the fused path this runs off the critical path.
template <int R>
__device__ void inverse_warp(OrthW& o) {
  const int c = threadIdx.x & 31;
  double* X = o.Li;
  if (c < R) {
#pragma unroll 1
    for (int i = 0; i < R; i++) {
      double v0 = (i == c) ? 1.0 : 0.0, v1 = 0.0;
#pragma unroll 2
      for (int k = c; k < i; k++) {
        if (k & 1) v1 = fma(-o.L[i * LD + k], X[k * LD + c], v1);
        else v0 = fma(-o.L[i * LD + k], X[k * LD + c], v0);
      }
      X[i * LD + c] = (i >= c) ? v0 + v1 : 0.0;
    }
  }
  double nl = 0.0, ni = 0.0, na = 0.0;
  if (c < R) {
    const double sdc = sqrt(o.D[c] > 0.0 ? o.D[c] : 0.0);
#pragma unroll 1
    for (int i = 0; i < R; i++) {
      const double v = X[i * LD + c] * o.dinv[i];
      X[i * LD + c] = v;
      ni = fma(v, v, ni);
      const double lc = o.L[i * LD + c] * sdc;   // (L D^1/2)[i][c]
      nl = fma(lc, lc, nl);
    }
    na = o.gdiag[c] * ni;   // ||p_c||^2 * ||Li[:, c]||^2
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    nl += __shfl_xor_sync(0xffffffffu, nl, off);
    ni += __shfl_xor_sync(0xffffffffu, ni, off);
    na += __shfl_xor_sync(0xffffffffu, na, off);
  }
  if (c == 0) {
    o.kappa = sqrt(nl) * sqrt(ni);
    o.amp = sqrt(na);
  }
  __syncwarp();
}

// The same factorisation fully unrolled (register rows, static indices): the
// dynamic instruction count is ~35% lower than the rotated loop's (3.9k vs
// 6.0k cycles for R = 16, tools/la_bench.cu), at ~1.2k more instructions of
// code.  Used on the hot path (publishes only a degenerate column; Li, kappa
// and amp are published by inverse_warp_unrolled); same
// results as ldl_warp.
template <int R>
__device__ int ldl_warp_unrolled(OrthW& o, double tau2, bool detect) {
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
    if (i > j && i < R) {
      row[j] = lij;
      o.L[i * LD + j] = lij;
    }
    if (i == j) { o.D[j] = d; row[j] = 1.0; }
    __syncwarp();   // (no per-step publish: the other warps wait for Li, o.prog = R + 2)
  }
  if (!deg && i < R) {
#pragma unroll
    for (int k = 0; k < R; k++) o.L[i * LD + k] = (k <= i) ? row[k] : 0.0;
    o.dinv[i] = 1.0 / sqrt(o.D[i]);
  }
  __syncwarp();
  if (deg && i == 0) prog_release(o, -1);
  return deg;
}

// inverse_warp fully unrolled (column c of L^-1 in lane c's registers): ~2.5k
// cycles for R = 16 against ~11k for the rolled loop (tools/la_bench.cu); used
// on the hot path, right after the factorisation.  Then publishes o.prog = R + 2.
template <int R>
__device__ void inverse_warp_unrolled(OrthW& o) {
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
  const double sdc = (c < R) ? sqrt(o.D[c] > 0.0 ? o.D[c] : 0.0) : 0.0;
  double nl = 0.0, ni = 0.0;
  if (c < R) {
#pragma unroll
    for (int i = 0; i < R; i++) {
      const double v = col[i] * o.dinv[i];
      o.Li[i * LD + c] = v;
      ni = fma(v, v, ni);
      const double lc = o.L[i * LD + c] * sdc;   // (L D^1/2)[i][c]
      nl = fma(lc, lc, nl);
    }
  }
  double na = (c < R) ? o.gdiag[c] * ni : 0.0;   // ||p_c||^2 * ||Li[:, c]||^2
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    nl += __shfl_xor_sync(0xffffffffu, nl, off);
    ni += __shfl_xor_sync(0xffffffffu, ni, off);
    na += __shfl_xor_sync(0xffffffffu, na, off);
  }
  if (c == 0) {
    o.kappa = sqrt(nl) * sqrt(ni);
    o.amp = sqrt(na);
  }
  __syncwarp();
  if (c == 0) prog_release(o, R + 2);
}

// Fused path (reading C20): rows -> D^-1/2 L^-1 rows = rows Li^T with the
// explicit Li, for the H8 rows of the P band (rows >= th zero; -> P_hat) and
// the nqc rows of the reduced Q~ slice (-> Q).  4 threads per row, each forming
// the outputs k = kg, kg+4, ...: independent dot products (full ILP), fp64.
// Threads [0, nthr).
template <int R>
__device__ __forceinline__ void apply_li(const float* ps, int H8, int th, const float* qt, int nqc, const OrthW& o,
                                         float* phat, float* qout, int x0, int nthr) {
  constexpr int RP = K<R>::RP, KPT = (R + 3) / 4;
  for (int x = x0; x < (H8 + nqc) * 4; x += nthr) {
    const int it = x >> 2, kg = x & 3;
    const bool isP = it < H8;
    const float* src = isP ? ps + (size_t)it * RP : qt + (size_t)(it - H8) * R;
    const bool zero = isP && it >= th;
    double xv[R];
#pragma unroll
    for (int j = 0; j < R; j++) xv[j] = zero ? 0.0 : (double)src[j];
    float* dst = isP ? phat + (size_t)it * RP : qout + (size_t)(it - H8) * R;
#pragma unroll
    for (int s2 = 0; s2 < KPT; s2++) {
      const int k = kg + 4 * s2;
      if (k >= R) break;
      const double* li = o.Li + k * LD;
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int j = 0; j < R; j++) {   // Li is lower triangular: the j > k terms are zero
        if (j & 1) a1 = fma(xv[j], li[j], a1);
        else a0 = fma(xv[j], li[j], a0);
      }
      dst[k] = (float)(a0 + a1);
    }
  }
}

// Wait until ldl_warp (publish mode) has passed step `a` (o.prog >= a); returns
// false if it stopped at a degenerate column.  `seen` caches the last value
// read, so steps the factorisation is already past cost no shared load.
__device__ __forceinline__ bool wait_prog(const OrthW& o, int a, int& seen) {
  while (seen < a && seen >= 0) {
    seen = prog_acquire(o);
    if (seen < a && seen >= 0) __nanosleep(16);
  }
  return seen >= 0;
}
__device__ __forceinline__ bool wait_prog(const OrthW& o, int a) {
  int seen = 0;
  return wait_prog(o, a, seen);
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
// per row, threads [t0, t0 + nthr).
// On the slow path ps already holds P_m (substituted columns replaced by their
// fallback vectors, orth_slow).  fp64, rounded to fp32.
template <int R>
__device__ void band_solve(const float* ps, float* out, int nr, const OrthW& o, int t0, int nthr) {
  constexpr int RP = K<R>::RP;
  for (int i = (int)threadIdx.x - t0; i < nr && i >= 0 && (int)threadIdx.x < t0 + nthr; i += nthr) {
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

// fp64 tensor-core MMA, D(8x8) += A(8x4) B(4x8); lane l holds A[l/4][l%4],
// B[l%4][l/4], D[l/4][2(l%4)], D[l/4][2(l%4)+1].
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// Gram partial (packed upper triangle) of rows [0,nr) of an fp32 [.][RP] array
// (RP = 8 MT8; rows >= nr of the array are zero up to a multiple of 4), fp64 on
// the tensor cores (DMMA), by ONE warp while the other warps compute Q_part.
// G = P^T P: A = P^T, B = P; tile (mi, nj) of 8x8, mi <= nj; two accumulator
// sets (even / odd k-steps).  Fixed order: deterministic.
template <int R>
__device__ void band_gram_warp(const float* ps, int nr, double* part) {
  constexpr int RP = K<R>::RP, T8 = RP / 8, NT8 = T8 * (T8 + 1) / 2;
  const int lane = threadIdx.x & 31, gq = lane >> 2, tq = lane & 3;
  double acc[2][NT8][2];
#pragma unroll
  for (int h = 0; h < 2; h++)
#pragma unroll
    for (int u = 0; u < NT8; u++) acc[h][u][0] = acc[h][u][1] = 0.0;
  const int nk = (nr + 3) / 4;
  for (int ks = 0; ks < nk; ks++) {
    const int row = 4 * ks + tq;   // K index of this lane
    double v[T8];                   // P[row][8 t + gq]: A-fragment of tile t, and B-fragment of tile t
#pragma unroll
    for (int t8 = 0; t8 < T8; t8++) v[t8] = (row < nr) ? (double)ps[row * RP + 8 * t8 + gq] : 0.0;
    int u = 0;
#pragma unroll
    for (int mi = 0; mi < T8; mi++)
#pragma unroll
      for (int nj = mi; nj < T8; nj++, u++) dmma(acc[ks & 1][u], v[mi], v[nj]);
  }
  int u = 0;
#pragma unroll
  for (int mi = 0; mi < T8; mi++)
#pragma unroll
    for (int nj = mi; nj < T8; nj++, u++)
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int a = 8 * mi + gq, b = 8 * nj + 2 * tq + h;
        if (a <= b && b < R) part[a * R - a * (a - 1) / 2 + (b - a)] = acc[0][u][h] + acc[1][u][h];
      }
}

}  // namespace v2
}  // namespace occ
