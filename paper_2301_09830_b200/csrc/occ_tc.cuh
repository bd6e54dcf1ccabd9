// occ_tc.cuh -- tensor-core sweeps of the per-phase path (phases A and D of
// occ_kernels.cuh), for the shapes the fused kernel does not take (r = 64,
// tiles larger than on-chip memory: BASELINE configs[2] and configs[3]).
//
//   A  P_part[s][i][k] = sum_{c in split s} A[i][c] Q_prev[c][k]      (a1, a2)
//   D  Q_part[s][c][k] = sum_{i in split s} A[i][c] P_hat[i][k]       (a1, a5)
//
// Both run on mma.sync.m16n8k8 TF32 with the 3-term split (A_hi B_hi + A_hi
// B_lo + A_lo B_hi: fp32-level accuracy, as the fused kernel).  A = M + e is
// read straight from HBM into registers with 128-bit loads (no staging): the
// contraction index is permuted so that a lane's fragment is 4 consecutive
// elements of one row.  Each warp owns whole output rows of its tile (16 rows
// of P in A, 32 columns of Q in D) and runs the whole reduction of its split
// over them, so there is no cross-warp reduction.  The small operand (the
// Q_prev slab in A, the P_hat rows in D) is split into hi / lo once per tile
// and staged in shared memory in fragment order (two 16-byte loads per
// fragment, conflict free).  Loads run PD steps ahead in registers.
//
// Index maps (legal permutations of a contraction or output index, applied to
// both operands / undone at the store):
//   A: m = row (g, g+8); k-step pair over 16 columns: k-step 0 uses columns
//      4t, 4t+1 (k = t, t+4), k-step 1 columns 4t+2, 4t+3.
//   D: k = row (t, t+4 of an 8-row step); m over 32 columns: m-tile 0 has
//      m = g <-> column 4g, m = g+8 <-> 4g+1; m-tile 1 columns 4g+2, 4g+3.
#pragma once
#include "occ_kernels.cuh"

#include <type_traits>

namespace occ {
namespace tc {

__device__ __forceinline__ void split_tf32(float x, unsigned& hi, unsigned& lo) {
  hi = __float_as_uint(x) & 0xffffe000u;
  lo = __float_as_uint(x - __uint_as_float(hi));
}
__device__ __forceinline__ void mma1(float (&d)[4], unsigned a0, unsigned a1, unsigned a2, unsigned a3, unsigned b0,
                                     unsigned b1) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// d += A . B, A = (ah + al), B = (bh + bl), al.bl dropped; small terms first
__device__ __forceinline__ void mma3x(float (&d)[4], const unsigned (&ah)[4], const unsigned (&al)[4], unsigned bh0,
                                      unsigned bh1, unsigned bl0, unsigned bl1) {
  mma1(d, al[0], al[1], al[2], al[3], bh0, bh1);
  mma1(d, ah[0], ah[1], ah[2], ah[3], bl0, bl1);
  mma1(d, ah[0], ah[1], ah[2], ah[3], bh0, bh1);
}
__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}

// 4 consecutive elements of A = M + e at (row i, column c) (c % 4 == 0), or 0.
// Loaded raw (ldA4) and combined only when consumed (val): a load whose value
// is used right away stalls the warp on HBM latency, so the sweeps keep PD
// steps of raw loads in flight and add M + e at the step that uses them.
struct A4 {
  float4 m;   // fp32 M, or bf16 M in m.x, m.y (4 values)
  float4 e;
};
template <bool MBF>
__device__ __forceinline__ A4 ldA4(const Params& p, int i, int c, bool ok) {
  A4 a;
  a.m = make_float4(0.f, 0.f, 0.f, 0.f);
  a.e = a.m;
  if (!ok) return a;
  if (MBF) {
    const uint2 raw = __ldcs(reinterpret_cast<const uint2*>(reinterpret_cast<const __nv_bfloat16*>(p.M) +
                                                            (size_t)i * p.ldm + c));
    a.m.x = __uint_as_float(raw.x);
    a.m.y = __uint_as_float(raw.y);
  } else {
    a.m = __ldcs(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(p.M) + (size_t)i * p.ldm + c));
  }
  if (p.err_in) a.e = __ldcs(reinterpret_cast<const float4*>(p.err_in + (size_t)i * p.lde_in + c));
  return a;
}
template <bool MBF>
__device__ __forceinline__ float4 val(const A4& a) {
  float4 m = a.m;
  if (MBF) {
    const unsigned x = __float_as_uint(a.m.x), y = __float_as_uint(a.m.y);
    const float2 f0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&x));
    const float2 f1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&y));
    m = make_float4(f0.x, f0.y, f1.x, f1.y);
  }
  return add4(m, a.e);
}

template <int R>
struct TcCfg {
  static constexpr int NTL = (R + 7) / 8;     // n-tiles of 8 over the rank (R = 4: one, half zero)
  static constexpr int A_ROWS = 16 * NW;      // phase A: rows per unit (one m-tile per warp)
  static constexpr int D_COLS = 32 * NW;      // phase D: columns per unit (two m-tiles per warp)
  static constexpr int PD = (R <= 16) ? 4 : 6;   // steps of raw loads in flight per warp (one CTA of 8 warps per SM)
};

// shared memory of phase A for a split of width cs1: the Q slab fragments
template <int R>
__host__ __device__ constexpr size_t smem_A_tc(int cs1) {
  return (size_t)((cs1 + 15) / 16) * TcCfg<R>::NTL * 32 * 32;
}
// phase D for splits of rs2 rows: the P_hat fragments
template <int R>
__host__ __device__ constexpr size_t smem_D_tc(int rs2) {
  return (size_t)((rs2 + 7) / 8) * TcCfg<R>::NTL * 32 * 16;
}

// ------------------------------------------------------------------ phase A
template <int R, bool MBF>
__device__ void phase_A_tc(const Params& p, unsigned char* smraw) {
  constexpr int NT = TcCfg<R>::NTL, UR = TcCfg<R>::A_ROWS, PD = TcCfg<R>::PD;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  uint4* qh = reinterpret_cast<uint4*>(smraw);   // [kc][nt][lane]: hi(q0..q3); then lo in the same order
  uint4* ql = qh + (size_t)((p.cs1 + 15) / 16) * NT * 32;
  const int nrb = (p.n + UR - 1) / UR;
  const int units = nrb * p.s1;
  for (int u = blockIdx.x; u < units; u += gridDim.x) {
    const int rb = u % nrb, s = u / nrb;
    const int c0 = s * p.cs1, cw = min(p.cs1, p.m - c0);
    const int nkc = (cw + 15) / 16;
    const int r0 = rb * UR + 16 * warp;
    const bool ok0 = r0 + g < p.n, ok1 = r0 + g + 8 < p.n;
    __syncthreads();   // the previous unit's readers are done with the slab
    // the first PD steps of A are independent of the slab: in flight during the fill
    A4 buf[PD][2];
#pragma unroll
    for (int sgi = 0; sgi < PD; sgi++) {
      const int c = 16 * sgi + 4 * t;
      buf[sgi][0] = ldA4<MBF>(p, r0 + g, c0 + c, ok0 && c < cw);
      buf[sgi][1] = ldA4<MBF>(p, r0 + g + 8, c0 + c, ok1 && c < cw);
    }
    // Q_prev slab (cw x R, contiguous): coalesced 16-byte loads, then scattered
    // into fragment order: Q[c][k] -> entry (kc = c/16, nt = k/8, lane (k%8, (c%16)/4)), q = c%4
    {
      unsigned* qh32 = reinterpret_cast<unsigned*>(qh);
      unsigned* ql32 = reinterpret_cast<unsigned*>(ql);
      const int nvec = nkc * 16 * NT * 2;   // float4 of the zero-padded [16 nkc][8 NT] slab
      for (int x = threadIdx.x; x < nvec; x += occ::NT) {
        const int cc = x / (NT * 2), k0 = 4 * (x % (NT * 2));
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (cc < cw && k0 < R) v = __ldg(reinterpret_cast<const float4*>(p.Qprev + (size_t)(c0 + cc) * R + k0));
        const float vv[4] = {v.x, v.y, v.z, v.w};
        const int kc = cc >> 4, tt = (cc & 15) >> 2, q = cc & 3;
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const int k = k0 + j, nt = k >> 3, gg = k & 7;
          const size_t e = ((((size_t)kc * NT + nt) * 32) + gg * 4 + tt) * 4 + q;
          unsigned h, l;
          split_tf32(vv[j], h, l);
          qh32[e] = h;
          ql32[e] = l;
        }
      }
    }
    __syncthreads();
    float acc[NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; nt++) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.f;
    for (int kc0 = 0; kc0 < nkc; kc0 += PD) {
#pragma unroll
      for (int sgi = 0; sgi < PD; sgi++) {
        const int kc = kc0 + sgi;
        const float4 v0 = val<MBF>(buf[sgi][0]), v1 = val<MBF>(buf[sgi][1]);
        {   // prefetch step kc + PD into this slot
          const int c = 16 * (kc + PD) + 4 * t;
          buf[sgi][0] = ldA4<MBF>(p, r0 + g, c0 + c, ok0 && c < cw);
          buf[sgi][1] = ldA4<MBF>(p, r0 + g + 8, c0 + c, ok1 && c < cw);
        }
        if (kc < nkc) {
          // k-step 0: columns 4t (k = t), 4t+1 (k = t+4); k-step 1: 4t+2, 4t+3
          unsigned h0[4], l0[4], h1[4], l1[4];
          split_tf32(v0.x, h0[0], l0[0]); split_tf32(v1.x, h0[1], l0[1]);
          split_tf32(v0.y, h0[2], l0[2]); split_tf32(v1.y, h0[3], l0[3]);
          split_tf32(v0.z, h1[0], l1[0]); split_tf32(v1.z, h1[1], l1[1]);
          split_tf32(v0.w, h1[2], l1[2]); split_tf32(v1.w, h1[3], l1[3]);
          const size_t o = (size_t)kc * NT * 32 + lane;
#pragma unroll
          for (int nt = 0; nt < NT; nt++) {
            const uint4 bh = qh[o + nt * 32], bl = ql[o + nt * 32];
            mma3x(acc[nt], h0, l0, bh.x, bh.y, bl.x, bl.y);
            mma3x(acc[nt], h1, l1, bh.z, bh.w, bl.z, bl.w);
          }
        }
      }
    }
    // D (row, k): c0 = (g, 8nt + 2t), c1 = (g, +1), c2 = (g + 8, 2t), c3 = (g + 8, +1)
    float* dst = p.P_part + ((size_t)s * p.n + r0) * R;
#pragma unroll
    for (int nt = 0; nt < NT; nt++) {
      const int k = 8 * nt + 2 * t;
      if (k >= R) continue;
      if (ok0) *reinterpret_cast<float2*>(dst + (size_t)g * R + k) = make_float2(acc[nt][0], acc[nt][1]);
      if (ok1) *reinterpret_cast<float2*>(dst + (size_t)(g + 8) * R + k) = make_float2(acc[nt][2], acc[nt][3]);
    }
  }
}

// ------------------------------------------------------------------ phase D
template <int R, bool MBF>
__device__ void phase_D_tc(const Params& p, unsigned char* smraw) {
  constexpr int NT = TcCfg<R>::NTL, CB = TcCfg<R>::D_COLS, PD = TcCfg<R>::PD;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  uint4* pf = reinterpret_cast<uint4*>(smraw);   // [ks][nt][lane]: hi(b0, b1), lo(b0, b1)
  const int ncb = (p.m + CB - 1) / CB;
  const int units = ncb * p.s2;
  for (int u = blockIdx.x; u < units; u += gridDim.x) {
    const int cb = u % ncb, s = u / ncb;
    const int r0 = s * p.rs2, nr = min(p.rs2, p.n - r0);
    const int nks = (nr + 7) / 8;
    const int cw0 = cb * CB + 32 * warp;   // this warp's 32 columns
    const int c = cw0 + 4 * g;
    const bool cok = c < p.m;              // m % 8 == 0: four columns in or out together
    __syncthreads();   // the previous unit's readers are done with the P_hat fragments
    A4 buf[PD][2];   // the first PD steps of A: in flight during the fill
#pragma unroll
    for (int sgi = 0; sgi < PD; sgi++) {
      const int i = 8 * sgi + t;
      buf[sgi][0] = ldA4<MBF>(p, r0 + i, c, cok && i < nr);
      buf[sgi][1] = ldA4<MBF>(p, r0 + i + 4, c, cok && i + 4 < nr);
    }
    // P_hat rows of the split (nr x R, contiguous): coalesced 16-byte loads, then
    // scattered into fragment order: P[i][k] -> entry (ks = i/8, nt = k/8, lane
    // (k%8, i%4)), component hi (i%8)/4 and lo 2 + (i%8)/4
    {
      unsigned* pf32 = reinterpret_cast<unsigned*>(pf);
      const int nvec = nks * 8 * NT * 2;
      for (int x = threadIdx.x; x < nvec; x += occ::NT) {
        const int i = x / (NT * 2), k0 = 4 * (x % (NT * 2));
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (i < nr && k0 < R) v = __ldcg(reinterpret_cast<const float4*>(p.P + (size_t)(r0 + i) * R + k0));
        const float vv[4] = {v.x, v.y, v.z, v.w};
        const int ks = i >> 3, tt = i & 3, which = (i & 7) >> 2;
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const int k = k0 + j, nt = k >> 3, gg = k & 7;
          const size_t e = ((((size_t)ks * NT + nt) * 32) + gg * 4 + tt) * 4;
          unsigned h, l;
          split_tf32(vv[j], h, l);
          pf32[e + which] = h;
          pf32[e + 2 + which] = l;
        }
      }
    }
    __syncthreads();
    float acc[2][NT][4];
#pragma unroll
    for (int mt = 0; mt < 2; mt++)
#pragma unroll
      for (int nt = 0; nt < NT; nt++) acc[mt][nt][0] = acc[mt][nt][1] = acc[mt][nt][2] = acc[mt][nt][3] = 0.f;
    for (int ks0 = 0; ks0 < nks; ks0 += PD) {
#pragma unroll
      for (int sgi = 0; sgi < PD; sgi++) {
        const int ks = ks0 + sgi;
        const float4 v0 = val<MBF>(buf[sgi][0]), v1 = val<MBF>(buf[sgi][1]);   // rows 8ks + t, 8ks + t + 4
        {
          const int i = 8 * (ks + PD) + t;
          buf[sgi][0] = ldA4<MBF>(p, r0 + i, c, cok && i < nr);
          buf[sgi][1] = ldA4<MBF>(p, r0 + i + 4, c, cok && i + 4 < nr);
        }
        if (ks < nks) {
          // m-tile 0: m = g <-> column 4g (.x), m = g+8 <-> 4g+1 (.y); m-tile 1: .z, .w
          // a0 = (m = g, k = t), a1 = (g + 8, t), a2 = (g, t + 4), a3 = (g + 8, t + 4)
          unsigned h0[4], l0[4], h1[4], l1[4];
          split_tf32(v0.x, h0[0], l0[0]); split_tf32(v0.y, h0[1], l0[1]);
          split_tf32(v1.x, h0[2], l0[2]); split_tf32(v1.y, h0[3], l0[3]);
          split_tf32(v0.z, h1[0], l1[0]); split_tf32(v0.w, h1[1], l1[1]);
          split_tf32(v1.z, h1[2], l1[2]); split_tf32(v1.w, h1[3], l1[3]);
          const uint4* pk = pf + (size_t)ks * NT * 32 + lane;
#pragma unroll
          for (int nt = 0; nt < NT; nt++) {
            const uint4 b = pk[nt * 32];
            mma3x(acc[0][nt], h0, l0, b.x, b.y, b.z, b.w);
            mma3x(acc[1][nt], h1, l1, b.x, b.y, b.z, b.w);
          }
        }
      }
    }
    // D (m, k): c0 = (g, 2t), c1 = (g, 2t+1), c2 = (g+8, 2t), c3 = (g+8, 2t+1); m-tile mt:
    // m = g <-> column 4g + 2mt, m = g + 8 <-> 4g + 2mt + 1
    if (cok) {
      float* dst = p.Q_part + ((size_t)s * p.m + c) * R;
#pragma unroll
      for (int mt = 0; mt < 2; mt++)
#pragma unroll
        for (int nt = 0; nt < NT; nt++) {
          const int k = 8 * nt + 2 * t;
          if (k >= R) continue;
          *reinterpret_cast<float2*>(dst + (size_t)(2 * mt) * R + k) = make_float2(acc[mt][nt][0], acc[mt][nt][1]);
          *reinterpret_cast<float2*>(dst + (size_t)(2 * mt + 1) * R + k) = make_float2(acc[mt][nt][2], acc[mt][nt][3]);
        }
    }
  }
}

// ------------------------------------------------------------------ phase F (DP)
// The data-parallel reconstruction on the tensor cores (occ_allreduce_factors,
// reading C1/C2/C15): M' = round(P_hat (scale Q_sum)^T) into G, e_new = A -
// P_hat Q_w^T (local convention, DPL) or A - M' (OCC_EF_GLOBAL), and the warm
// start Q <- scale Q_sum.  Unit = 128 rows x 64 columns; warp (wr, wc) owns
// rows 32 wr .. + 31 (two m-tiles) and columns 32 wc .. + 31 (four n-tiles).
// MMA: D[row][col] = sum_k P_hat[row][k] Q[col][k] (m = row, k = rank,
// n = column), n permuted so that a lane's outputs are 4 consecutive columns:
// in a 16-column group q, n-tile j = 2q + {0, 1} has n <-> column
// 16 q + 4 (n >> 1) + 2 j + (n & 1).  Both factors are staged per unit in
// fragment order, pre-split hi / lo; the unit's A = M + e is in flight while
// they are staged.  (Not the receiver-side arithmetic of reading C8: a DP
// group has no receiver; every rank runs this same code on the same P_hat and
// Q_sum, so M' is identical on all ranks.)
constexpr int F_TC_ROWS = 128, F_TC_COLS = 128;
template <int R>
__host__ __device__ constexpr size_t smem_F_tc() {
  constexpr int KS = (R + 7) / 8;
  // A1 [8 m-tiles][KS][32] x 2 uint4 (hi, lo); X = A2 (same size, OCC_ORIENT_T) or B2
  // [16 n-tiles][KS][32] uint4 (plain DP); B1 [16 n-tiles][KS][32] uint4
  return (size_t)48 * KS * 32 * 16;
}

template <int R, bool DPL, bool MBF>
__device__ void phase_F_tc(const Params& p, unsigned char* smraw) {
  constexpr int KS = (R + 7) / 8;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  const int wr = warp & 3, wc = warp >> 2;
  // row factors A1 (M'), A2 (e_new) and column factors B1 (M'), B2 (e_new):
  //   plain:         A1 = A2 = P_hat,       B1 = scale Q_sum, B2 = Q_w (DPL)
  //   OCC_ORIENT_T:  A1 = scale V_sum, A2 = V_w (DPL), B1 = B2 = U_hat   (reading C6; the
  //                  row-side warm start goes to Pstate_out, which only this form sets)
  const bool rowloc = p.Pstate_out != nullptr;
  uint4* ph = reinterpret_cast<uint4*>(smraw);   // [mt8][ks][lane]: hi(a0..a3); lo at + 8 KS 32
  uint4* pl = ph + 8 * KS * 32;
  uint4* ph2 = pl + 8 * KS * 32;                 // X region: A2 (OCC_ORIENT_T) ...
  uint4* pl2 = ph2 + 8 * KS * 32;
  uint4* qw = ph2;                               // ... or B2 (plain DP): [nt16][ks][lane]
  uint4* qs = pl2 + 8 * KS * 32;                 // B1 [nt16][ks][lane]: (h(b0), h(b1), l(b0), l(b1))
  const int nrb = (p.n + F_TC_ROWS - 1) / F_TC_ROWS, ncb = (p.m + F_TC_COLS - 1) / F_TC_COLS;
  const int units = nrb * ncb;
  const bool rbf = p.r_bf16 != 0;
  for (int u = blockIdx.x; u < units; u += gridDim.x) {
    const int cb = u % ncb, rb = u / ncb;
    const int R0 = rb * F_TC_ROWS, C0 = cb * F_TC_COLS;
    const int nr = min(F_TC_ROWS, p.n - R0), nc = min(F_TC_COLS, p.m - C0);
    __syncthreads();
    // this lane's A = M + e for one 64-column half (2 m-tiles x rows g, g + 8 x 2 column groups)
    A4 av[2][2][2];
    const int cl = 32 * wc + 4 * t;   // first column of group 0 within a half
    auto load_av = [&](int hf) {
#pragma unroll
      for (int mt = 0; mt < 2; mt++)
#pragma unroll
        for (int h = 0; h < 2; h++)
#pragma unroll
          for (int q = 0; q < 2; q++) {
            const int i = 32 * wr + 16 * mt + g + 8 * h, j = 64 * hf + cl + 16 * q;
            av[mt][h][q] = ldA4<MBF>(p, R0 + i, C0 + j, p.err_out && i < nr && j < nc);
          }
    };
    load_av(0);   // in flight during the staging
    // stage the row factors: X[i][k] -> m-tile i/16, ks = k/8, lane (g = i%8, t = k%4),
    // a-slot (i%16)/8 + 2 ((k%8)/4); A1 = P (scaled with OCC_ORIENT_T, and the row-side warm
    // start scale P -> Pstate_out), A2 = Ploc (OCC_ORIENT_T, DPL)
    {
      unsigned* h32 = reinterpret_cast<unsigned*>(ph);
      unsigned* l32 = reinterpret_cast<unsigned*>(pl);
      unsigned* h232 = reinterpret_cast<unsigned*>(ph2);
      unsigned* l232 = reinterpret_cast<unsigned*>(pl2);
      const bool a2 = rowloc && DPL && p.Ploc;
      for (int x = threadIdx.x; x < F_TC_ROWS * KS * 2; x += occ::NT) {
        const int i = x / (KS * 2), k0 = 4 * (x % (KS * 2));
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f), w = v;
        if (i < nr && k0 < R) {
          v = __ldcg(reinterpret_cast<const float4*>(p.P + (size_t)(R0 + i) * R + k0));
          if (rowloc) {
            v = make_float4(p.scale * v.x, p.scale * v.y, p.scale * v.z, p.scale * v.w);
            if (p.Pstate_out && cb == 0) *reinterpret_cast<float4*>(p.Pstate_out + (size_t)(R0 + i) * R + k0) = v;
          }
          if (a2) w = __ldcg(reinterpret_cast<const float4*>(p.Ploc + (size_t)(R0 + i) * R + k0));
        }
        const float vv[4] = {v.x, v.y, v.z, v.w}, ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const int k = k0 + j;
          const size_t e = ((((size_t)(i >> 4) * KS + (k >> 3)) * 32) + (i & 7) * 4 + (k & 3)) * 4 + ((i & 15) >> 3) +
                           2 * ((k & 7) >> 2);
          unsigned hh, ll;
          split_tf32(vv[j], hh, ll);
          h32[e] = hh;
          l32[e] = ll;
          if (a2) {
            split_tf32(ww[j], hh, ll);
            h232[e] = hh;
            l232[e] = ll;
          }
        }
      }
    }
    // stage the column factors: Q[c][k] -> n-tile (c / 16) * 2 + (c % 4) / 2, n = 2 ((c % 16) / 4) + c % 2,
    // ks = k / 8, lane (g = n, t = k % 4), b-slot (k % 8) / 4
    {
      unsigned* s32 = reinterpret_cast<unsigned*>(qs);
      unsigned* w32 = reinterpret_cast<unsigned*>(qw);
      for (int x = threadIdx.x; x < F_TC_COLS * KS * 2; x += occ::NT) {
        const int c = x / (KS * 2), k0 = 4 * (x % (KS * 2));
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f), w = v;
        if (c < nc && k0 < R) {
          v = __ldcg(reinterpret_cast<const float4*>(p.Qrec + (size_t)(C0 + c) * R + k0));
          if (!rowloc) {
            v = make_float4(p.scale * v.x, p.scale * v.y, p.scale * v.z, p.scale * v.w);
            if (p.Qstate_out && rb == 0) *reinterpret_cast<float4*>(p.Qstate_out + (size_t)(C0 + c) * R + k0) = v;
            if (DPL) w = __ldcg(reinterpret_cast<const float4*>(p.Qloc + (size_t)(C0 + c) * R + k0));
          }
        }
        const float vv[4] = {v.x, v.y, v.z, v.w}, ww[4] = {w.x, w.y, w.z, w.w};
        const int nt = (c >> 4) * 2 + ((c & 3) >> 1), n = 2 * ((c & 15) >> 2) + (c & 1);
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const int k = k0 + j;
          const size_t e = ((((size_t)nt * KS + (k >> 3)) * 32) + n * 4 + (k & 3)) * 4 + ((k & 7) >> 2);
          unsigned hh, ll;
          split_tf32(vv[j], hh, ll);
          s32[e] = hh;
          s32[e + 2] = ll;
          if (DPL && !rowloc) {
            split_tf32(ww[j], hh, ll);
            w32[e] = hh;
            w32[e + 2] = ll;
          }
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int hf = 0; hf < 2; hf++) {
      if (hf == 1) load_av(1);   // (after half 0's stores; in flight during half 1's MMAs)
      float ds[2][4][4], dw[2][4][4];
#pragma unroll
      for (int mt = 0; mt < 2; mt++)
#pragma unroll
        for (int nt = 0; nt < 4; nt++)
#pragma unroll
          for (int q = 0; q < 4; q++) ds[mt][nt][q] = dw[mt][nt][q] = 0.f;
      const int ntb = 8 * hf + 4 * wc;   // this warp's first n-tile
      auto mma_loop = [&](auto ot) {   // ot: the e_new product has its own row factor (A2)
        constexpr bool OT = decltype(ot)::value;
#pragma unroll 2
        for (int ks = 0; ks < KS; ks++) {
          unsigned ah[2][4], al[2][4], ah2[2][4], al2[2][4];
#pragma unroll
          for (int mt = 0; mt < 2; mt++) {
            const size_t o = ((size_t)(2 * wr + mt) * KS + ks) * 32 + lane;
            const uint4 hv = ph[o], lv = pl[o];
            ah[mt][0] = hv.x; ah[mt][1] = hv.y; ah[mt][2] = hv.z; ah[mt][3] = hv.w;
            al[mt][0] = lv.x; al[mt][1] = lv.y; al[mt][2] = lv.z; al[mt][3] = lv.w;
            if (OT && DPL) {
              const uint4 hv2 = ph2[o], lv2 = pl2[o];
              ah2[mt][0] = hv2.x; ah2[mt][1] = hv2.y; ah2[mt][2] = hv2.z; ah2[mt][3] = hv2.w;
              al2[mt][0] = lv2.x; al2[mt][1] = lv2.y; al2[mt][2] = lv2.z; al2[mt][3] = lv2.w;
            }
          }
#pragma unroll
          for (int nt = 0; nt < 4; nt++) {
            const size_t o = ((size_t)(ntb + nt) * KS + ks) * 32 + lane;
            const uint4 b = qs[o];
#pragma unroll
            for (int mt = 0; mt < 2; mt++) mma3x(ds[mt][nt], ah[mt], al[mt], b.x, b.y, b.z, b.w);
            if (DPL) {
              if (OT) {
#pragma unroll
                for (int mt = 0; mt < 2; mt++) mma3x(dw[mt][nt], ah2[mt], al2[mt], b.x, b.y, b.z, b.w);
              } else {
                const uint4 bw = qw[o];
#pragma unroll
                for (int mt = 0; mt < 2; mt++) mma3x(dw[mt][nt], ah[mt], al[mt], bw.x, bw.y, bw.z, bw.w);
              }
            }
          }
        }
      };
      if (rowloc) mma_loop(std::true_type{});
      else mma_loop(std::false_type{});
      // outputs: m-tile mt, rows g (+8 h); group q: columns 64 hf + cl + 16 q .. + 3 =
      // (n-tile 2q: c0, c1 | n-tile 2q+1: c0, c1) for row g, (c2, c3 | c2, c3) for row g + 8
#pragma unroll
      for (int mt = 0; mt < 2; mt++)
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int i = 32 * wr + 16 * mt + g + 8 * h;
          if (i >= nr) continue;
#pragma unroll
          for (int q = 0; q < 2; q++) {
            const int j = 64 * hf + cl + 16 * q;
            if (j >= nc) continue;
            float mr[4] = {ds[mt][2 * q][2 * h], ds[mt][2 * q][2 * h + 1], ds[mt][2 * q + 1][2 * h],
                           ds[mt][2 * q + 1][2 * h + 1]};
            if (rbf) {
#pragma unroll
              for (int z = 0; z < 4; z++) mr[z] = __bfloat162float(__float2bfloat16_rn(mr[z]));
            }
            const size_t row = (size_t)(R0 + i), col = (size_t)(C0 + j);
            if (p.recon) {
              if (rbf) {
                __nv_bfloat162 b01 = __floats2bfloat162_rn(mr[0], mr[1]), b23 = __floats2bfloat162_rn(mr[2], mr[3]);
                uint2 raw;
                raw.x = *reinterpret_cast<unsigned*>(&b01);
                raw.y = *reinterpret_cast<unsigned*>(&b23);
                *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(p.recon) + row * p.ldr + col) = raw;
              } else {
                *reinterpret_cast<float4*>(reinterpret_cast<float*>(p.recon) + row * p.ldr + col) =
                    make_float4(mr[0], mr[1], mr[2], mr[3]);
              }
            }
            if (p.err_out) {
              const float4 a = val<MBF>(av[mt][h][q]);
              float4 e;
              if (DPL) {
                e = make_float4(a.x - dw[mt][2 * q][2 * h], a.y - dw[mt][2 * q][2 * h + 1],
                                a.z - dw[mt][2 * q + 1][2 * h], a.w - dw[mt][2 * q + 1][2 * h + 1]);
              } else {
                e = make_float4(a.x - mr[0], a.y - mr[1], a.z - mr[2], a.w - mr[3]);
              }
              *reinterpret_cast<float4*>(p.err_out + row * p.lde_out + col) = e;
            }
          }
        }
    }
  }
}

}  // namespace tc
}  // namespace occ
