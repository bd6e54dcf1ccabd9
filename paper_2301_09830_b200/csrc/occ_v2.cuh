// occ_v2.cuh -- the fused single-GPU step, TMEM-resident version (sm_100a).
//
// One persistent CTA per SM owns one tile (H rows x W cols, W wide enough
// that one tile row is a >= 2-4 KB contiguous segment) for the whole step:
//
//  phase 1  cp.async.bulk streams the tile's rows of M and e, 8 rows per
//           stage, into a padded staging ring (mbarrier complete_tx).  A = M+e
//           (a1) is formed in registers; P^T_rows = Q_prev^T A^T_rows (a2) runs
//           on the tensor cores (mma.sync m16n8k8 tf32, 3-term hi/lo split =
//           fp32 accuracy), warps splitting the columns; A is stored in TENSOR
//           MEMORY (tcgen05.st) in the per-lane fragment layout phases 3 and 5
//           consume, so M and e are read from HBM exactly once.
//  barrier  (P partials of the row band visible)
//  phase 2  P_band = sum of the nc column-tile partials; the band's Gram
//           partial P_band^T P_band in fp64 (a4).
//  barrier
//  phase 3  G = sum of the nr band partials; warp-level Cholesky in fp64 with
//           the degenerate-column fallback (reading C3; slow paths add
//           barriers); P_hat_band = P_band L^-T (a4); Q_part = A^T P_hat (a5)
//           from TMEM on the tensor cores, complete per column group.
//  barrier
//  phase 4  Q = sum of the nr row-band partials, distributed over the CTAs of
//           the column band, written to the output Q (a5, a9).
//  barrier
//  phase 5  M'^T = Q P_hat^T on the tensor cores (a7) in the same fragments
//           as A in TMEM, e_new = A - round(M') (a8); stores M' and e_new.
//
// Fragment bookkeeping.  A tile is cut into cells of 8 rows x 16 cols; compute
// warp w owns the column groups cg = w (mod NCW) and every cell in them.  In
// a cell at (r0, c0) lane (g = lane/4, t = lane%4) owns the four elements
//   A[r0+t][c0+2g], A[r0+t+4][c0+2g], A[r0+t][c0+2g+1], A[r0+t+4][c0+2g+1]
// which are (i) the B-operand registers of the two m16n8k8 MMAs computing
// Q^T += P_hat^T A over that cell (even / odd columns), and (ii) the
// accumulator registers of the m16n8k8 MMA computing M'^T = Q P_hat^T over
// it (column index n <-> 2n / 2(n-8)+1, row index n <-> n/2 + 4(n&1); see
// occ_v2_kernel.cuh).  The four values live in four TMEM columns of the
// warp's lanes (slot = (cg / NCW) * nrblk + rblk).
#pragma once
#include "occ_kernels.cuh"

#include <type_traits>

namespace occ {
namespace v2 {

constexpr int NT = 512;
constexpr int NW = 16;
constexpr int NCW = NW - 1;     // compute warps; warp NW-1 is the phase-1 copy producer
constexpr int SR = 8;           // tile rows per staging stage (one cell row block)
constexpr int MAX_STAGES = 6;
constexpr int TMEM_CELLS = 512 / (NW / 4) / 4;  // cells per warp in TMEM (its columns / 4)
constexpr int kTrStamps = 24;   // per-CTA phase-trace stamps (occ_read_trace)

struct Params2 {
  const void* M; long long ldm;
  const float* err_in; long long lde_in;
  float* err_out; long long lde_out;
  void* recon; long long ldr;
  int n, m;
  const float* Qprev;  // m x R
  float* Pout;         // n x R (P_hat)
  float* Qout;         // m x R (Q)
  int nr, nc, H, W;    // tile grid / tile shape
  int ns, sw;          // staging stages, staging row stride (floats)
  // shared-memory carve (bytes)
  int off_stm, off_ste, off_qs, off_red, off_pa, off_pb, off_orth, off_ps, off_gs, off_qsm, smem_total;
  // workspace
  float* P_part;       // [nc][n][R]
  double* G_band;      // [nr][NP]
  double* G2_band;     // [nr][NP]
  double* XY_band;     // [nr][2 R R]
  float* Q_part;       // [nr][m][R]
  unsigned* bar;        // [0] unused here, [1] exit counter
  unsigned* barl;       // grid_barrier_spread arrival lines (kBarLines x 32 words)
  unsigned long long* trace;   // [grid][2 kTrStamps]: clock64 stamps, then globaltimer stamps
  DevStats* stats;
  unsigned long long fb_seed;
  double tau, kappa_thr;
  double amp_thr;      // fused-Q gate on ||S Li^T||_F (phase 3)
  int check_finite;    // OCC_CHECK_FINITE (phase 3)
  int wire_bf16;       // OCC_WIRE_BF16: P_hat rows and the Q slice rounded to bf16 before phase 5
  int force_two_pass;
  int debug;           // bit 0: skip phase-1 compute (streaming floor measurement only)
  LinkPush push;       // occ_link sender: warp NW-1 pushes this CTA's P_hat rows / Q slice during phase 5
};

// ------------------------------------------------------------------ grid barrier
// Arrivals are spread over kBarLines counters on separate 128-B lines (CTA b
// adds to line b % kBarLines), so 148 red.release ops do not serialise on one
// L2 line; lanes 0..kBarLines-1 of warp 0 poll one line each.  Barrier number
// `epoch` (1, 2, ...) of the launch completes when line j holds epoch x (the
// CTAs mapped to it).  sync() is the CTA-level barrier of the participating
// threads (warp 0 must participate): the phase-3 compute-warp barrier lets warp
// NW-1 keep working through it.  Ordering: bar.sync + gpu-scope release /
// acquire, as in the single-counter barrier (occ_kernels.cuh grid_barrier).
constexpr int kBarLines = 8;
struct SyncBlock {
  __device__ __forceinline__ void operator()() const { __syncthreads(); }
};
template <class Sync = SyncBlock>
__device__ __forceinline__ void grid_barrier_spread(unsigned* lines, unsigned epoch, Sync sync = Sync()) {
  sync();
  if (threadIdx.x < 32) {
    const unsigned lane = threadIdx.x;
    if (lane == 0)
      asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(lines + (blockIdx.x % kBarLines) * 32), "r"(1u)
                   : "memory");
    if (lane < kBarLines) {
      const unsigned cnt = gridDim.x > lane ? (gridDim.x - lane + kBarLines - 1) / kBarLines : 0u;
      const unsigned target = epoch * cnt;
      const unsigned* ln = lines + lane * 32;
      unsigned v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ln) : "memory");
      } while (v < target);
    }
    __syncwarp();
  }
  sync();
}

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// L2 policy for data streamed once (M, e in; M', e_new out): evict first, so
// the step's streaming does not push the kernel's code and the small partial
// sums out of L2 (the code of the middle phases is fetched once per step).
__device__ __forceinline__ unsigned long long l2_evict_first() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ unsigned long long l2_evict_normal() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                              unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void st_f2_hint(float* p, float2 v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(p), "f"(v.x), "f"(v.y), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_b32_hint(void* p, unsigned v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ unsigned tf32_rna(float x) {
  unsigned r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
// x = hi + lo with hi an exact tf32 value (the low 13 mantissa bits masked off)
// and lo = x - hi exact in fp32; the tensor core reads lo's top 19 bits, so
// the split is accurate to ~2^-21 |x|.  Two ALU ops: cvt.rna.tf32.f32 is
// emulated with ~3 integer ops per conversion on sm_100a.
__device__ __forceinline__ void split3(float x, unsigned& hi, unsigned& lo) {
  hi = __float_as_uint(x) & 0xffffe000u;
  lo = __float_as_uint(x - __uint_as_float(hi));
}
// a + b on a float pair in one FADD2 (sm_100 packed fp32)
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  unsigned long long x, y, d;
  memcpy(&x, &a, 8);
  memcpy(&y, &b, 8);
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(x), "l"(y));
  float2 r;
  memcpy(&r, &d, 8);
  return r;
}
// a - b on a float pair in one FADD2
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
  unsigned long long x, y, d;
  memcpy(&x, &a, 8);
  memcpy(&y, &b, 8);
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(x), "l"(y));
  float2 r;
  memcpy(&r, &d, 8);
  return r;
}
__device__ __forceinline__ void mma_tf32(float (&d)[4], const unsigned (&a)[4], unsigned b0, unsigned b1) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// d += A . B with fp32-level accuracy: A = ah + al, B = bh + bl, drop al.bl
__device__ __forceinline__ void mma3(float (&d)[4], const unsigned (&ah)[4], const unsigned (&al)[4], unsigned bh0,
                                     unsigned bh1, unsigned bl0, unsigned bl1) {
  mma_tf32(d, al, bh0, bh1);
  mma_tf32(d, ah, bl0, bl1);
  mma_tf32(d, ah, bh0, bh1);
}

__device__ __forceinline__ void tmem_st4(unsigned taddr, float a, float b, float c, float d) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(__float_as_uint(a)),
               "r"(__float_as_uint(b)), "r"(__float_as_uint(c)), "r"(__float_as_uint(d))
               : "memory");
}
__device__ __forceinline__ void tmem_ld4(unsigned taddr, float (&v)[4]) {
  unsigned a, b, c, d;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
               : "r"(taddr)
               : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  v[0] = __uint_as_float(a); v[1] = __uint_as_float(b); v[2] = __uint_as_float(c); v[3] = __uint_as_float(d);
}

// four consecutive cells (16 TMEM columns) in one load
__device__ __forceinline__ void tmem_ld16(unsigned taddr, float (&v)[16]) {
  unsigned r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int q = 0; q < 16; q++) v[q] = __uint_as_float(r[q]);
}

// ------------------------------------------------------------------ geometry helpers
struct Tile {
  int rb, cb, row0, col0, th, tw, nrblk, ncg, ncells;
};
__device__ __forceinline__ Tile tile_of(const Params2& p) {
  Tile t;
  t.rb = blockIdx.x / p.nc;
  t.cb = blockIdx.x % p.nc;
  t.row0 = t.rb * p.H;
  t.col0 = t.cb * p.W;
  t.th = max(0, min(p.H, p.n - t.row0));
  t.tw = max(0, min(p.W, p.m - t.col0));
  t.nrblk = (t.th + 7) / 8;
  t.ncg = (t.tw + 15) / 16;
  t.ncells = t.nrblk * t.ncg;
  return t;
}

// A element (i, j) of the tile from global memory (non-resident cells).
template <bool MBF>
__device__ __forceinline__ float gA(const Params2& p, int gi, int gj) {
  float v;
  if (MBF) v = __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p.M)[(size_t)gi * p.ldm + gj]);
  else v = __ldcg(reinterpret_cast<const float*>(p.M) + (size_t)gi * p.ldm + gj);
  if (p.err_in) v += __ldcg(p.err_in + (size_t)gi * p.lde_in + gj);
  return v;
}

// Cold paths, kept out of line so the hot unrolled loops of phases 3a/5 stay
// compact in the instruction stream (all 148 SMs fetch the same code at once).
// Values travel as float4 (registers), never through local memory.
//
// The 4 values of lane (g,t) for cell (rblk, cg) (order (r,c), (r+4,c),
// (r,c+1), (r+4,c+1), r = 8 rblk + t, c = 16 cg + 2g): from TMEM slot cs when
// it is resident, else recomputed from M and e in global memory.
template <bool MBF>
__device__ __noinline__ float4 cell_slow(const Params2& p, const Tile T, unsigned taddr, int cs, int rblk, int cg,
                                         int g, int t) {
  if (cs < TMEM_CELLS) {
    float v[4];
    tmem_ld4(taddr + (unsigned)(cs * 4), v);
    return make_float4(v[0], v[1], v[2], v[3]);
  }
  const int r = 8 * rblk + t, c = 16 * cg + 2 * g;
  const int gi = T.row0 + r, gj = T.col0 + c;
  float4 v;
  v.x = (r < T.th && c < T.tw) ? gA<MBF>(p, gi, gj) : 0.f;
  v.y = (r + 4 < T.th && c < T.tw) ? gA<MBF>(p, gi + 4, gj) : 0.f;
  v.z = (r < T.th && c + 1 < T.tw) ? gA<MBF>(p, gi, gj + 1) : 0.f;
  v.w = (r + 4 < T.th && c + 1 < T.tw) ? gA<MBF>(p, gi + 4, gj + 1) : 0.f;
  return v;
}

// phase-5 stores of a cell on the tile edge, element-wise and bounds-checked
template <bool MBF>
__device__ __noinline__ void store_cell_edge(const Params2& p, const Tile T, int r, int c, float4 mr4, float4 v4) {
  const float mr[4] = {mr4.x, mr4.y, mr4.z, mr4.w}, v[4] = {v4.x, v4.y, v4.z, v4.w};
  const int rows[4] = {r, r + 4, r, r + 4}, cols[4] = {c, c, c + 1, c + 1};
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

}  // namespace v2
}  // namespace occ
