// Single-warp micro-benchmark of the phase-3 small linear algebra of the fused
// kernel (occ_v2_la.cuh): ldl_warp + inverse_warp on an R x R SPD Gram, timed
// with clock64 per call.  Call 0 of every launch follows an L2 flush (the code
// is then fetched from HBM, as in the real step); calls 1.. are warm.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude \
//        -Ipaper_2301_09830_b200/csrc tools/la_bench.cu -o tools/la_bench
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "occ_v2_la.cuh"

using namespace occ::v2;
namespace occ { namespace v2 {
// Warp-level right-looking LDL^T of the Gram in o.L (R <= 32), square-root free
// so the sequential chain per column is one fp64 reciprocal.  Lane i holds row
// i in registers; column j is broadcast through o.col.  detect: stop at the
// first column whose squared residual D_j is below tau2 * its own squared norm
// (reading C3: the MGS test ||v|| < tau ||p_j||) and return 1.  Warp 0 only.
template <int R>
__device__ int ldl_warp_v0(OrthW& o, double tau2, bool detect) {
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
__device__ void inverse_warp_v0(OrthW& o) {
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


}}
constexpr int R = 16;
constexpr int REPS = 4;

template <int V>
__global__ void la_kernel(const double* G, long long* cyc, double* out) {
  extern __shared__ __align__(16) unsigned char smem[];
  OrthW& o = *reinterpret_cast<OrthW*>(smem);
  const int lane = threadIdx.x;
  for (int rep = 0; rep < REPS; rep++) {
    for (int x = lane; x < R * R; x += 32) {
      o.L[(x / R) * LD + x % R] = G[x];
      if (x / R == x % R) o.gdiag[x / R] = G[x];
    }
    __syncwarp();
    const long long t0 = clock64();
    if (V >= 2) o.prog = 0;
    __syncwarp();
    const int d = V == 3 ? ldl_warp_unrolled<R>(o, 1e-10, true) : V == 2 ? ldl_warp<R>(o, 1e-10, true, true) : V ? ldl_warp<R>(o, 1e-10, true) : ldl_warp_v0<R>(o, 1e-10, true);
    const long long t1 = clock64();
    if (V) inverse_warp<R>(o); else inverse_warp_v0<R>(o);
    long long t3 = clock64();
    if (V == 3 && !d) {   // the pipelined substitution of 32 rows after the factorisation (warm, no waiting)
      __shared__ float rows[32 * 16], outr[32 * 16];
      for (int x = lane; x < 32 * 16; x += 32) rows[x] = (float)((x * 37) % 101) * 0.01f;
      __syncwarp();
      const long long t4 = clock64();
      solve_rows_pipelined<R>(rows, 16, 32, 32, outr, 16, o, lane, 32);
      t3 = clock64() - t4;
      if (lane == 0) out[rep] += outr[5] * 0.f;
    }
    const long long t2 = clock64();
    if (lane == 0 && V == 3) printf("solve 32 rows: %lld cycles\n", t3);
    if (lane == 0) {
      cyc[rep * 2] = t1 - t0;
      cyc[rep * 2 + 1] = t2 - t1;
      out[rep] = d ? -1.0 : o.kappa;
    }
    __syncwarp();
  }
}

__global__ void flush_kernel(float* buf, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) buf[i] += 1.f;
}

int main() {
  // P: 4096 x R with column scales 1/(j+1) and a common component (grad-like)
  const int n = 4096;
  std::vector<double> P((size_t)n * R), G(R * R, 0.0);
  srand(7);
  for (int i = 0; i < n; i++) {
    const double c = (rand() / (double)RAND_MAX - 0.5);
    for (int j = 0; j < R; j++) P[(size_t)i * R + j] = (c + (rand() / (double)RAND_MAX - 0.5)) / (j + 1);
  }
  for (int a = 0; a < R; a++)
    for (int b = 0; b < R; b++) {
      double s = 0;
      for (int i = 0; i < n; i++) s += P[(size_t)i * R + a] * P[(size_t)i * R + b];
      G[a * R + b] = s;
    }
  double *dG, *dout;
  long long* dcyc;
  float* fbuf;
  const size_t fn = (size_t)256 << 20;   // 1 GiB of floats
  cudaMalloc(&dG, R * R * 8);
  cudaMalloc(&dout, REPS * 8);
  cudaMalloc(&dcyc, REPS * 2 * 8);
  cudaMalloc(&fbuf, fn * 4);
  cudaMemcpy(dG, G.data(), R * R * 8, cudaMemcpyHostToDevice);
  const int smem = (int)sizeof(OrthW);
  cudaFuncSetAttribute(la_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(la_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(la_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(la_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int launch = 0; launch < 4; launch++) {
    flush_kernel<<<148 * 4, 512>>>(fbuf, fn);
    if (launch == 3) la_kernel<3><<<1, 32, smem>>>(dG, dcyc, dout);
    else if (launch == 2) la_kernel<2><<<1, 32, smem>>>(dG, dcyc, dout);
    else if (launch == 1) la_kernel<1><<<1, 32, smem>>>(dG, dcyc, dout);
    else la_kernel<0><<<1, 32, smem>>>(dG, dcyc, dout);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    long long cyc[REPS * 2];
    double out[REPS];
    cudaMemcpy(cyc, dcyc, sizeof cyc, cudaMemcpyDeviceToHost);
    cudaMemcpy(out, dout, sizeof out, cudaMemcpyDeviceToHost);
    printf("variant %d kappa %.3g:", launch, out[0]);
    for (int r = 0; r < REPS; r++) printf("  [%d] ldl %lld inv %lld", r, cyc[2 * r], cyc[2 * r + 1]);
    printf("\n");
  }
  return 0;
}
