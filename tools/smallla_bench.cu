// Cycle counts of the fused kernel's small fp64 linear algebra in isolation (not part of the product).
#include "../paper_2301_09830_b200/csrc/occ_v2.cu"
#include <cstdio>
#include <vector>
#include <cstdlib>
using namespace occ;
using namespace occ::v2;
template <int R>
__global__ void __launch_bounds__(512, 1) k_small(const double* part, int nparts, float* ps_in, int nr, unsigned long long* cyc) {
  extern __shared__ __align__(128) unsigned char sm[];
  OrthW& o = *reinterpret_cast<OrthW*>(sm);
  double* scr = reinterpret_cast<double*>(sm + sizeof(OrthW) + 128);
  float* ps = reinterpret_cast<float*>(sm + sizeof(OrthW) + 128 + 1024 * 8);
  float* ps2 = ps + 256 * 16;
  for (int x = threadIdx.x; x < nr * 16; x += blockDim.x) ps[x] = ps_in[x];
  __syncthreads();
  unsigned long long t0 = clock64();
  reduce_partials<R>(part, nparts, o, scr);
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x < 32) { int d = ldl_warp<R>(o, 1e-10, true); if (threadIdx.x == 0) o.deg = d; }
  __syncthreads();
  unsigned long long t2 = clock64();
  if (threadIdx.x < 32) inverse_warp<R>(o);
  __syncthreads();
  unsigned long long t3 = clock64();
  band_apply<R>(ps, ps2, nr, o, false, 0, 0);
  __syncthreads();
  unsigned long long t4 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = o.deg; }
}
int main() {
  const int R = 16, NP = R * (R + 1) / 2, nparts = 37, nr = 112;
  // a well-conditioned Gram: sum of partials of random P rows
  std::vector<double> part(nparts * NP);
  std::vector<float> P(nr * 16);
  srand(1);
  for (auto& v : P) v = (rand() / (float)RAND_MAX) - 0.5f;
  for (int u = 0; u < nparts; u++) {
    int q = 0;
    for (int a = 0; a < R; a++) for (int b = a; b < R; b++) {
      double g = 0; for (int i = 0; i < nr; i++) g += (double)P[i * 16 + a] * P[i * 16 + b];
      part[u * NP + q++] = g + (a == b ? 1.0 : 0.0);
    }
  }
  double* dpart; float* dps; unsigned long long* dc;
  cudaMalloc(&dpart, part.size() * 8); cudaMalloc(&dps, P.size() * 4); cudaMalloc(&dc, 64);
  cudaMemcpy(dpart, part.data(), part.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dps, P.data(), P.size() * 4, cudaMemcpyHostToDevice);
  size_t smem = sizeof(OrthW) + 128 + 1024 * 8 + 2 * 256 * 16 * 4;
  cudaFuncSetAttribute(k_small<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int it = 0; it < 3; it++) {
    k_small<16><<<148, 512, smem>>>(dpart, nparts, dps, nr, dc);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long c[5]; cudaMemcpy(c, dc, 40, cudaMemcpyDeviceToHost);
    printf("(%s) cycles: reduce_partials %llu  ldl_warp %llu  inverse_warp %llu  band_apply %llu  deg=%llu\n", cudaGetErrorString(e), c[0], c[1], c[2], c[3], c[4]);
  }
}
