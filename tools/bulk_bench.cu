// cp.async.bulk streaming bandwidth vs copy size (148 CTAs, mbarrier ring). Not part of the product.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void __launch_bounds__(256, 1) k(const char* src, size_t per_cta, int chunk, int stages, int per_stage, float* out) {
  extern __shared__ __align__(128) char sm[];
  __shared__ uint64_t bar[8];
  if (threadIdx.x == 0) { for (int s = 0; s < 8; s++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su(&bar[s]))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  const char* base = src + blockIdx.x * per_cta;
  const size_t stage_bytes = (size_t)chunk * per_stage;
  const int nst = (int)(per_cta / stage_bytes);
  auto issue = [&](int s) {
    int slot = s % stages;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su(&bar[slot])), "r"((unsigned)stage_bytes) : "memory");
    for (int c = 0; c < per_stage; c++)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        :: "r"(su(sm + slot * stage_bytes + c * chunk)), "l"(base + (size_t)s * stage_bytes + (size_t)c * chunk), "r"(chunk), "r"(su(&bar[slot])) : "memory");
  };
  if (threadIdx.x == 0) for (int s = 0; s < stages && s < nst; s++) issue(s);
  float acc = 0;
  for (int s = 0; s < nst; s++) {
    int slot = s % stages;
    unsigned par = (s / stages) & 1;
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" :: "r"(su(&bar[slot])), "r"(par) : "memory");
    acc += ((float*)(sm + slot * stage_bytes))[threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0 && s + stages < nst) issue(s + stages);
  }
  out[blockIdx.x * 256 + threadIdx.x] = acc;
}
int main() {
  size_t total = 148ull * 2 * 1024 * 1024;  // 2 MiB per CTA
  char* src; float* out;
  cudaMalloc(&src, total); cudaMalloc(&out, 148 * 256 * 4);
  cudaMemset(src, 0, total);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int chunks[] = {512, 1024, 2048, 4096, 16384};
  for (int chunk : chunks) for (int stages : {2, 4}) {
    int per_stage = 32768 / chunk; if (per_stage < 1) per_stage = 1;
    size_t smem = (size_t)stages * chunk * per_stage;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<148, 256, smem>>>(src, total / 148, chunk, stages, per_stage, out);
    cudaEventRecord(a);
    for (int it = 0; it < 5; it++) k<<<148, 256, smem>>>(src, total / 148, chunk, stages, per_stage, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("chunk %6d B x %2d per stage, %d stages (%zu KB in flight): %.0f GB/s (%s)\n", chunk, per_stage, stages, smem / 1024, 5.0 * total / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
}
