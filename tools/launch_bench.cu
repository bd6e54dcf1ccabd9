// Launch + drain cost of an empty persistent kernel shaped like the fused step
// (148 CTAs x 512 threads, ~200 KB dynamic SMEM): cooperative vs normal
// launch, with and without TMEM alloc/dealloc.  Not part of the product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/launch_bench.cu -o tools/bin/launch_bench
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(512, 1) k_empty(int* out, int tmem) {
  extern __shared__ unsigned char sm[];
  __shared__ unsigned tb;
  if (tmem && threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((unsigned)__cvta_generic_to_shared(&tb)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  if (threadIdx.x == 0) sm[0] = 1;
  __syncthreads();
  if (tmem && threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
  if (threadIdx.x == 0 && sm[0] == 2) out[blockIdx.x] = 1;
}
int main() {
  int* d; cudaMalloc(&d, 4096);
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int coop = 0; coop < 2; coop++)
    for (int tmem = 0; tmem < 2; tmem++) {
      float best = 1e9, sum = 0; const int N = 200;
      for (int i = 0; i < N + 10; i++) {
        cudaEventRecord(a);
        if (coop) { void* args[] = {&d, &tmem}; cudaLaunchCooperativeKernel((void*)k_empty, 148, 512, args, smem, 0); }
        else k_empty<<<148, 512, smem>>>(d, tmem);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (i >= 10) { sum += ms; if (ms < best) best = ms; }
      }
      printf("%s launch, tmem %d: mean %.2f us, best %.2f us (event to event, synchronous)\n", coop ? "cooperative" : "normal     ", tmem, sum / N * 1e3, best * 1e3);
    }
  // back-to-back throughput
  for (int coop = 0; coop < 2; coop++) {
    int tmem = 1; const int N = 200;
    cudaEventRecord(a);
    for (int i = 0; i < N; i++) {
      if (coop) { void* args[] = {&d, &tmem}; cudaLaunchCooperativeKernel((void*)k_empty, 148, 512, args, smem, 0); }
      else k_empty<<<148, 512, smem>>>(d, tmem);
    }
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%s back-to-back: %.2f us per launch\n", coop ? "cooperative" : "normal     ", ms / N * 1e3);
  }
  return 0;
}
