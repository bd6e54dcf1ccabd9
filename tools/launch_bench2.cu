// What drives the launch+drain cost of an empty persistent kernel: dynamic
// SMEM size and block size, back to back.  Not part of the product.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(512, 1) k_empty(int* out) {
  extern __shared__ unsigned char sm[];
  if (threadIdx.x == 0) sm[0] = 1;
  __syncthreads();
  if (threadIdx.x == 0 && sm[0] == 2) out[blockIdx.x] = 1;
}
__global__ void k_other(int* out) { if (threadIdx.x == 9999) out[0] = 1; }
int main() {
  int* d; cudaMalloc(&d, 4096);
  if (cudaFuncSetAttribute(k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024) != cudaSuccess) { printf("attr failed\n"); return 1; }
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int interleave = 0; interleave < 2; interleave++)
  for (int threads : {128, 512})
    for (int kb : {1, 48, 100, 200, 225}) {
      const int N = 200;
      for (int w = 0; w < 2; w++) {
        cudaEventRecord(a);
        for (int i = 0; i < N; i++) {
          if (interleave) k_other<<<148, 256>>>(d);
          k_empty<<<148, threads, kb * 1024>>>(d);
        }
        cudaEventRecord(b); cudaEventSynchronize(b);
        { cudaError_t le = cudaGetLastError(); if (le != cudaSuccess) { printf("launch failed: %s (threads %d smem %d)\n", cudaGetErrorString(le), threads, kb); return 1; } }
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (w) printf("%s threads %3d smem %3d KB: %.2f us per launch\n", interleave ? "with small kernel between" : "back-to-back             ", threads, kb, ms / N * 1e3);
      }
    }
  return 0;
}
