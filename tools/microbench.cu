// Microbenchmarks that size the design (not part of the product):
//  1. grid barrier latency (148 CTAs x 512 threads, release/acquire counter)
//  2. mma.sync.m16n8k8 tf32 throughput per SM
//  3. FFMA throughput (3-register form) per SM
//  4. tcgen05.st / tcgen05.ld round trip bandwidth per SM (TMEM as scratch)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb tools/microbench.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ unsigned g_ctr;

__device__ __forceinline__ void gbar(unsigned* ctr, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    unsigned v;
    while (true) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
      if (v >= target) break;
    }
  }
  __syncthreads();
}

__global__ void k_barrier(int iters, unsigned long long* out) {
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; i++) gbar(&g_ctr, (i + 1) * gridDim.x);
  unsigned long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
}

__global__ void k_mma(int iters, float* out) {
  unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  float c[4][4] = {};
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 4; j++)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
  for (int j = 0; j < 4; j++) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma(int iters, float* out) {
  float a[16], x = threadIdx.x * 1e-3f, y = 1.0001f;
  for (int j = 0; j < 16; j++) a[j] = j;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 16; j++) a[j] = fmaf(a[j], y, x);
    y += 1e-9f;   // keep y a register operand
  }
  float s = 0;
  for (int j = 0; j < 16; j++) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  unsigned long long* d;
  float* f;
  cudaMalloc(&d, 8);
  cudaMalloc(&f, 148 * 1024 * 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // 1. barrier
  for (int threads : {256, 512}) {
    unsigned z = 0;
    cudaMemcpyToSymbol(g_ctr, &z, 4);
    int iters = 1000;
    void* args[] = {&iters, &d};
    cudaEventRecord(e0);
    cudaLaunchCooperativeKernel((void*)k_barrier, sms, threads, args, 0, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("grid barrier: %d CTAs x %d thr: %.3f us per barrier (%s)\n", sms, threads, ms * 1e3 / iters,
           cudaGetErrorString(cudaGetLastError()));
  }
  // 2. mma.sync tf32
  {
    int iters = 20000;
    k_mma<<<sms, 512>>>(100, f);
    cudaEventRecord(e0);
    k_mma<<<sms, 512>>>(iters, f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double mmas = (double)sms * 16 * iters * 4;   // warp-level mma instructions
    double flops = mmas * 16 * 8 * 8 * 2;
    printf("mma.sync m16n8k8 tf32: %.1f TFLOP/s, %.3f warp-mma/clk/SM at 1.965GHz (%s)\n", flops / ms / 1e9,
           mmas / sms / (ms * 1e-3 * 1.965e9), cudaGetErrorString(cudaGetLastError()));
  }
  // 3. FFMA
  {
    int iters = 20000;
    k_ffma<<<sms, 512>>>(100, f);
    cudaEventRecord(e0);
    k_ffma<<<sms, 512>>>(iters, f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double fma = (double)sms * 512 * iters * 16;
    printf("FFMA: %.1f TFMA/s, %.1f FMA/clk/SM at 1.965GHz\n", fma / ms / 1e9, fma / sms / (ms * 1e-3 * 1.965e9));
  }
  return 0;
}
