// TMEM load latency: tcgen05.ld.32x32b.x16 + tcgen05.wait::ld, dependent
// chain (the next address depends on the loaded value), with 1 or 16 warps
// per CTA loading concurrently.  Not part of the product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/tmem_lat.cu -o tools/bin/tmem_lat
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512, 1) k_lat(int iters, int active_warps, unsigned long long* cyc, float* out) {
  __shared__ unsigned tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((unsigned)__cvta_generic_to_shared(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const unsigned taddr = tbase + ((unsigned)((warp & 3) * 32) << 16) + (unsigned)((warp >> 2) * 128);
  // fill with zeros so the dependent address offset stays 0
  unsigned z = 0;
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%1,%1,%1};" ::"r"(taddr), "r"(z));
  asm volatile("tcgen05.wait::st.sync.aligned;");
  __syncthreads();
  float acc = 0.f;
  unsigned off = 0;
  unsigned long long t0 = clock64();
  if (warp < active_warps) {
    for (int it = 0; it < iters; it++) {
      unsigned r[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
            "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
          : "r"(taddr + off));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      off = r[0] & 0;   // dependency on the loaded value (stays 0)
      acc += __uint_as_float(r[15]);
    }
  }
  unsigned long long t1 = clock64();
  if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * 16 + warp] = t1 - t0;
  out[blockIdx.x * 512 + threadIdx.x] = acc + off;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

int main() {
  unsigned long long* cyc;
  float* out;
  cudaMalloc(&cyc, 148 * 16 * 8);
  cudaMalloc(&out, 148 * 512 * 4);
  const int iters = 256;
  for (int aw : {1, 4, 16}) {
    for (int rep = 0; rep < 2; rep++) {
      k_lat<<<148, 512>>>(iters, aw, cyc, out);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    }
    unsigned long long h[148 * 16];
    cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
    double s = 0;
    for (int b = 0; b < 148; b++) s += h[b * 16];
    printf("active warps %2d: %.1f cycles per dependent tcgen05.ld x16 + wait\n", aw, s / 148 / iters);
  }
  return 0;
}
