// TMEM as on-chip scratch: tcgen05.st / tcgen05.ld bandwidth per SM (not part of the product).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(512, 1) k_tmem(int iters, float* out, unsigned long long* cyc) {
  __shared__ unsigned tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"((unsigned)__cvta_generic_to_shared(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const unsigned base = tbase;
  // lane quadrant (warp % 4) in bits 31:16, columns: warp/4 * 128
  const unsigned taddr = base + ((unsigned)((warp & 3) * 32) << 16) + (unsigned)((warp >> 2) * 128);
  float acc = 0.f;
  unsigned v[32];
  for (int j = 0; j < 32; j++) v[j] = __float_as_uint((float)(threadIdx.x + j));
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
    for (int c = 0; c < 128; c += 32) {
      asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
        :: "r"(taddr + c), "r"(v[0]),"r"(v[1]),"r"(v[2]),"r"(v[3]),"r"(v[4]),"r"(v[5]),"r"(v[6]),"r"(v[7]),"r"(v[8]),"r"(v[9]),"r"(v[10]),"r"(v[11]),"r"(v[12]),"r"(v[13]),"r"(v[14]),"r"(v[15]),
           "r"(v[16]),"r"(v[17]),"r"(v[18]),"r"(v[19]),"r"(v[20]),"r"(v[21]),"r"(v[22]),"r"(v[23]),"r"(v[24]),"r"(v[25]),"r"(v[26]),"r"(v[27]),"r"(v[28]),"r"(v[29]),"r"(v[30]),"r"(v[31]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  unsigned long long t1 = clock64();
  for (int it = 0; it < iters; it++) {
    for (int c = 0; c < 128; c += 32) {
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]),"=r"(v[1]),"=r"(v[2]),"=r"(v[3]),"=r"(v[4]),"=r"(v[5]),"=r"(v[6]),"=r"(v[7]),"=r"(v[8]),"=r"(v[9]),"=r"(v[10]),"=r"(v[11]),"=r"(v[12]),"=r"(v[13]),"=r"(v[14]),"=r"(v[15]),
          "=r"(v[16]),"=r"(v[17]),"=r"(v[18]),"=r"(v[19]),"=r"(v[20]),"=r"(v[21]),"=r"(v[22]),"=r"(v[23]),"=r"(v[24]),"=r"(v[25]),"=r"(v[26]),"=r"(v[27]),"=r"(v[28]),"=r"(v[29]),"=r"(v[30]),"=r"(v[31])
        : "r"(taddr + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      for (int j = 0; j < 32; j++) acc += __uint_as_float(v[j]);
    }
  }
  unsigned long long t2 = clock64();
  out[blockIdx.x * 512 + threadIdx.x] = acc;
  if (threadIdx.x == 0) { cyc[blockIdx.x * 2] = t1 - t0; cyc[blockIdx.x * 2 + 1] = t2 - t1; }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(base));
}
int main() {
  float* o; unsigned long long* c;
  cudaMalloc(&o, 148 * 512 * 4); cudaMalloc(&c, 148 * 16);
  int iters = 200;
  k_tmem<<<148, 512>>>(iters, o, c);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[2];
  cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
  double bytes = (double)iters * 512 * 128 * 4;   // per CTA per direction
  printf("tmem (%s): st %.1f B/clk/SM, ld(+wait+add) %.1f B/clk/SM\n", cudaGetErrorString(e), bytes / h[0], bytes / h[1]);
  return 0;
}
