// Can device code read (and L2-prefetch) its own instruction bytes through a
// function pointer?  Prints the pointer and the first 16 bytes read from it, to
// compare against cuobjdump's encoding of the same function.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -rdc=false tools/codeptr_test.cu -o tools/codeptr_test
#include <cstdio>
#include <cuda_runtime.h>

__device__ __noinline__ int foo(int x) { return x * 3 + 1; }

__global__ void probe(unsigned long long* out, int mode) {
  int (*fp)(int) = foo;
  const unsigned long long a = (unsigned long long)fp;
  out[0] = a;
  out[1] = __isGlobal((const void*)a);
  if (mode >= 1) asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
  if (mode >= 2) {
    unsigned long long v0, v1;
    asm volatile("ld.global.nc.v2.u64 {%0,%1}, [%2];" : "=l"(v0), "=l"(v1) : "l"(a));
    out[2] = v0;
    out[3] = v1;
  }
  out[4] = foo((int)out[5]);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  cudaMemset(d, 0, 64);
  for (int mode = 0; mode < 3; mode++) {
    probe<<<1, 1>>>(d, mode);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[6] = {};
    cudaMemcpy(h, d, 48, cudaMemcpyDeviceToHost);
    printf("mode %d: err=%s fp=0x%llx isGlobal=%llu bytes=%016llx %016llx\n", mode, cudaGetErrorString(e), h[0], h[1], h[2],
           h[3]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
