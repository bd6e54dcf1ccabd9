// fp64 FMA latency / throughput and sqrt/rcp cost on this part (not part of the product).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, int iters, long long* cyc) {
  double a = threadIdx.x * 1e-3, b = 1.0000001, c = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) { a = fma(a, b, c); a = fma(a, b, c); a = fma(a, b, c); a = fma(a, b, c); }
  long long t1 = clock64();
  double s = 1.0 + threadIdx.x;
  for (int i = 0; i < iters; i++) { s = sqrt(s) + 1.0; }
  long long t2 = clock64();
  double r = 3.0 + threadIdx.x;
  for (int i = 0; i < iters; i++) { r = 1.0 / r + 1.0; }
  long long t3 = clock64();
  float f = 1.0f + threadIdx.x;
  for (int i = 0; i < iters; i++) { f = fmaf(f, 1.0001f, 1e-9f); f = fmaf(f, 1.0001f, 1e-9f); f = fmaf(f, 1.0001f, 1e-9f); f = fmaf(f, 1.0001f, 1e-9f); }
  long long t4 = clock64();
  out[threadIdx.x] = a + s + r + f;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
}
__global__ void thr(double* out, int iters) {
  double a[8];
  for (int j = 0; j < 8; j++) a[j] = threadIdx.x + j;
  for (int i = 0; i < iters; i++)
#pragma unroll
    for (int j = 0; j < 8; j++) a[j] = fma(a[j], 1.0000001, 1e-9);
  double s = 0; for (int j = 0; j < 8; j++) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 148 * 1024 * 8); cudaMalloc(&c, 64);
  int it = 1000;
  lat<<<1, 32>>>(o, it, c); cudaDeviceSynchronize();
  long long h[4]; cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
  printf("latency (cycles): dfma %.1f  dsqrt+add %.1f  drcp+add %.1f  ffma %.1f\n", h[0] / (4.0 * it), h[1] / (double)it, h[2] / (double)it, h[3] / (4.0 * it));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  thr<<<148, 512>>>(o, 100);
  cudaEventRecord(a); thr<<<148, 512>>>(o, 10000); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double fl = 148.0 * 512 * 10000 * 8 * 2;
  printf("fp64 FMA throughput: %.2f TFLOP/s (%.1f DFMA/clk/SM at 1.965 GHz)\n", fl / ms / 1e9, fl / 2 / 148 / (ms * 1e-3 * 1.965e9));
}
