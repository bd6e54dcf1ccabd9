"""Instruction-cache capacity probe (B200): kernels of N straight-line FMAs
(16 B each; 8 independent chains so issue, not latency, bounds the warm rate),
one CTA per SM.  Each size is launched 3x: after an L2 flush (code from HBM
unless the SM's instruction cache still holds it), then twice back to back.
Prints cycles per instruction for each launch.

  python tools/icache_bench.py   (needs nvcc + a GPU; writes /tmp/icache_*.cu)
"""
import os, subprocess, sys

SIZES = [1024, 2048, 4096, 6144, 8192, 10240, 12288, 16384]
HERE = os.path.dirname(os.path.abspath(__file__))


def kernel_src(n):
    body = []
    for i in range(n):
        a = i % 8
        body.append(f'"fma.rn.f32 %{a}, %{a}, %8, %9;\\n"')
    asm = "\n      ".join(body)
    return f"""
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(float* out, long long* cyc, float s, float t) {{
  float r0 = threadIdx.x, r1 = r0 + 1, r2 = r0 + 2, r3 = r0 + 3, r4 = r0 + 4, r5 = r0 + 5, r6 = r0 + 6, r7 = r0 + 7;
  long long t0 = clock64();
  asm volatile(
      {asm}
      : "+f"(r0), "+f"(r1), "+f"(r2), "+f"(r3), "+f"(r4), "+f"(r5), "+f"(r6), "+f"(r7) : "f"(s), "f"(t));
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = r0 + r1 + r2 + r3 + r4 + r5 + r6 + r7;
}}
__global__ void flush(float* b, size_t n) {{
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] += 1.f;
}}
int main() {{
  float *out, *fb; long long* cyc; const size_t fn = (size_t)256 << 20;
  cudaMalloc(&out, 148 * 32 * 4); cudaMalloc(&cyc, 148 * 8); cudaMalloc(&fb, fn * 4);
  long long h[148];
  for (int rep = 0; rep < 2; rep++) {{
    flush<<<592, 512>>>(fb, fn);
    for (int l = 0; l < 3; l++) {{
      k<<<148, 32>>>(out, cyc, 1.0001f, 0.5f);
      cudaDeviceSynchronize();
      cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
      long long s = 0; for (int i = 0; i < 148; i++) s += h[i];
      printf("%s%.2f", l ? " " : "", (double)s / 148 / {n});
    }}
    printf(rep ? "\\n" : " |");
  }}
  return cudaGetLastError() != cudaSuccess;
}}
"""


def main():
    os.makedirs(os.path.join(HERE, "bin"), exist_ok=True)
    build_only = "--build" in sys.argv
    for n in SIZES:
        src = f"/tmp/icache_{n}.cu"
        exe = os.path.join(HERE, "bin", f"icache_{n}")
        if not os.path.exists(exe):
            open(src, "w").write(kernel_src(n))
            subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", src, "-o", exe], check=True)
        if build_only:
            continue
        r = subprocess.run([exe], capture_output=True, text=True)
        print(f"{n:6d} instr ({n * 16 // 1024:4d} KB) cycles/instr [flushed, warm, warm | again]: {r.stdout.strip()}",
              flush=True)


if __name__ == "__main__":
    main()
