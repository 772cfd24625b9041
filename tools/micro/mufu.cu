// MUFU.EX2 vs FFMA issue throughput per SM (B200): 8 independent chains per
// thread, 1 CTA of 256 threads per SM, clock64 around the loop.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
template <int MODE>
__global__ void k(float* out, long long* cyc, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) a[i] = ex2(a[i]) - 1.0f;          // MUFU + FADD
      else if (MODE == 1) a[i] = fmaf(a[i], 0.999f, -0.001f);  // FFMA
      else a[i] = ex2(fmaf(a[i], 0.999f, -0.001f));   // FFMA + MUFU
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* o; long long* c; cudaMalloc(&o, 148 * 1024 * 4); cudaMalloc(&c, 148 * 8);
  const int iters = 4096;
  for (int threads : {128, 256, 512, 1024}) {
    for (int mode = 0; mode < 3; ++mode) {
      auto f = mode == 0 ? k<0> : mode == 1 ? k<1> : k<2>;
      f<<<148, threads>>>(o, c, iters); cudaDeviceSynchronize();
      f<<<148, threads>>>(o, c, iters); cudaDeviceSynchronize();
      long long h[148]; cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
      double ops = (double)threads * iters * 8;
      printf("threads %4d mode %d (%s): %.2f ops/clk/SM\n", threads, mode,
             mode == 0 ? "ex2+fadd" : mode == 1 ? "ffma" : "ffma+ex2", ops / h[0]);
    }
  }
  return 0;
}
