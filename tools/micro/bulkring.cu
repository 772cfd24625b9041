// Streaming bandwidth of a 1-D bulk-copy ring (cp.async.bulk global -> shared,
// one producer lane, mbarrier full/empty per stage) vs plain 16-B loads, one
// CTA per SM reading a disjoint contiguous range of a 2 GB buffer.  Consumers
// either touch nothing (mode 0: pure stream) or sum the stage with 16-B shared
// loads (mode 1).  Prints GB/s per (stage KB, stages, mode).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void init(uint32_t b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(c)); }
__device__ __forceinline__ void expect(uint32_t b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(n) : "memory"); }
__device__ __forceinline__ void arrive(uint32_t b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory"); }
__device__ __forceinline__ void wait(uint32_t b, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(b), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(uint32_t dst, const void* src, uint32_t n, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst), "l"(src), "r"(n), "r"(bar) : "memory");
}

__global__ void __launch_bounds__(512, 1) ring(const uint8_t* buf, size_t per_cta, int stage, int nst, int mode, int chunks, float* out, int P) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bars[64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint8_t* src = buf + (size_t)blockIdx.x * per_cta;
  const int ntask = (int)(per_cta / stage);
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) { init(su(&bars[s]), 1); init(su(&bars[32 + s]), 8); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp >= 8) {
    if (lane == 0)
      for (int t = warp - 8; t < ntask; t += P) {
        const int s = t % nst;
        if (t >= nst) wait(su(&bars[32 + s]), ((t / nst) - 1) & 1);
        expect(su(&bars[s]), stage);
        const int cb = stage / chunks;
        for (int c = 0; c < chunks; ++c) bulk(su(sm + (size_t)s * stage + c * cb), src + (size_t)t * stage + c * cb, cb, su(&bars[s]));
      }
    return;
  }
  float acc = 0.f;
  for (int t = 0; t < ntask; ++t) {
    const int s = t % nst;
    wait(su(&bars[s]), (t / nst) & 1);
    if (mode == 1) {
      const uint4* p = reinterpret_cast<const uint4*>(sm + (size_t)s * stage);
      for (int u = threadIdx.x; u < stage / 16; u += 256) { uint4 v = p[u]; acc += __uint_as_float(v.x) + __uint_as_float(v.y); }
    }
    __syncwarp();
    if (lane == 0) arrive(su(&bars[32 + s]));
  }
  if (acc == 12345.f) out[0] = acc;
}

__global__ void ldg(const uint4* buf, size_t n, float* out) {
  float acc = 0.f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = __ldcs(buf + i);
    acc += __uint_as_float(v.x);
  }
  if (acc == 12345.f) out[0] = acc;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t total = (size_t)2 << 30;
  uint8_t* buf; float* out;
  cudaMalloc(&buf, total); cudaMalloc(&out, 4); cudaMemset(buf, 0, total);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  {
    for (int r = 0; r < 2; ++r) {
      cudaEventRecord(e0);
      ldg<<<sms * 8, 256>>>((const uint4*)buf, total / 16, out);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("ldg 16B grid %d x 256: %.0f GB/s\n", sms * 8, total / ms / 1e6);
    }
  }
  for (int P : {1, 2, 4, 8})
  for (int mode = 0; mode < 1; ++mode)
    for (int kb : {4, 10, 20})
      for (int nst : {8, 16})
        for (int chunks : {1}) {
          if (nst % P) continue;
          const int stage = kb * 1024;
          if ((size_t)stage * nst > 216 * 1024 || nst > 32) continue;
          const size_t per = (total / sms) / stage * stage;
          float best = 1e9;
          for (int r = 0; r < 3; ++r) {
            cudaEventRecord(e0);
            ring<<<sms, 256 + 32 * P, (size_t)stage * nst>>>(buf, per, stage, nst, mode, chunks, out, P);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
          }
          cudaError_t err = cudaGetLastError();
          printf("P %d ring mode %d stage %2d KB x %2d (%3d KB in flight) copies/stage %d: %6.0f GB/s %s\n", P, mode, kb, nst, kb * nst, chunks,
                 per * sms / best / 1e6, err == cudaSuccess ? "" : cudaGetErrorString(err));
        }
  return 0;
}
