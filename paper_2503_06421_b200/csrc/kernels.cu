// kernels.cu — memory-bound kernels of the prefill path (sm_100a):
// embedding gather, RMSNorm, LoRA shrink (x A^T, legacy mma.sync — a skinny
// r <= 64 product whose cost is reading x), the lm-head GEMV with fused final
// RMSNorm and argmax, and debug/invariant kernels.  All HBM-bound: 16-byte
// vector loads, one row per CTA or warp, grids sized to the SM count.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"

namespace tidal {

namespace {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int NT>
__device__ __forceinline__ float block_sum(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = (threadIdx.x < NT / 32) ? red[threadIdx.x] : 0.f;
  if (w == 0) t = warp_sum(t);
  if (threadIdx.x == 0) red[0] = t;
  __syncthreads();
  t = red[0];
  __syncthreads();
  return t;
}

// ---------------- embedding gather ----------------
__global__ void embed_kernel(const int32_t* __restrict__ tok, const bf16* __restrict__ E,
                             float* __restrict__ X, int d, int row0, int rows) {
  const int s = blockIdx.x;
  const int t = tok[s] - row0;
  const bool mine = t >= 0 && t < rows;
  float* x = X + (size_t)s * d;
  for (int c = threadIdx.x * 8; c < d; c += blockDim.x * 8) {
    float4 lo = make_float4(0.f, 0.f, 0.f, 0.f), hi = lo;
    if (mine) {
      uint4 w = *reinterpret_cast<const uint4*>(E + (size_t)t * d + c);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w);
      float2 a = __bfloat1622float2(h[0]), b = __bfloat1622float2(h[1]);
      float2 e = __bfloat1622float2(h[2]), f = __bfloat1622float2(h[3]);
      lo = make_float4(a.x, a.y, b.x, b.y);
      hi = make_float4(e.x, e.y, f.x, f.y);
    }
    *reinterpret_cast<float4*>(x + c) = lo;
    *reinterpret_cast<float4*>(x + c + 4) = hi;
  }
}

// ---------------- RMSNorm ----------------
constexpr int NORM_THREADS = 256;
__global__ void __launch_bounds__(NORM_THREADS) rmsnorm_kernel(const float* __restrict__ X,
                                                               const bf16* __restrict__ g,
                                                               bf16* __restrict__ Y, int d,
                                                               float eps) {
  __shared__ float red[32];
  const float4* x = reinterpret_cast<const float4*>(X + (size_t)blockIdx.x * d);
  const int n4 = d >> 2;
  float ss = 0.f;
  for (int i = threadIdx.x; i < n4; i += NORM_THREADS) {
    float4 v = x[i];
    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  ss = block_sum<NORM_THREADS>(ss, red);
  const float inv = rsqrtf(ss / (float)d + eps);
  uint2* y = reinterpret_cast<uint2*>(Y + (size_t)blockIdx.x * d);
  const uint2* g2 = reinterpret_cast<const uint2*>(g);
  for (int i = threadIdx.x; i < n4; i += NORM_THREADS) {
    float4 v = x[i];
    uint2 gw = g2[i];
    const __nv_bfloat162* gh = reinterpret_cast<const __nv_bfloat162*>(&gw);
    float2 g01 = __bfloat1622float2(gh[0]), g23 = __bfloat1622float2(gh[1]);
    __nv_bfloat162 r0 = __floats2bfloat162_rn(v.x * inv * g01.x, v.y * inv * g01.y);
    __nv_bfloat162 r1 = __floats2bfloat162_rn(v.z * inv * g23.x, v.w * inv * g23.y);
    uint2 o;
    o.x = *reinterpret_cast<uint32_t*>(&r0);
    o.y = *reinterpret_cast<uint32_t*>(&r1);
    y[i] = o;
  }
}

// ---------------- LoRA shrink: T = scale * X A^T (mma.sync m16n8k16) ----------------
// CTA = 64 rows x one target; 4 warps x 16 rows; K in steps of 32 through a
// 2-stage cp.async ring.  r <= 64.
constexpr int SH_BM = 64, SH_BK = 32, SH_LD = 40;  // smem row stride (elements), conflict-free

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(n)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(p);
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(s));
}
__device__ __forceinline__ void ldsm_x2(uint32_t (&r)[2], const void* p) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(p);
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];"
               : "=r"(r[0]), "=r"(r[1])
               : "r"(s));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4],
                                         const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

struct ShrinkArgs {
  const bf16* A[3];
  bf16* T[3];
};

template <int R>
__global__ void __launch_bounds__(128) lora_shrink_kernel(const bf16* __restrict__ X, int ldx, int M,
                                                          int K, ShrinkArgs args, float scale) {
  __shared__ __align__(16) bf16 xs[2][SH_BM * SH_LD];
  __shared__ __align__(16) bf16 as[2][R * SH_LD];
  const int t = blockIdx.y;
  const bf16* __restrict__ A = args.A[t];
  const int m0 = blockIdx.x * SH_BM;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float acc[R / 8][4];
#pragma unroll
  for (int i = 0; i < R / 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
  const int nk = (K + SH_BK - 1) / SH_BK;
  auto load = [&](int kb, int buf) {
    const int k0 = kb * SH_BK;
    for (int c = threadIdx.x; c < SH_BM * 4; c += 128) {
      const int r = c >> 2, ch = c & 3;
      const int m = m0 + r, k = k0 + ch * 8;
      const bool ok = m < M && k < K;
      cp_async16(&xs[buf][r * SH_LD + ch * 8], ok ? X + (size_t)m * ldx + k : X, ok);
    }
    for (int c = threadIdx.x; c < R * 4; c += 128) {
      const int r = c >> 2, ch = c & 3;
      const int k = k0 + ch * 8;
      const bool ok = k < K;
      cp_async16(&as[buf][r * SH_LD + ch * 8], ok ? A + (size_t)r * K + k : A, ok);
    }
    cp_commit();
  };
  load(0, 0);
  for (int kb = 0; kb < nk; ++kb) {
    const int buf = kb & 1;
    if (kb + 1 < nk) {
      load(kb + 1, buf ^ 1);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < SH_BK / 16; ++kk) {
      uint32_t a[4];
      const int ar = warp * 16 + (lane & 15), ac = kk * 16 + (lane >> 4) * 8;
      ldsm_x4(a, &xs[buf][ar * SH_LD + ac]);
#pragma unroll
      for (int nt = 0; nt < R / 8; ++nt) {
        uint32_t b[2];
        const int br = nt * 8 + (lane & 7), bc = kk * 16 + ((lane >> 3) & 1) * 8;
        ldsm_x2(b, &as[buf][br * SH_LD + bc]);
        mma16816(acc[nt], a, b);
      }
    }
    __syncthreads();
  }
  bf16* T = args.T[t];
  const int r0 = m0 + warp * 16 + (lane >> 2);
#pragma unroll
  for (int nt = 0; nt < R / 8; ++nt) {
    const int c = nt * 8 + 2 * (lane & 3);
    if (r0 < M)
      *reinterpret_cast<__nv_bfloat162*>(T + (size_t)r0 * R + c) =
          __floats2bfloat162_rn(acc[nt][0] * scale, acc[nt][1] * scale);
    if (r0 + 8 < M)
      *reinterpret_cast<__nv_bfloat162*>(T + (size_t)(r0 + 8) * R + c) =
          __floats2bfloat162_rn(acc[nt][2] * scale, acc[nt][3] * scale);
  }
}

// ---------------- lm head: final norm + GEMV + argmax ----------------
constexpr int HEAD_THREADS = 256;
__device__ __forceinline__ unsigned long long argmax_key(float v, int idx) {
  uint32_t u = __float_as_uint(v);
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return ((unsigned long long)u << 32) | (unsigned long long)(0xFFFFFFFFu - (uint32_t)idx);
}

__global__ void __launch_bounds__(HEAD_THREADS) head_kernel(const float* __restrict__ xlast,
                                                            const bf16* __restrict__ g,
                                                            const bf16* __restrict__ W, int V,
                                                            int d, float eps,
                                                            float* __restrict__ logits,
                                                            unsigned long long* key, int voff) {
  extern __shared__ float hs[];  // d floats
  __shared__ float red[32];
  __shared__ unsigned long long kred[HEAD_THREADS / 32];
  float ss = 0.f;
  for (int i = threadIdx.x; i < d; i += HEAD_THREADS) {
    const float v = xlast[i];
    ss += v * v;
  }
  ss = block_sum<HEAD_THREADS>(ss, red);
  const float inv = rsqrtf(ss / (float)d + eps);
  for (int i = threadIdx.x; i < d; i += HEAD_THREADS) hs[i] = xlast[i] * inv * __bfloat162float(g[i]);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * (HEAD_THREADS / 32) + warp;
  const int nw = gridDim.x * (HEAD_THREADS / 32);
  unsigned long long best = 0;
  for (int v = gw; v < V; v += nw) {
    const bf16* w = W + (size_t)v * d;
    float acc = 0.f;
    for (int c = lane * 8; c < d; c += 256) {
      uint4 q = __ldg(reinterpret_cast<const uint4*>(w + c));
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
      const float4 x0 = *reinterpret_cast<const float4*>(hs + c);
      const float4 x1 = *reinterpret_cast<const float4*>(hs + c + 4);
      float2 a = __bfloat1622float2(h[0]), b = __bfloat1622float2(h[1]);
      float2 e = __bfloat1622float2(h[2]), f = __bfloat1622float2(h[3]);
      acc += a.x * x0.x + a.y * x0.y + b.x * x0.z + b.y * x0.w + e.x * x1.x + e.y * x1.y +
             f.x * x1.z + f.y * x1.w;
    }
    acc = warp_sum(acc);
    if (lane == 0) {
      logits[v] = acc;
      const unsigned long long k = argmax_key(acc, v + voff);
      best = k > best ? k : best;
    }
  }
  if (lane == 0) kred[warp] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long b = 0;
    for (int i = 0; i < HEAD_THREADS / 32; ++i) b = kred[i] > b ? kred[i] : b;
    if (b) atomicMax(key, b);
  }
}

// ---------------- debug / invariants ----------------
__global__ void poison_kernel(uint16_t* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    p[i] = 0x7FC0;
}

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
// order-independent: sum_i mix(word_i + i * golden)
__global__ void checksum_kernel(const unsigned long long* p, size_t n, unsigned long long* out) {
  unsigned long long s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    s += mix64(p[i] + i * 0x9E3779B97F4A7C15ull);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, s);
}

__global__ void nan_check_kernel(const float* x, int n, int* flag) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    if (isnan(x[i])) *flag = 1;
}

}  // namespace

cudaError_t embed_launch(const int32_t* tok, const bf16* E, float* X, int S, int d, int row0,
                         int rows, cudaStream_t s) {
  int th = d / 8;
  if (th > 1024) th = 1024;
  if (th < 32) th = 32;
  embed_kernel<<<S, th, 0, s>>>(tok, E, X, d, row0, rows);
  return cudaGetLastError();
}

cudaError_t rmsnorm_launch(const float* X, const bf16* g, bf16* Y, int S, int d, float eps,
                           cudaStream_t s) {
  rmsnorm_kernel<<<S, NORM_THREADS, 0, s>>>(X, g, Y, d, eps);
  return cudaGetLastError();
}

cudaError_t lora_shrink_launch(const bf16* X, int ldx, int M, int K, const bf16* const* A,
                               bf16* const* T, int nt, int r, float scale, cudaStream_t s) {
  ShrinkArgs a{};
  for (int i = 0; i < nt && i < 3; ++i) {
    a.A[i] = A[i];
    a.T[i] = T[i];
  }
  dim3 grid((M + SH_BM - 1) / SH_BM, nt);
  switch (r) {
    case 8: lora_shrink_kernel<8><<<grid, 128, 0, s>>>(X, ldx, M, K, a, scale); break;
    case 16: lora_shrink_kernel<16><<<grid, 128, 0, s>>>(X, ldx, M, K, a, scale); break;
    case 32: lora_shrink_kernel<32><<<grid, 128, 0, s>>>(X, ldx, M, K, a, scale); break;
    case 64: lora_shrink_kernel<64><<<grid, 128, 0, s>>>(X, ldx, M, K, a, scale); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t head_launch(const float* X_last, const bf16* g, const bf16* W, int V, int d, float eps,
                        float* logits, unsigned long long* key, int vocab_offset, int num_sms,
                        cudaStream_t s) {
  const size_t smem = (size_t)d * sizeof(float);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(head_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
  }
  int grid = num_sms * 4;
  const int need = (V + HEAD_THREADS / 32 - 1) / (HEAD_THREADS / 32);
  if (grid > need) grid = need;
  head_kernel<<<grid, HEAD_THREADS, smem, s>>>(X_last, g, W, V, d, eps, logits, key, vocab_offset);
  return cudaGetLastError();
}

cudaError_t poison_launch(void* p, size_t bytes, cudaStream_t s) {
  if (!bytes) return cudaSuccess;
  poison_kernel<<<1184, 256, 0, s>>>(reinterpret_cast<uint16_t*>(p), bytes / 2);
  return cudaGetLastError();
}

cudaError_t checksum_launch(const void* p, size_t bytes, unsigned long long* out, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
  if (bytes >= 8)
    checksum_kernel<<<1184, 256, 0, s>>>(reinterpret_cast<const unsigned long long*>(p), bytes / 8,
                                         out);
  return cudaGetLastError();
}

cudaError_t scrub_launch(void* p, size_t bytes, cudaStream_t s) {
  return cudaMemsetAsync(p, 0x5A, bytes, s);
}

cudaError_t nan_check_launch(const float* x, int n, int* flag, cudaStream_t s) {
  nan_check_kernel<<<64, 256, 0, s>>>(x, n, flag);
  return cudaGetLastError();
}

}  // namespace tidal
