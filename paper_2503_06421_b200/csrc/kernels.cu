// kernels.cu — memory-bound kernels of the prefill path (sm_100a):
// embedding gather, RMSNorm, the lm-head GEMV with fused final RMSNorm and
// argmax, the TP bf16-allreduce pack/add, and debug/invariant kernels.  All HBM-bound: 16-byte
// vector loads, one row per CTA or warp, grids sized to the SM count.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"
#include "launch.cuh"
#include "ptx.cuh"

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
                             float* __restrict__ X, int d, int row0, int rows,
                             unsigned long long* key_reset, int n_keys) {
  ptx::pdl_begin();
  if (key_reset && blockIdx.x == 0 && threadIdx.x < n_keys) key_reset[threadIdx.x] = 0ull;  // argmax keys
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
constexpr int NORM_THREADS = 256, NORM_VEC = 8;
__global__ void __launch_bounds__(NORM_THREADS) rmsnorm_kernel(const float* __restrict__ X,
                                                               const bf16* __restrict__ g,
                                                               bf16* __restrict__ Y, int d,
                                                               float eps) {
  __shared__ float red[32];
  ptx::pdl_begin();
  const float4* x = reinterpret_cast<const float4*>(X + (size_t)blockIdx.x * d);
  const int n4 = d >> 2;
  // the row stays in registers: one HBM read of X (d <= 4 * 256 * NORM_VEC)
  float4 v[NORM_VEC];
  float ss = 0.f;
#pragma unroll
  for (int j = 0; j < NORM_VEC; ++j) {
    const int i = threadIdx.x + j * NORM_THREADS;
    v[j] = i < n4 ? x[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    ss += v[j].x * v[j].x + v[j].y * v[j].y + v[j].z * v[j].z + v[j].w * v[j].w;
  }
  ss = block_sum<NORM_THREADS>(ss, red);
  const float inv = rsqrtf(ss / (float)d + eps);
  uint2* y = reinterpret_cast<uint2*>(Y + (size_t)blockIdx.x * d);
  const uint2* g2 = reinterpret_cast<const uint2*>(g);
#pragma unroll
  for (int j = 0; j < NORM_VEC; ++j) {
    const int i = threadIdx.x + j * NORM_THREADS;
    if (i >= n4) break;
    const float4 vv = v[j];
    uint2 gw = g2[i];
    const __nv_bfloat162* gh = reinterpret_cast<const __nv_bfloat162*>(&gw);
    float2 g01 = __bfloat1622float2(gh[0]), g23 = __bfloat1622float2(gh[1]);
    __nv_bfloat162 r0 = __floats2bfloat162_rn(vv.x * inv * g01.x, vv.y * inv * g01.y);
    __nv_bfloat162 r1 = __floats2bfloat162_rn(vv.z * inv * g23.x, vv.w * inv * g23.y);
    uint2 o;
    o.x = *reinterpret_cast<uint32_t*>(&r0);
    o.y = *reinterpret_cast<uint32_t*>(&r1);
    y[i] = o;
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
                                                            size_t x_stride, int nrows,
                                                            const bf16* __restrict__ g,
                                                            const bf16* __restrict__ W, int V,
                                                            int d, float eps,
                                                            float* __restrict__ logits, int ldl,
                                                            unsigned long long* key, int voff) {
  extern __shared__ float hs[];  // nrows x d floats: the normalised last rows
  __shared__ float red[32];
  __shared__ unsigned long long kred[HEAD_MAX_ROWS][HEAD_THREADS / 32];
  ptx::pdl_begin();
  for (int b = 0; b < nrows; ++b) {
    const float* x = xlast + (size_t)b * x_stride;
    float ss = 0.f;
    for (int i = threadIdx.x; i < d; i += HEAD_THREADS) {
      const float v = x[i];
      ss += v * v;
    }
    ss = block_sum<HEAD_THREADS>(ss, red);
    const float inv = rsqrtf(ss / (float)d + eps);
    for (int i = threadIdx.x; i < d; i += HEAD_THREADS)
      hs[b * d + i] = x[i] * inv * __bfloat162float(g[i]);
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * (HEAD_THREADS / 32) + warp;
  const int nw = gridDim.x * (HEAD_THREADS / 32);
  unsigned long long best[HEAD_MAX_ROWS];
#pragma unroll
  for (int b = 0; b < HEAD_MAX_ROWS; ++b) best[b] = 0;
  // The warp's rows v = gw, gw + nw, ... are streamed as one sequence of
  // 2048-element batches (8 x 16-B loads per lane); the next batch — possibly
  // the next row's first — is issued before the current one is consumed, so
  // every warp keeps two batches (16 loads per lane) in flight and a row costs
  // no dependent round trip of its own.
  constexpr int BU = 8, BE = BU * 256;  // loads per lane, elements per batch
  const int nbr = (d + BE - 1) / BE;    // batches per row
  auto load = [&](int v, int b, uint4 (&q)[BU]) {
    const bf16* w = W + (size_t)v * d + b * BE + lane * 8;
#pragma unroll
    for (int u = 0; u < BU; ++u)
      q[u] = (b * BE + u * 256 + lane * 8 < d) ? __ldcs(reinterpret_cast<const uint4*>(w + u * 256))
                                               : make_uint4(0, 0, 0, 0);
  };
  float acc[HEAD_MAX_ROWS];
#pragma unroll
  for (int r = 0; r < HEAD_MAX_ROWS; ++r) acc[r] = 0.f;
  uint4 cur[BU];
  int v = gw, b = 0;
  if (v < V) load(v, b, cur);
  while (v < V) {
    int vn = v, bn = b + 1;
    if (bn == nbr) {
      bn = 0;
      vn = v + nw;
    }
    uint4 nxt[BU];
    if (vn < V) load(vn, bn, nxt);
#pragma unroll
    for (int u = 0; u < BU; ++u) {
      const int c = b * BE + u * 256 + lane * 8;
      if (c >= d) break;
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&cur[u]);
      const float2 a = __bfloat1622float2(h[0]), bb = __bfloat1622float2(h[1]);
      const float2 e = __bfloat1622float2(h[2]), f = __bfloat1622float2(h[3]);
#pragma unroll
      for (int r = 0; r < HEAD_MAX_ROWS; ++r) {
        if (r >= nrows) break;
        const float4 x0 = *reinterpret_cast<const float4*>(hs + r * d + c);
        const float4 x1 = *reinterpret_cast<const float4*>(hs + r * d + c + 4);
        acc[r] += a.x * x0.x + a.y * x0.y + bb.x * x0.z + bb.y * x0.w + e.x * x1.x + e.y * x1.y +
                  f.x * x1.z + f.y * x1.w;
      }
    }
    if (bn == 0) {  // row v complete
#pragma unroll
      for (int r = 0; r < HEAD_MAX_ROWS; ++r) {
        if (r >= nrows) break;
        const float t = warp_sum(acc[r]);
        acc[r] = 0.f;
        if (lane == 0) {
          logits[(size_t)r * ldl + v] = t;
          const unsigned long long k = argmax_key(t, v + voff);
          best[r] = k > best[r] ? k : best[r];
        }
      }
    }
#pragma unroll
    for (int u = 0; u < BU; ++u) cur[u] = nxt[u];
    v = vn;
    b = bn;
  }
  if (lane == 0)
#pragma unroll
    for (int b = 0; b < HEAD_MAX_ROWS; ++b) kred[b][warp] = best[b];
  __syncthreads();
  if (threadIdx.x < nrows) {
    unsigned long long m = 0;
    for (int i = 0; i < HEAD_THREADS / 32; ++i) m = kred[threadIdx.x][i] > m ? kred[threadIdx.x][i] : m;
    if (m) atomicMax(key + threadIdx.x, m);
  }
}

// ---------------- TP bf16 allreduce option ----------------
// Pb = bf16(P) (the row-parallel partial sum), and after the allreduce X += Pb.
__global__ void f32_to_bf16_kernel(const float4* __restrict__ P, uint2* __restrict__ Pb, size_t n4) {
  ptx::pdl_begin();
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4;
       i += (size_t)gridDim.x * blockDim.x) {
    const float4 v = P[i];
    __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    uint2 o;
    o.x = *reinterpret_cast<uint32_t*>(&a);
    o.y = *reinterpret_cast<uint32_t*>(&b);
    Pb[i] = o;
  }
}

__global__ void add_bf16_kernel(const uint2* __restrict__ Pb, float4* __restrict__ X, size_t n4) {
  ptx::pdl_begin();
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4;
       i += (size_t)gridDim.x * blockDim.x) {
    uint2 w = Pb[i];
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w);
    const float2 a = __bfloat1622float2(h[0]), b = __bfloat1622float2(h[1]);
    float4 x = X[i];
    x.x += a.x;
    x.y += a.y;
    x.z += b.x;
    x.w += b.y;
    X[i] = x;
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
                         int rows, cudaStream_t s, unsigned long long* key_reset, int n_keys) {
  int th = d / 8;
  if (th > 1024) th = 1024;
  if (th < 32) th = 32;
  if (key_reset && n_keys > th) return cudaErrorInvalidValue;
  return launch_k(embed_kernel, dim3(S), dim3(th), 0, s, 1, tok, E, X, d, row0, rows, key_reset,
                  n_keys);
}

cudaError_t rmsnorm_launch(const float* X, const bf16* g, bf16* Y, int S, int d, float eps,
                           cudaStream_t s) {
  return launch_k(rmsnorm_kernel, dim3(S), dim3(NORM_THREADS), 0, s, 1, X, g, Y, d, eps);
}

cudaError_t head_launch(const float* X_last, size_t x_stride, int nseq, const bf16* g, const bf16* W,
                        int V, int d, float eps, float* logits, int ldl, unsigned long long* key,
                        int vocab_offset, int num_sms, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(head_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         200 * 1024);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  // rows per launch: the normalised rows must fit the 200 KB of shared memory
  int per = (int)((200 * 1024) / ((size_t)d * sizeof(float)));
  per = per < HEAD_MAX_ROWS ? per : HEAD_MAX_ROWS;
  if (per < 1) return cudaErrorInvalidValue;
  // one wave of co-resident CTAs (the shared rows and ~125 registers per
  // thread allow 2 per SM at d = 5120)
  static size_t occ_smem = 0;
  static int per_sm = 0;
  const size_t smem = (size_t)(nseq < per ? nseq : per) * d * sizeof(float);
  if (smem != occ_smem || per_sm < 1) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, head_kernel, HEAD_THREADS, smem) !=
            cudaSuccess ||
        per_sm < 1)
      per_sm = 1;
    occ_smem = smem;
  }
  int grid = num_sms * per_sm;
  const int need = (V + HEAD_THREADS / 32 - 1) / (HEAD_THREADS / 32);
  if (grid > need) grid = need;
  for (int b0 = 0; b0 < nseq; b0 += per) {
    const int nr = nseq - b0 < per ? nseq - b0 : per;
    const cudaError_t e = launch_k(head_kernel, dim3(grid), dim3(HEAD_THREADS),
                                   (size_t)nr * d * sizeof(float), s, 1, X_last + b0 * x_stride,
                                   x_stride, nr, g, W, V, d, eps, logits + (size_t)b0 * ldl, ldl,
                                   key + b0, vocab_offset);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t tp_pack_bf16_launch(const float* P, bf16* Pb, size_t n, int num_sms, cudaStream_t s) {
  if (n % 4) return cudaErrorInvalidValue;
  return launch_k(f32_to_bf16_kernel, dim3(num_sms * 4), dim3(256), 0, s, 1,
                  reinterpret_cast<const float4*>(P), reinterpret_cast<uint2*>(Pb), n / 4);
}

cudaError_t tp_add_bf16_launch(const bf16* Pb, float* X, size_t n, int num_sms, cudaStream_t s) {
  if (n % 4) return cudaErrorInvalidValue;
  return launch_k(add_bf16_kernel, dim3(num_sms * 4), dim3(256), 0, s, 1,
                  reinterpret_cast<const uint2*>(Pb), reinterpret_cast<float4*>(X), n / 4);
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
