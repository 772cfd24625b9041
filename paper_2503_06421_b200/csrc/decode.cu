// decode.cu — decode continuation after a template-start prefill (SURVEY.md
// §8(f) f3; §7 l.831, 849-851: the paper continues the first token
// with greedy decode steps).  One token per step through the same model:
//   embed -> L x [shrink, QKV GEMV + RoPE + K/V append, attention over the
//   cache, shrink, O GEMV + residual, shrink, gate/up GEMV + SiLU*mul, shrink,
//   down GEMV + residual] -> head (final norm + GEMV + argmax)
// Every step is HBM-bound: it reads every weight once (the bound is model
// bytes / HBM bandwidth), so the kernels are GEMVs built to keep enough 16-B
// loads in flight per SM, with RMSNorm, RoPE, LoRA, SiLU*mul and the residual
// add fused in.  The step reads its position and input token from device
// state and writes its argmax back, so a step is a fixed launch sequence that
// is captured once as a CUDA graph and replayed: no host round trip per token.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"
#include "launch.cuh"
#include "ptx.cuh"

namespace tidal {

namespace {

constexpr int DT = 256;  // threads per CTA (8 warps)

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float block_sum(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = (threadIdx.x < DT / 32) ? red[threadIdx.x] : 0.f;
  if (w == 0) t = warp_sum(t);
  if (threadIdx.x == 0) red[0] = t;
  __syncthreads();
  t = red[0];
  __syncthreads();
  return t;
}

// x (fp32, shared) <- RMSNorm(X) * g rounded to bf16 (as the prefill's Xn), or
// <- a bf16 vector (attention output / H).  Every CTA builds its own copy.
__device__ __forceinline__ void load_input(float* xs, const float* X, const bf16* g,
                                           const bf16* xin, int K, float eps, float* red) {
  if (X) {
    float ss = 0.f;
    for (int i = threadIdx.x; i < K; i += DT) {
      const float v = X[i];
      ss += v * v;
    }
    const float inv = rsqrtf(block_sum(ss, red) / (float)K + eps);
    for (int i = threadIdx.x; i < K; i += DT)
      xs[i] = __bfloat162float(__float2bfloat16_rn(X[i] * inv * __bfloat162float(g[i])));
  } else {
    for (int i = threadIdx.x; i < K; i += DT) xs[i] = __bfloat162float(xin[i]);
  }
  __syncthreads();
}

// dot products of two weight rows with xs (fp32 in shared memory): 16-B loads,
// four per row in flight per lane, fp32 accumulation
__device__ __forceinline__ void dot2(const bf16* __restrict__ w0, const bf16* __restrict__ w1,
                                     const float* xs, int K, float& a0, float& a1) {
  const int lane = threadIdx.x & 31;
  const uint4* r0 = reinterpret_cast<const uint4*>(w0);
  const uint4* r1 = reinterpret_cast<const uint4*>(w1);
  const int n = K >> 3;
  float s0 = 0.f, s1 = 0.f;
  int i = lane;
  for (; i + 96 < n; i += 128) {
    uint4 u0[4], u1[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      u0[k] = __ldcs(r0 + i + 32 * k);
      u1[k] = __ldcs(r1 + i + 32 * k);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float4* xv = reinterpret_cast<const float4*>(xs + 8 * (i + 32 * k));
      const float4 xa = xv[0], xb = xv[1];
      const __nv_bfloat162* h0 = reinterpret_cast<const __nv_bfloat162*>(&u0[k]);
      const __nv_bfloat162* h1 = reinterpret_cast<const __nv_bfloat162*>(&u1[k]);
      float2 f;
      f = __bfloat1622float2(h0[0]); s0 = fmaf(f.x, xa.x, fmaf(f.y, xa.y, s0));
      f = __bfloat1622float2(h0[1]); s0 = fmaf(f.x, xa.z, fmaf(f.y, xa.w, s0));
      f = __bfloat1622float2(h0[2]); s0 = fmaf(f.x, xb.x, fmaf(f.y, xb.y, s0));
      f = __bfloat1622float2(h0[3]); s0 = fmaf(f.x, xb.z, fmaf(f.y, xb.w, s0));
      f = __bfloat1622float2(h1[0]); s1 = fmaf(f.x, xa.x, fmaf(f.y, xa.y, s1));
      f = __bfloat1622float2(h1[1]); s1 = fmaf(f.x, xa.z, fmaf(f.y, xa.w, s1));
      f = __bfloat1622float2(h1[2]); s1 = fmaf(f.x, xb.x, fmaf(f.y, xb.y, s1));
      f = __bfloat1622float2(h1[3]); s1 = fmaf(f.x, xb.z, fmaf(f.y, xb.w, s1));
    }
  }
  for (; i < n; i += 32) {
    const uint4 u0 = __ldcs(r0 + i), u1 = __ldcs(r1 + i);
    const float4* xv = reinterpret_cast<const float4*>(xs + 8 * i);
    const float4 xa = xv[0], xb = xv[1];
    const __nv_bfloat162* h0 = reinterpret_cast<const __nv_bfloat162*>(&u0);
    const __nv_bfloat162* h1 = reinterpret_cast<const __nv_bfloat162*>(&u1);
    float2 f;
    f = __bfloat1622float2(h0[0]); s0 = fmaf(f.x, xa.x, fmaf(f.y, xa.y, s0));
    f = __bfloat1622float2(h0[1]); s0 = fmaf(f.x, xa.z, fmaf(f.y, xa.w, s0));
    f = __bfloat1622float2(h0[2]); s0 = fmaf(f.x, xb.x, fmaf(f.y, xb.y, s0));
    f = __bfloat1622float2(h0[3]); s0 = fmaf(f.x, xb.z, fmaf(f.y, xb.w, s0));
    f = __bfloat1622float2(h1[0]); s1 = fmaf(f.x, xa.x, fmaf(f.y, xa.y, s1));
    f = __bfloat1622float2(h1[1]); s1 = fmaf(f.x, xa.z, fmaf(f.y, xa.w, s1));
    f = __bfloat1622float2(h1[2]); s1 = fmaf(f.x, xb.x, fmaf(f.y, xb.y, s1));
    f = __bfloat1622float2(h1[3]); s1 = fmaf(f.x, xb.z, fmaf(f.y, xb.w, s1));
  }
  a0 = warp_sum(s0);
  a1 = warp_sum(s1);
}

// LoRA expand term of one output row, B[row, :r] . T (T fp32, scale folded),
// the r products spread over the warp (r <= 64); every lane gets the sum
__device__ __forceinline__ float lora_row(const bf16* B, int row, int r, const float* T) {
  if (!B) return 0.f;
  const int lane = threadIdx.x & 31;
  float s = 0.f;
  if (lane < r) s = __bfloat162float(B[(size_t)row * r + lane]) * T[lane];
  if (lane + 32 < r) s = fmaf(__bfloat162float(B[(size_t)row * r + lane + 32]), T[lane + 32], s);
  return warp_sum(s);
}

// ---------------- embed (token from the previous argmax) ----------------
__global__ void __launch_bounds__(DT) dec_embed_kernel(DecodeState* st, const bf16* __restrict__ E,
                                                       float* __restrict__ X, int d,
                                                       int32_t* toks_out) {
  ptx::pdl_begin();
  const unsigned long long key = st->key;
  const int tok = (int)(0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFu));
  const int t = st->step;
  __syncthreads();  // every thread has read key and step before thread 0 resets them
  if (threadIdx.x == 0) {
    if (t > 0) toks_out[t - 1] = tok;
    st->key = 0ull;  // this step's argmax
    st->step = t + 1;
    st->pos = st->pos0 + t;  // position of the token fed now
  }
  for (int c = threadIdx.x * 8; c < d; c += DT * 8) {
    const uint4 w = *reinterpret_cast<const uint4*>(E + (size_t)tok * d + c);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 f = __bfloat1622float2(h[k]);
      X[c + 2 * k] = f.x;
      X[c + 2 * k + 1] = f.y;
    }
  }
}

__global__ void dec_finish_kernel(DecodeState* st, int32_t* toks_out) {
  ptx::pdl_begin();
  const unsigned long long key = st->key;
  if (threadIdx.x == 0 && st->step > 0)
    toks_out[st->step - 1] = (int)(0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFu));
}

// ---------------- LoRA shrink: T_t = s * A_t . x ----------------
// one warp per output (nt * r <= 192 rows); x = RMSNorm(X)*g or a bf16 vector
__global__ void __launch_bounds__(DT) dec_shrink_kernel(DecShrink a, const float* X, const bf16* g,
                                                        const bf16* xin, int K, float eps,
                                                        float scale) {
  extern __shared__ float xs[];
  __shared__ float red[32];
  ptx::pdl_begin();
  load_input(xs, X, g, xin, K, eps, red);
  const int warp = threadIdx.x >> 5;
  const int rows = a.nt * a.r;
  for (int o = blockIdx.x * (DT / 32) + warp; o < rows; o += gridDim.x * (DT / 32)) {
    const int t = o / a.r, j = o - t * a.r;
    float s0, s1;
    dot2(a.A[t] + (size_t)j * K, a.A[t] + (size_t)j * K, xs, K, s0, s1);
    if ((threadIdx.x & 31) == 0) a.T[t][j] = s0 * scale;
  }
}

// ---------------- GEMV family ----------------
// Row pairs per warp.  QKV: q/k pairs are RoPE partners (h*hd + i, h*hd + i +
// hd/2), v pairs are adjacent rows; GU: (gate i, up i); O / DOWN: adjacent rows.
template <int MODE>
__global__ void __launch_bounds__(DT) dec_gemv_kernel(DecGemv p) {
  extern __shared__ float xs[];
  __shared__ float red[32];
  __shared__ float Ts[3][64];
  ptx::pdl_begin();
  load_input(xs, p.X, p.g, p.xin, p.K, p.eps, red);
  for (int i = threadIdx.x; i < 3 * 64; i += DT) {
    const int t = i / 64, j = i - t * 64;
    Ts[t][j] = (p.T[t] && j < p.r) ? p.T[t][j] : 0.f;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pos = p.st ? p.st->pos : 0;
  for (int pr = blockIdx.x * (DT / 32) + warp; pr < p.npairs; pr += gridDim.x * (DT / 32)) {
    if (MODE == DEC_QKV) {
      const int half = p.hd >> 1;
      const int nqp = p.nq >> 1, nkp = p.nkv >> 1;
      int seg, r0, r1;
      if (pr < nqp + nkp) {  // q or k: RoPE partners
        seg = pr < nqp ? 0 : 1;
        const int pp = seg == 0 ? pr : pr - nqp;
        const int h = pp / half, i = pp - h * half;
        r0 = h * p.hd + i;
        r1 = r0 + half;
      } else {
        seg = 2;
        r0 = 2 * (pr - nqp - nkp);
        r1 = r0 + 1;
      }
      const bf16* W = p.W[seg];
      float a0, a1;
      dot2(W + (size_t)r0 * p.K, W + (size_t)r1 * p.K, xs, p.K, a0, a1);
      a0 += lora_row(p.B[seg], r0, p.r, Ts[seg]);
      a1 += lora_row(p.B[seg], r1, p.r, Ts[seg]);
      if (lane == 0) {
        if (seg < 2) {  // rotate-half RoPE at this token's position
          const float2 cs0 = p.rope[(size_t)pos * half + (r0 % p.hd)];
          const float x1 = a0, x2 = a1;
          a0 = x1 * cs0.x - x2 * cs0.y;
          a1 = x2 * cs0.x + x1 * cs0.y;
        }
        bf16* dst = seg == 0 ? p.q : (seg == 1 ? p.kc + (size_t)pos * p.nkv : p.vc + (size_t)pos * p.nkv);
        dst[r0] = __float2bfloat16_rn(a0);
        dst[r1] = __float2bfloat16_rn(a1);
      }
    } else if (MODE == DEC_GU) {
      float a0, a1;
      dot2(p.W[0] + (size_t)pr * p.K, p.W[1] + (size_t)pr * p.K, xs, p.K, a0, a1);
      const float gt = a0 + lora_row(p.B[0], pr, p.r, Ts[0]);
      const float up = a1 + lora_row(p.B[1], pr, p.r, Ts[1]);
      if (lane == 0) p.h[pr] = __float2bfloat16_rn(gt / (1.f + __expf(-gt)) * up);
    } else {  // DEC_RESID: X[row] += W[row] . x
      const int r0 = 2 * pr, r1 = r0 + 1 < p.N ? r0 + 1 : r0;
      float a0, a1;
      dot2(p.W[0] + (size_t)r0 * p.K, p.W[0] + (size_t)r1 * p.K, xs, p.K, a0, a1);
      a0 += lora_row(p.B[0], r0, p.r, Ts[0]);
      a1 += lora_row(p.B[0], r1, p.r, Ts[0]);
      if (lane == 0) {
        p.Xout[r0] += a0;
        if (r1 != r0) p.Xout[r1] += a1;
      }
    }
  }
}

// ---------------- attention over the cache (one query token) ----------------
// CTA = (head, 256-key chunk): lane = key for the scores, lane = 4 dims for PV;
// partial (max, sum, o[hd]) per chunk; dec_combine folds the chunks in order.
constexpr int ACH = 256;
__global__ void __launch_bounds__(DT) dec_attn_kernel(DecAttn a) {
  __shared__ float qs[128];
  __shared__ float ps[ACH];
  __shared__ float red[32];
  __shared__ float os[DT / 32][128];
  ptx::pdl_begin();
  const int h = blockIdx.x, c = blockIdx.y;
  const int g = h / (a.H / a.KV);
  const int nkeys = a.st->pos + 1;
  const int k0 = c * ACH, k1 = min(nkeys, k0 + ACH);
  float* part = a.part + ((size_t)h * gridDim.y + c) * (2 + 128);
  if (k0 >= k1) {
    if (threadIdx.x == 0) {
      part[0] = -INFINITY;
      part[1] = 0.f;
    }
    return;
  }
  for (int i = threadIdx.x; i < a.hd; i += DT) qs[i] = __bfloat162float(a.q[h * a.hd + i]) * a.scale_log2;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // scores: thread t <-> key k0 + t
  float s = -INFINITY;
  const int k = k0 + threadIdx.x;
  if (k < k1) {
    const uint4* kr = reinterpret_cast<const uint4*>(a.kc + (size_t)k * a.ldkv + g * a.hd);
    float acc = 0.f;
#pragma unroll 4
    for (int i = 0; i < a.hd / 8; ++i) {
      const uint4 u = kr[i];
      const __nv_bfloat162* hh = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(hh[e]);
        acc = fmaf(f.x, qs[8 * i + 2 * e], fmaf(f.y, qs[8 * i + 2 * e + 1], acc));
      }
    }
    s = acc;  // log2 domain (q pre-scaled)
  }
  float m = warp_max(s);
  if (lane == 0) red[warp] = m;
  __syncthreads();
  m = red[0];
  for (int w = 1; w < DT / 32; ++w) m = fmaxf(m, red[w]);
  const float pk = k < k1 ? ptx::ex2(s - m) : 0.f;
  ps[threadIdx.x] = pk;
  __syncthreads();
  float l = warp_sum(pk);
  __syncthreads();
  if (lane == 0) red[warp] = l;
  // PV: warp w takes keys w, w+8, ...; lane owns dims dpl*lane .. (hd = 32 dpl)
  const int dpl = a.hd >> 5;  // 2 or 4
  float o[4] = {0.f, 0.f, 0.f, 0.f};
  for (int kk = warp; kk < k1 - k0; kk += DT / 32) {
    const float pv = ps[kk];
    const bf16* vr = a.vc + (size_t)(k0 + kk) * a.ldkv + g * a.hd + dpl * lane;
    if (dpl == 4) {
      const uint2 u = *reinterpret_cast<const uint2*>(vr);
      const __nv_bfloat162* hh = reinterpret_cast<const __nv_bfloat162*>(&u);
      const float2 f0 = __bfloat1622float2(hh[0]), f1 = __bfloat1622float2(hh[1]);
      o[0] = fmaf(pv, f0.x, o[0]);
      o[1] = fmaf(pv, f0.y, o[1]);
      o[2] = fmaf(pv, f1.x, o[2]);
      o[3] = fmaf(pv, f1.y, o[3]);
    } else {
      const float2 f0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(vr));
      o[0] = fmaf(pv, f0.x, o[0]);
      o[1] = fmaf(pv, f0.y, o[1]);
    }
  }
  for (int e = 0; e < dpl; ++e) os[warp][dpl * lane + e] = o[e];
  __syncthreads();
  if (threadIdx.x < a.hd) {
    float acc = 0.f;
    for (int w = 0; w < DT / 32; ++w) acc += os[w][threadIdx.x];  // fixed order
    part[2 + threadIdx.x] = acc;
  }
  if (threadIdx.x == 0) {
    float lt = 0.f;
    for (int w = 0; w < DT / 32; ++w) lt += red[w];
    part[0] = m;
    part[1] = lt;
  }
}

__global__ void dec_combine_kernel(DecAttn a, int nchunks) {
  ptx::pdl_begin();
  const int h = blockIdx.x, i = threadIdx.x;
  const float* part = a.part + (size_t)h * nchunks * (2 + 128);
  float m = -INFINITY;
  for (int c = 0; c < nchunks; ++c) m = fmaxf(m, part[c * 130]);
  float l = 0.f, o = 0.f;
  for (int c = 0; c < nchunks; ++c) {  // chunk order: deterministic
    const float mc = part[c * 130];
    if (mc == -INFINITY) continue;
    const float w = ptx::ex2(mc - m);
    l = fmaf(w, part[c * 130 + 1], l);
    o = fmaf(w, part[c * 130 + 2 + i], o);
  }
  if (i < a.hd) a.out[h * a.hd + i] = __float2bfloat16_rn(o / l);
}

__global__ void dec_save_logits_kernel(const DecodeState* st, const float* logits, float* all, int V) {
  ptx::pdl_begin();
  float* dst = all + (size_t)(st->step - 1) * V;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < V; i += gridDim.x * blockDim.x)
    dst[i] = logits[i];
}

int gemv_grid(int num_sms) { return num_sms * 2; }

}  // namespace

cudaError_t dec_embed_launch(DecodeState* st, const bf16* E, float* X, int d, int32_t* toks_out,
                             cudaStream_t s) {
  return launch_k(dec_embed_kernel, dim3(1), dim3(DT), 0, s, 1, st, E, X, d, toks_out);
}
cudaError_t dec_finish_launch(DecodeState* st, int32_t* toks_out, cudaStream_t s) {
  return launch_k(dec_finish_kernel, dim3(1), dim3(32), 0, s, 1, st, toks_out);
}

cudaError_t dec_save_logits_launch(const DecodeState* st, const float* logits, float* all, int V,
                                   cudaStream_t s) {
  return launch_k(dec_save_logits_kernel, dim3((V + 1023) / 1024), dim3(1024), 0, s, 1, st, logits,
                  all, V);
}

cudaError_t dec_shrink_launch(const DecShrink& a, const float* X, const bf16* g, const bf16* xin,
                              int K, float eps, float scale, int num_sms, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(dec_shrink_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         160 * 1024);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int rows = a.nt * a.r;
  int grid = (rows + DT / 32 - 1) / (DT / 32);
  (void)num_sms;
  return launch_k(dec_shrink_kernel, dim3(grid), dim3(DT), (size_t)K * 4, s, 1, a, X, g, xin, K, eps,
                  scale);
}

cudaError_t dec_gemv_launch(const DecGemv& p, int mode, int num_sms, cudaStream_t s) {
  static bool attr[3] = {false, false, false};
  auto k = mode == DEC_QKV ? dec_gemv_kernel<DEC_QKV>
                           : (mode == DEC_GU ? dec_gemv_kernel<DEC_GU> : dec_gemv_kernel<DEC_RESID>);
  if (!attr[mode]) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    if (e != cudaSuccess) return e;
    attr[mode] = true;
  }
  int grid = gemv_grid(num_sms);
  const int need = (p.npairs + DT / 32 - 1) / (DT / 32);
  if (grid > need) grid = need;
  return launch_k(k, dim3(grid), dim3(DT), (size_t)p.K * 4, s, 1, p);
}

cudaError_t dec_attn_launch(const DecAttn& a, int max_keys, cudaStream_t s) {
  const int nchunks = (max_keys + ACH - 1) / ACH;
  cudaError_t e = launch_k(dec_attn_kernel, dim3(a.H, nchunks), dim3(DT), 0, s, 1, a);
  if (e != cudaSuccess) return e;
  return launch_k(dec_combine_kernel, dim3(a.H), dim3(128), 0, s, 1, a, nchunks);
}

}  // namespace tidal
