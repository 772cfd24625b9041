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
#include <cstdlib>

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
template <int NT = DT>
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

// x (fp32, shared) <- RMSNorm(X) * g rounded to bf16 (as the prefill's Xn), or
// <- a bf16 vector (attention output / H).  Every CTA builds its own copy;
// 16-B vector loads, all of a thread's loads issued before any is consumed
// (K <= 16384: at most 16 float4 per thread), the raw row parked in shared
// memory between the two passes.
template <int NT = DT>
__device__ __forceinline__ void load_input(float* xs, const float* X, const bf16* g,
                                           const bf16* xin, int K, float eps, float* red) {
  if (X) {  // K = d_model <= 16384
    const float4* X4 = reinterpret_cast<const float4*>(X);
    float4* xs4 = reinterpret_cast<float4*>(xs);
    const int n4 = K >> 2;
    float4 v[16 * DT / NT];
#pragma unroll
    for (int k = 0; k < 16 * DT / NT; ++k) {
      const int i = threadIdx.x + k * NT;
      if (i < n4) v[k] = X4[i];
    }
    float ss = 0.f;
#pragma unroll
    for (int k = 0; k < 16 * DT / NT; ++k) {
      const int i = threadIdx.x + k * NT;
      if (i < n4) {
        ss += v[k].x * v[k].x + v[k].y * v[k].y + v[k].z * v[k].z + v[k].w * v[k].w;
        xs4[i] = v[k];
      }
    }
    const float inv = rsqrtf(block_sum<NT>(ss, red) / (float)K + eps);
    const uint2* g4 = reinterpret_cast<const uint2*>(g);
#pragma unroll
    for (int k = 0; k < 16 * DT / NT; ++k) {
      const int i = threadIdx.x + k * NT;
      if (i < n4) {
        const uint2 gw = g4[i];
        const __nv_bfloat162* gh = reinterpret_cast<const __nv_bfloat162*>(&gw);
        const float2 g01 = __bfloat1622float2(gh[0]), g23 = __bfloat1622float2(gh[1]);
        const float4 x = v[k];
        xs4[i] = make_float4(__bfloat162float(__float2bfloat16_rn(x.x * inv * g01.x)),
                             __bfloat162float(__float2bfloat16_rn(x.y * inv * g01.y)),
                             __bfloat162float(__float2bfloat16_rn(x.z * inv * g23.x)),
                             __bfloat162float(__float2bfloat16_rn(x.w * inv * g23.y)));
      }
    }
  } else {
    const uint4* x8 = reinterpret_cast<const uint4*>(xin);
    const int n8 = K >> 3;
    for (int base = 0; base < n8; base += 8 * NT) {  // rounds of 8 loads per thread
    uint4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int i = base + threadIdx.x + k * NT;
      if (i < n8) v[k] = x8[i];
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int i = base + threadIdx.x + k * NT;
      if (i < n8) {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v[k]);
        float4* d = reinterpret_cast<float4*>(xs + 8 * i);
        const float2 a = __bfloat1622float2(h[0]), b = __bfloat1622float2(h[1]);
        const float2 c = __bfloat1622float2(h[2]), e = __bfloat1622float2(h[3]);
        d[0] = make_float4(a.x, a.y, b.x, b.y);
        d[1] = make_float4(c.x, c.y, e.x, e.y);
      }
    }
    }
  }
  __syncthreads();
}

// Two weight rows against xs (fp32 in shared memory): 16-B loads in batches
// of 4 per row per lane, the next batch issued before the current one is
// consumed (16 loads in flight per lane), fp32 accumulation.  `ca`/`cb` hold
// the first batch (loaded by the caller, possibly before the PDL wait).
__device__ __forceinline__ void load_batch(const uint4* r0, const uint4* r1, int i, int n,
                                           uint4 (&a)[4], uint4 (&b)[4]) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int j = i + 32 * k;
    if (j < n) {
      a[k] = __ldcs(r0 + j);
      b[k] = __ldcs(r1 + j);
    } else {
      a[k] = make_uint4(0, 0, 0, 0);
      b[k] = a[k];
    }
  }
}
__device__ __forceinline__ void fma8(const uint4& u, const float* x, float& s) {
  const float4 xa = reinterpret_cast<const float4*>(x)[0], xb = reinterpret_cast<const float4*>(x)[1];
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
  float2 f;
  f = __bfloat1622float2(h[0]); s = fmaf(f.x, xa.x, fmaf(f.y, xa.y, s));
  f = __bfloat1622float2(h[1]); s = fmaf(f.x, xa.z, fmaf(f.y, xa.w, s));
  f = __bfloat1622float2(h[2]); s = fmaf(f.x, xb.x, fmaf(f.y, xb.y, s));
  f = __bfloat1622float2(h[3]); s = fmaf(f.x, xb.z, fmaf(f.y, xb.w, s));
}
// nx0/nx1 (nullable): the next pair's rows — their first batch is issued in
// place of this pair's (empty) batch past the end, so the stream never drains
// xs1 (nullable): row w1's input (the second K half of a split row), else xs
__device__ __forceinline__ void dot2(const bf16* __restrict__ w0, const bf16* __restrict__ w1,
                                     const float* xs, int K, uint4 (&ca)[4], uint4 (&cb)[4],
                                     float& a0, float& a1, const bf16* nx0 = nullptr,
                                     const bf16* nx1 = nullptr, const float* xs1 = nullptr) {
  if (!xs1) xs1 = xs;
  const int lane = threadIdx.x & 31;
  const uint4* r0 = reinterpret_cast<const uint4*>(w0);
  const uint4* r1 = reinterpret_cast<const uint4*>(w1);
  const int n = K >> 3;
  float s0 = 0.f, s1 = 0.f;
  for (int i = lane; i < n; i += 128) {
    uint4 na[4], nb[4];
    if (i + 128 < n || nx0 == nullptr)
      load_batch(r0, r1, i + 128, n, na, nb);
    else
      load_batch(reinterpret_cast<const uint4*>(nx0), reinterpret_cast<const uint4*>(nx1), lane, n,
                 na, nb);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int j = i + 32 * k;
      if (j < n) {
        fma8(ca[k], xs + 8 * j, s0);
        fma8(cb[k], xs1 + 8 * j, s1);
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      ca[k] = na[k];
      cb[k] = nb[k];
    }
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

// same, with this lane's T values in registers (t0 = T[lane], t1 = T[lane + 32])
__device__ __forceinline__ float lora_row_r(const bf16* B, int row, int r, float t0, float t1) {
  if (!B) return 0.f;
  const int lane = threadIdx.x & 31;
  float s = 0.f;
  if (lane < r) s = __bfloat162float(B[(size_t)row * r + lane]) * t0;
  if (lane + 32 < r) s = fmaf(__bfloat162float(B[(size_t)row * r + lane + 32]), t1, s);
  return warp_sum(s);
}

__device__ __forceinline__ int ld_acquire_i32(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
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

// ---------------- GEMV family ----------------
// Row pairs per warp.  QKV: q/k pairs are RoPE partners (h*hd + i, h*hd + i +
// hd/2), v pairs are adjacent rows; GU: (gate i, up i); RESID: adjacent rows.
template <int MODE>
__device__ __forceinline__ void pair_rows(const DecGemv& p, int pr, const bf16*& w0,
                                          const bf16*& w1, int& seg, int& r0, int& r1) {
  if (MODE == DEC_QKV) {
    const int half = p.hd >> 1;
    const int nqp = p.nq >> 1, nkp = p.nkv >> 1;
    if (pr < nqp + nkp) {
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
    w0 = p.W[seg] + (size_t)r0 * p.K;
    w1 = p.W[seg] + (size_t)r1 * p.K;
  } else if (MODE == DEC_GU) {
    seg = 0;
    r0 = r1 = pr;
    w0 = p.W[0] + (size_t)pr * p.K;
    w1 = p.W[1] + (size_t)pr * p.K;
  } else if (p.split) {  // one row, its two K halves (summed in the epilogue)
    seg = 0;
    r0 = r1 = pr;
    w0 = p.W[0] + (size_t)pr * p.K;
    w1 = w0 + (p.K >> 1);
  } else {
    seg = 0;
    r0 = 2 * pr;
    r1 = r0 + 1 < p.N ? r0 + 1 : r0;
    w0 = p.W[0] + (size_t)r0 * p.K;
    w1 = p.W[0] + (size_t)r1 * p.K;
  }
}

// The LoRA shrink of this GEMV's input rides in the same launch: CTAs
// [0, nsh) compute T's K parts (8 rows x one part each) and count themselves
// on sh_cnt; GEMV warps stream their first weights meanwhile and wait for the
// count (monotonic over steps: nsh x step) only before their first LoRA term.
// The whole grid is co-resident (<= 2 CTAs per SM), so the wait cannot block
// a shrink CTA from being scheduled.
template <int MODE>
__global__ void __launch_bounds__(DT) dec_gemv_kernel(DecGemv p) {
  extern __shared__ float xs[];
  __shared__ float red[32];
  ptx::pdl_launch();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if ((int)blockIdx.x < p.nsh) {  // ---- LoRA shrink role ----
    const DecShrink& a = p.sh;
    const int o = (blockIdx.x / DEC_TSPLIT) * (DT / 32) + warp, part = blockIdx.x % DEC_TSPLIT;
    const int rows = a.nt * a.r, K = p.K;
    const int t = o / a.r, j = o - t * a.r;
    const int per = ((K >> 3) + DEC_TSPLIT - 1) / DEC_TSPLIT;
    const int u0 = part * per, u1 = min(K >> 3, u0 + per);
    uint4 w[4] = {};
    const uint4* Ar = o < rows ? reinterpret_cast<const uint4*>(a.A[t] + (size_t)j * K) : nullptr;
    if (Ar) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (u0 + lane + 32 * k < u1) w[k] = __ldcs(Ar + u0 + lane + 32 * k);
    }
    ptx::pdl_wait();
    load_input(xs, p.X, p.g, p.xin, K, p.eps, red);
    if (Ar) {
      float sacc = 0.f;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (u0 + lane + 32 * k < u1) fma8(w[k], xs + 8 * (u0 + lane + 32 * k), sacc);
      for (int i = u0 + lane + 128; i < u1; i += 32) fma8(__ldcs(Ar + i), xs + 8 * i, sacc);
      sacc = warp_sum(sacc);
      if (lane == 0) a.T[t][(size_t)part * DEC_TSTRIDE + j] = sacc * p.sh_scale;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(p.sh_cnt, 1);
    return;
  }
  const int stride = (gridDim.x - p.nsh) * (DT / 32);
  int pr = (blockIdx.x - p.nsh) * (DT / 32) + warp;
  // the first pair's first batch of weights streams in while the previous
  // kernel finishes (weights are read-only during the step)
  uint4 ca[4], cb[4];
  const bf16 *w0 = nullptr, *w1 = nullptr;
  int seg = 0, r0 = 0, r1 = 0;
  const int kd = MODE == DEC_RESID && p.split ? p.K >> 1 : p.K;  // dot length per "row"
  if (pr < p.npairs) {
    pair_rows<MODE>(p, pr, w0, w1, seg, r0, r1);
    load_batch(reinterpret_cast<const uint4*>(w0), reinterpret_cast<const uint4*>(w1), lane,
               kd >> 3, ca, cb);
  }
  ptx::pdl_wait();
  load_input(xs, p.X, p.g, p.xin, p.K, p.eps, red);
  // this lane's LoRA T values (j = lane, lane + 32) per segment, loaded once
  float tv[3][2] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
  bool t_ready = p.nsh == 0;
  auto fetch_t = [&]() {
    if (lane == 0) {
      const int want = p.nsh * p.st->step;
      uint32_t n = 0;
      while (ld_acquire_i32(p.sh_cnt) < want)
        if (++n == (1u << 30)) __trap();
    }
    __syncwarp();
    for (int t = 0; t < 3; ++t)
      if (p.T[t])
        for (int h = 0; h < 2; ++h) {
          const int j = lane + 32 * h;
          float v = 0.f;
          if (j < p.r)
            for (int q = 0; q < DEC_TSPLIT; ++q) v += __ldcg(p.T[t] + (size_t)q * DEC_TSTRIDE + j);
          tv[t][h] = v;  // part order
        }
    t_ready = true;
  };
  const int pos = p.st ? p.st->pos : 0;
  for (; pr < p.npairs; pr += stride) {
    // rows of the next pair: their first batch loads while this pair finishes
    const bf16 *n0 = nullptr, *n1 = nullptr;
    int nseg = 0, nr0 = 0, nr1 = 0;
    if (pr + stride < p.npairs) pair_rows<MODE>(p, pr + stride, n0, n1, nseg, nr0, nr1);
    float a0, a1;
    dot2(w0, w1, xs, kd, ca, cb, a0, a1, n0, n1, kd != p.K ? xs + kd : nullptr);
    if (!t_ready) fetch_t();
    if (MODE == DEC_QKV) {
      a0 += lora_row_r(p.B[seg], r0, p.r, tv[seg][0], tv[seg][1]);
      a1 += lora_row_r(p.B[seg], r1, p.r, tv[seg][0], tv[seg][1]);
      if (lane == 0) {
        if (seg < 2) {  // rotate-half RoPE at this token's position
          const int half = p.hd >> 1;
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
      const float gt = a0 + lora_row_r(p.B[0], pr, p.r, tv[0][0], tv[0][1]);
      const float up = a1 + lora_row_r(p.B[1], pr, p.r, tv[1][0], tv[1][1]);
      if (lane == 0) p.h[pr] = __float2bfloat16_rn(gt / (1.f + __expf(-gt)) * up);
    } else if (p.split) {  // DEC_RESID, split row: X[row] += (half0 + half1) + LoRA
      const float lr = lora_row_r(p.B[0], r0, p.r, tv[0][0], tv[0][1]);
      if (lane == 0) p.Xout[r0] += (a0 + a1) + lr;
    } else {  // DEC_RESID: X[row] += W[row] . x
      a0 += lora_row_r(p.B[0], r0, p.r, tv[0][0], tv[0][1]);
      a1 += lora_row_r(p.B[0], r1, p.r, tv[0][0], tv[0][1]);
      if (lane == 0) {
        p.Xout[r0] += a0;
        if (r1 != r0) p.Xout[r1] += a1;
      }
    }
    w0 = n0;
    w1 = n1;
    seg = nseg;
    r0 = nr0;
    r1 = nr1;
  }
}

// ---------------- attention over the cache (one query token) ----------------
// CTA = (head, 128-key chunk), 128 threads: thread = key for the scores, lane =
// hd/32 dims for PV; each chunk leaves (max, sum, o[hd]) and the last chunk of
// a head to finish folds all chunks in chunk order (deterministic) into the
// bf16 attention output, then re-arms the head's counter.
constexpr int ACH = 128, ATH = 128;
__global__ void __launch_bounds__(ATH) dec_attn_kernel(DecAttn a) {
  __shared__ float qs[128];
  __shared__ float ps[ACH];
  __shared__ float red[ATH / 32];
  __shared__ float os[ATH / 32][128];
  __shared__ int last;
  ptx::pdl_launch();
  ptx::pdl_wait();
  const int h = blockIdx.x, c = blockIdx.y;
  const int g = h / (a.H / a.KV);
  const int nkeys = a.st->pos + 1;
  const int k0 = c * ACH, k1 = min(nkeys, k0 + ACH);
  if (k0 >= k1) return;  // past the current position: not part of this step
  const int nchunks = (nkeys + ACH - 1) / ACH;
  float* part = a.part + ((size_t)h * gridDim.y + c) * (2 + 128);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < a.hd; i += ATH) qs[i] = __bfloat162float(a.q[h * a.hd + i]) * a.scale_log2;
  __syncthreads();
  float s = -INFINITY;
  const int k = k0 + threadIdx.x;
  if (k < k1) {
    const uint4* kr = reinterpret_cast<const uint4*>(a.kc + (size_t)k * a.ldkv + g * a.hd);
    uint4 u[16];
    const int nu = a.hd >> 3;
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (i < nu) u[i] = kr[i];
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (i < nu) fma8(u[i], qs + 8 * i, acc);
    s = acc;  // log2 domain (q pre-scaled)
  }
  float m = warp_max(s);
  if (lane == 0) red[warp] = m;
  __syncthreads();
  m = red[0];
  for (int w = 1; w < ATH / 32; ++w) m = fmaxf(m, red[w]);
  const float pk = k < k1 ? ptx::ex2(s - m) : 0.f;
  ps[threadIdx.x] = pk;
  const float lw = warp_sum(pk);
  __syncthreads();  // every thread read red (max) and wrote ps
  if (lane == 0) red[warp] = lw;
  // PV: warp w takes keys w, w+4, ...; lane owns dims dpl*lane .. (hd = 32 dpl)
  const int dpl = a.hd >> 5;  // 2 or 4
  float o[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 8
  for (int kk = warp; kk < k1 - k0; kk += ATH / 32) {
    const float pv = ps[kk];
    const bf16* vr = a.vc + (size_t)(k0 + kk) * a.ldkv + g * a.hd + dpl * lane;
    if (dpl == 4) {
      const uint2 uu = *reinterpret_cast<const uint2*>(vr);
      const __nv_bfloat162* hh = reinterpret_cast<const __nv_bfloat162*>(&uu);
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
    for (int w = 0; w < ATH / 32; ++w) acc += os[w][threadIdx.x];  // fixed order
    part[2 + threadIdx.x] = acc;
  }
  if (threadIdx.x == 0) {
    float lt = 0.f;
    for (int w = 0; w < ATH / 32; ++w) lt += red[w];
    part[0] = m;
    part[1] = lt;
  }
  // ---- the last chunk of this head combines ----
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(a.cnt + h, 1) == nchunks - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  // chunk statistics in parallel (thread = chunk), then every output dim folds
  // the chunks in chunk order with its loads batched
  const float* hp = a.part + (size_t)h * gridDim.y * (2 + 128);
  float* cw = ps;  // reuse: per-chunk weight 2^(m_c - max) and sums
  float* cl = qs;
  if (threadIdx.x < nchunks) {
    cw[threadIdx.x] = __ldcg(hp + threadIdx.x * 130);
    cl[threadIdx.x] = __ldcg(hp + threadIdx.x * 130 + 1);
  }
  __syncthreads();
  float mx = -INFINITY;
  for (int cc = 0; cc < nchunks; ++cc) mx = fmaxf(mx, cw[cc]);
  __syncthreads();
  if (threadIdx.x < nchunks) cw[threadIdx.x] = ptx::ex2(cw[threadIdx.x] - mx);
  __syncthreads();
  float l = 0.f;
  for (int cc = 0; cc < nchunks; ++cc) l = fmaf(cw[cc], cl[cc], l);  // chunk order
  const int i = threadIdx.x;
  float ov = 0.f;
  if (i < a.hd) {
#pragma unroll 8
    for (int cc = 0; cc < nchunks; ++cc) ov = fmaf(cw[cc], __ldcg(hp + cc * 130 + 2 + i), ov);
    a.out[h * a.hd + i] = __float2bfloat16_rn(ov / l);
  }
  if (i == 0) a.cnt[h] = 0;
}

__global__ void dec_save_logits_kernel(const DecodeState* st, const float* logits, float* all, int V) {
  ptx::pdl_begin();
  float* dst = all + (size_t)(st->step - 1) * V;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < V; i += gridDim.x * blockDim.x)
    dst[i] = logits[i];
}

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

cudaError_t dec_gemv_launch(const DecGemv& p0, int mode, int num_sms, cudaStream_t s) {
  // residual GEMVs (N = d rows): split every row into its two K halves so
  // twice as many warps stream (N / 2 row pairs leave half of them idle);
  // TIDAL_DEC_SPLIT=0 keeps row pairs
  static const bool split_off = [] {
    const char* e = getenv("TIDAL_DEC_SPLIT");
    return e && e[0] == '0';
  }();
  DecGemv p = p0;
  p.split = 0;
  if (mode == DEC_RESID && !split_off && p.K % 16 == 0) {
    p.split = 1;
    p.npairs = p.N;
  }
  static bool attr[3] = {false, false, false};
  auto k = mode == DEC_QKV ? dec_gemv_kernel<DEC_QKV>
                           : (mode == DEC_GU ? dec_gemv_kernel<DEC_GU> : dec_gemv_kernel<DEC_RESID>);
  if (!attr[mode]) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    if (e != cudaSuccess) return e;
    attr[mode] = true;
  }
  // every warp gets the same number of row pairs: as many CTAs as fit at
  // once (<= 4 per SM, shared-memory limited for long inputs), the pairs
  // spread evenly over their warps
  const int per_sm = 2;  // ~125 registers x 256 threads: two CTAs per SM (a 3-CTA bound spills)
  const int cap = num_sms * per_sm;  // co-resident CTAs (the shrink wait needs them all)
  const int g_max = cap - p.nsh;
  if (g_max < 1) return cudaErrorInvalidConfiguration;
  // every warp the same number of row pairs (measured equal or better than
  // filling all co-resident CTAs with some warps one pair longer)
  int iters = (p.npairs + g_max * (DT / 32) - 1) / (g_max * (DT / 32));
  iters = iters < 1 ? 1 : iters;
  const int grid = (p.npairs + iters * (DT / 32) - 1) / (iters * (DT / 32));
  return launch_k(k, dim3(p.nsh + grid), dim3(DT), (size_t)p.K * 4, s, 1, p);
}

cudaError_t dec_attn_launch(const DecAttn& a, int max_keys, cudaStream_t s) {
  const int nchunks = (max_keys + ACH - 1) / ACH;
  return launch_k(dec_attn_kernel, dim3(a.H, nchunks), dim3(ATH), 0, s, 1, a);
}

}  // namespace tidal
