// attention.cu — causal GQA prefill attention (first cut: FlashAttention-2
// style on legacy mma.sync m16n8k16).
//   O_h = softmax(Q_h K_g^T / sqrt(hd) + causal) V_g,   g = h / (H / KV)
// CTA = 64 queries of one head, 4 warps x 16 query rows; K/V tiles of 64 keys
// staged by a 2-stage cp.async ring into XOR-swizzled shared memory; online
// softmax (exp2, fp32 running max/sum, quad shuffles); P rounded to bf16 for
// the PV product, normalised at the end.  Heavy (late) query tiles first.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"
#include "launch.cuh"

namespace tidal {
namespace {

constexpr int BQ = 64, BKV = 64, NTH = 128;

__device__ __forceinline__ void cp_async16(uint32_t s, const void* g, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(g),
               "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], uint32_t s) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(s));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], uint32_t s) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(s));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// element offset of (row, col) in a [rows][HD] tile with 16-B chunks XOR-swizzled by row
template <int HD>
__device__ __forceinline__ int swz(int row, int col) {
  return row * HD + ((((col >> 3) ^ (row & 7))) << 3) + (col & 7);
}

template <int HD>
__global__ void __launch_bounds__(NTH, 2) attn_kernel(const bf16* __restrict__ qkv, bf16* __restrict__ O,
                                                      int S, int H, int KV, float scale_log2) {
  extern __shared__ __align__(128) uint8_t sm[];
  bf16* qs = reinterpret_cast<bf16*>(sm);
  bf16* ks = qs + BQ * HD;          // [2][BKV * HD]
  bf16* vs = ks + 2 * BKV * HD;     // [2][BKV * HD]
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL: previous kernel complete
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int nq = (S + BQ - 1) / BQ;
  const int qt = nq - 1 - blockIdx.x;
  const int h = blockIdx.y;
  const int g = h / (H / KV);
  const int ld = (H + 2 * KV) * HD;
  qkv += (size_t)blockIdx.z * S * ld;  // sequence blockIdx.z of a batch (rows z*S .. z*S+S-1)
  O += (size_t)blockIdx.z * S * (H * HD);
  const int q0 = qt * BQ;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bf16* Qg = qkv + (size_t)h * HD;
  const bf16* Kg = qkv + (size_t)(H + g) * HD;
  const bf16* Vg = qkv + (size_t)(H + KV + g) * HD;
  constexpr int CH = HD / 8;  // 16-B chunks per row

  const uint32_t qs_s = (uint32_t)__cvta_generic_to_shared(qs);
  const uint32_t ks_s = (uint32_t)__cvta_generic_to_shared(ks);
  const uint32_t vs_s = (uint32_t)__cvta_generic_to_shared(vs);

  // Q tile
  for (int c = threadIdx.x; c < BQ * CH; c += NTH) {
    const int r = c / CH, ch = c % CH;
    const int s = q0 + r;
    const bool ok = s < S;
    cp_async16(qs_s + 2 * swz<HD>(r, ch * 8), ok ? Qg + (size_t)s * ld + ch * 8 : Qg, ok);
  }
  auto load_kv = [&](int j, int buf) {
    const int k0 = j * BKV;
    for (int c = threadIdx.x; c < BKV * CH; c += NTH) {
      const int r = c / CH, ch = c % CH;
      const int s = k0 + r;
      const bool ok = s < S;
      const uint32_t off = 2 * (buf * BKV * HD + swz<HD>(r, ch * 8));
      cp_async16(ks_s + off, ok ? Kg + (size_t)s * ld + ch * 8 : Kg, ok);
      cp_async16(vs_s + off, ok ? Vg + (size_t)s * ld + ch * 8 : Vg, ok);
    }
  };
  load_kv(0, 0);
  cp_commit();

  const int nkv = min((q0 + BQ + BKV - 1) / BKV, (S + BKV - 1) / BKV);
  uint32_t qf[HD / 16][4];
  float o[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
  const int qrow0 = q0 + warp * 16 + (lane >> 2);  // this thread's rows: qrow0, qrow0 + 8

  for (int j = 0; j < nkv; ++j) {
    const int buf = j & 1;
    if (j + 1 < nkv) {
      load_kv(j + 1, buf ^ 1);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    if (j == 0) {
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        const int r = warp * 16 + (lane & 15), c = kk * 16 + (lane >> 4) * 8;
        ldsm_x4(qf[kk], qs_s + 2 * swz<HD>(r, c));
      }
    }
    const uint32_t kb = ks_s + 2 * buf * BKV * HD;
    const uint32_t vb = vs_s + 2 * buf * BKV * HD;
    // S = Q K^T   (16 x 64 per warp)
    float s[BKV / 8][4];
#pragma unroll
    for (int nt = 0; nt < BKV / 8; ++nt) s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < HD / 16; kk += 2) {
#pragma unroll
      for (int nt = 0; nt < BKV / 8; ++nt) {
        uint32_t b[4];
        const int r = nt * 8 + (lane & 7), c = kk * 16 + (lane >> 3) * 8;
        ldsm_x4(b, kb + 2 * swz<HD>(r, c));
        mma16816(s[nt], qf[kk], b[0], b[1]);
        mma16816(s[nt], qf[kk + 1], b[2], b[3]);
      }
    }
    // scale (log2 domain) + causal mask
    const bool diag = (j + 1) * BKV > q0;
#pragma unroll
    for (int nt = 0; nt < BKV / 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float v = s[nt][e] * scale_log2;
        if (diag) {
          const int key = j * BKV + nt * 8 + 2 * (lane & 3) + (e & 1);
          const int qi = qrow0 + (e >> 1) * 8;
          if (key > qi) v = -INFINITY;
        }
        s[nt][e] = v;
      }
    }
    // online softmax
    float mnew[2], corr[2];
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      float mx = mrow[hh];
#pragma unroll
      for (int nt = 0; nt < BKV / 8; ++nt) mx = fmaxf(mx, fmaxf(s[nt][2 * hh], s[nt][2 * hh + 1]));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      mnew[hh] = mx;
      corr[hh] = exp2f(mrow[hh] - mx);
      mrow[hh] = mx;
    }
    float lsum[2] = {0.f, 0.f};
    uint32_t pf[BKV / 16][4];
#pragma unroll
    for (int nt = 0; nt < BKV / 8; ++nt) {
      const float p0 = exp2f(s[nt][0] - mnew[0]);
      const float p1 = exp2f(s[nt][1] - mnew[0]);
      const float p2 = exp2f(s[nt][2] - mnew[1]);
      const float p3 = exp2f(s[nt][3] - mnew[1]);
      lsum[0] += p0 + p1;
      lsum[1] += p2 + p3;
      const int kk = nt >> 1, hi = nt & 1;
      pf[kk][hi * 2 + 0] = pack2(p0, p1);
      pf[kk][hi * 2 + 1] = pack2(p2, p3);
    }
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      float t = lsum[hh];
      t += __shfl_xor_sync(0xffffffffu, t, 1);
      t += __shfl_xor_sync(0xffffffffu, t, 2);
      lrow[hh] = lrow[hh] * corr[hh] + t;
    }
#pragma unroll
    for (int dt = 0; dt < HD / 8; ++dt) {
      o[dt][0] *= corr[0];
      o[dt][1] *= corr[0];
      o[dt][2] *= corr[1];
      o[dt][3] *= corr[1];
    }
    // O += P V
#pragma unroll
    for (int kk = 0; kk < BKV / 16; ++kk) {
#pragma unroll
      for (int dt = 0; dt < HD / 8; dt += 2) {
        uint32_t b[4];
        const int r = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int c = dt * 8 + (lane >> 4) * 8;
        ldsm_x4_t(b, vb + 2 * swz<HD>(r, c));
        mma16816(o[dt], pf[kk], b[0], b[1]);
        mma16816(o[dt + 1], pf[kk], b[2], b[3]);
      }
    }
    __syncthreads();
  }
  // normalise and store
  const float inv0 = 1.f / lrow[0], inv1 = 1.f / lrow[1];
  bf16* Oh = O + (size_t)h * HD;
  const int ldo = H * HD;
#pragma unroll
  for (int dt = 0; dt < HD / 8; ++dt) {
    const int c = dt * 8 + 2 * (lane & 3);
    if (qrow0 < S)
      *reinterpret_cast<uint32_t*>(Oh + (size_t)qrow0 * ldo + c) = pack2(o[dt][0] * inv0, o[dt][1] * inv0);
    if (qrow0 + 8 < S)
      *reinterpret_cast<uint32_t*>(Oh + (size_t)(qrow0 + 8) * ldo + c) =
          pack2(o[dt][2] * inv1, o[dt][3] * inv1);
  }
}

template <int HD>
cudaError_t launch(const bf16* qkv, bf16* O, int S, int H, int KV, cudaStream_t s, int nseq) {
  const int smem = (BQ + 4 * BKV) * HD * 2;
  static bool attr = false;
  if (!attr) {
    cudaError_t e =
        cudaFuncSetAttribute(attn_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid((S + BQ - 1) / BQ, H, nseq);
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)HD);
  return launch_k(attn_kernel<HD>, grid, dim3(NTH), smem, s, 1, qkv, O, S, H, KV, scale_log2);
}

}  // namespace

cudaError_t attention_launch(const bf16* qkv, bf16* O, int S, int H, int KV, int hd,
                             cudaStream_t s, int nseq) {
  if (nseq < 1 || nseq > 65535) return cudaErrorInvalidValue;
  if (hd == 128) return launch<128>(qkv, O, S, H, KV, s, nseq);
  if (hd == 64) return launch<64>(qkv, O, S, H, KV, s, nseq);
  return cudaErrorInvalidValue;
}

}  // namespace tidal
