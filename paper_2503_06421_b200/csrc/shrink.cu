// shrink.cu — LoRA shrink T_t = scale * X A_t^T for the targets that share X
// (q,k,v share Xn; gate,up share Xn; o reads O; down reads H).
// A skinny product (r <= 64 per target, <= 3 targets) whose cost is moving X
// (once, from HBM) and A (from L2, once per CTA), so it is latency-bound unless
// enough bytes are in flight: CTA = 16 rows x all targets, its warps each own
// a K slice (intra-CTA split-K) and stream X/A tiles of 64 K-columns through a
// private STG-deep cp.async ring (~100+ KB in flight per SM), mma.sync
// m16n8k16 accumulates, and the per-warp partials are summed through shared
// memory in a fixed order (deterministic) and stored as bf16.  One launch, no
// workspace, ceil(M/16) CTAs.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"

namespace tidal {
namespace {

constexpr int BM = 16, BK = 64, LD = BK + 8;  // smem row stride (elements): conflict-free ldmatrix

template <int R>
struct Cfg {
  static constexpr int NW = R >= 64 ? 2 : 4;               // warps (K slices) per CTA
  static constexpr int STG = R >= 32 ? 3 : (R >= 16 ? 4 : 6);  // ring depth per warp
};

__device__ __forceinline__ void cp_async16(uint32_t s, const void* gmem, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem),
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
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

struct Args {
  const bf16* A[3];
  bf16* T[3];
};

template <int R>
__global__ void __launch_bounds__(Cfg<R>::NW * 32) shrink_kernel(const bf16* __restrict__ X,
                                                                 int ldx, int M, int K, Args args,
                                                                 int nt, float scale, int kslice) {
  constexpr int NW = Cfg<R>::NW, STG = Cfg<R>::STG, NTH = NW * 32;
  extern __shared__ __align__(16) uint8_t sm[];
  const int RT = nt * R;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * BM;
  const int stage_bytes = (BM + RT) * LD * 2;
  const uint32_t wbase = (uint32_t)__cvta_generic_to_shared(sm) + warp * STG * stage_bytes;
  const int kbeg = warp * kslice, kend = min(K, kbeg + kslice);
  const int nk = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;
  float acc[3][R / 8][4];
#pragma unroll
  for (int t = 0; t < 3; ++t)
#pragma unroll
    for (int i = 0; i < R / 8; ++i) acc[t][i][0] = acc[t][i][1] = acc[t][i][2] = acc[t][i][3] = 0.f;
  auto load = [&](int kb) {
    if (kb < nk) {
      const int k0 = kbeg + kb * BK;
      const uint32_t sb = wbase + (kb % STG) * stage_bytes;
      for (int c = lane; c < (BM + RT) * 8; c += 32) {
        const int r = c >> 3, ch = c & 7;
        const int k = k0 + ch * 8;
        const uint32_t dst = sb + (r * LD + ch * 8) * 2;
        if (r < BM) {
          const int m = m0 + r;
          const bool ok = m < M && k < kend;
          cp_async16(dst, ok ? X + (size_t)m * ldx + k : X, ok);
        } else {
          const int ra = r - BM, t = ra / R, rr = ra - t * R;
          const bool ok = k < kend;
          const bf16* A = args.A[t];
          cp_async16(dst, ok ? A + (size_t)rr * K + k : A, ok);
        }
      }
    }
    cp_commit();  // always commit: uniform group accounting
  };
#pragma unroll
  for (int s = 0; s < STG - 1; ++s) load(s);
  for (int kb = 0; kb < nk; ++kb) {
    load(kb + STG - 1);
    cp_wait<STG - 1>();
    __syncwarp();
    const uint32_t sb = wbase + (kb % STG) * stage_bytes;
#pragma unroll
    for (int kk = 0; kk < BK / 16; ++kk) {
      uint32_t a[4];
      ldsm_x4(a, sb + ((lane & 15) * LD + kk * 16 + (lane >> 4) * 8) * 2);
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        if (t >= nt) break;
#pragma unroll
        for (int n = 0; n < R / 8; n += 2) {
          if (R == 8) {
            uint32_t b[4];
            // x4 over one 8-row n-tile: k lo/hi for this kk (matrices 2,3 unused)
            ldsm_x4(b, sb + ((BM + t * R + (lane & 7)) * LD + kk * 16 + ((lane >> 3) & 1) * 8) * 2);
            mma16816(acc[t][0], a, b[0], b[1]);
          } else {
            uint32_t b[4];
            // x4: n-tiles n and n+1, k lo/hi
            ldsm_x4(b, sb + ((BM + t * R + n * 8 + (lane & 7) + ((lane >> 4) << 3)) * LD + kk * 16 +
                             ((lane >> 3) & 1) * 8) * 2);
            mma16816(acc[t][n], a, b[0], b[1]);
            mma16816(acc[t][n + 1], a, b[2], b[3]);
          }
        }
      }
    }
    __syncwarp();
  }
  cp_wait<0>();
  // cross-warp reduction through shared memory (reuses the rings)
  __syncthreads();
  float* red = reinterpret_cast<float*>(sm);  // [NW][BM][RT]
  const int r0 = lane >> 2;
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    if (t >= nt) break;
#pragma unroll
    for (int n = 0; n < R / 8; ++n) {
      const int c = t * R + n * 8 + 2 * (lane & 3);
      float* p = red + (size_t)warp * BM * RT;
      p[r0 * RT + c] = acc[t][n][0];
      p[r0 * RT + c + 1] = acc[t][n][1];
      p[(r0 + 8) * RT + c] = acc[t][n][2];
      p[(r0 + 8) * RT + c + 1] = acc[t][n][3];
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < BM * RT; e += NTH) {
    const int rr = e / RT, c = e - rr * RT;
    const int m = m0 + rr;
    if (m >= M) continue;
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) s += red[(size_t)w * BM * RT + e];
    const int t = c / R;
    args.T[t][(size_t)m * R + (c - t * R)] = __float2bfloat16_rn(s * scale);
  }
}

template <int R>
cudaError_t launch(const bf16* X, int ldx, int M, int K, const Args& a, int nt, float scale,
                   cudaStream_t s) {
  constexpr int NW = Cfg<R>::NW, STG = Cfg<R>::STG;
  static bool attr = false;
  if (!attr) {
    const int maxb = NW * STG * (BM + 3 * R) * LD * 2;
    cudaError_t e =
        cudaFuncSetAttribute(shrink_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxb);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  int kslice = (K + NW - 1) / NW;
  kslice = (kslice + BK - 1) / BK * BK;
  const int ring = NW * STG * (BM + nt * R) * LD * 2;
  const int redb = NW * BM * nt * R * 4;
  const int need = ring > redb ? ring : redb;
  shrink_kernel<R><<<(M + BM - 1) / BM, NW * 32, need, s>>>(X, ldx, M, K, a, nt, scale, kslice);
  return cudaGetLastError();
}

}  // namespace

cudaError_t lora_shrink_launch(const bf16* X, int ldx, int M, int K, const bf16* const* A,
                               bf16* const* T, int nt, int r, float scale, cudaStream_t s) {
  if (nt < 1 || nt > 3) return cudaErrorInvalidValue;
  Args a{};
  for (int i = 0; i < nt; ++i) {
    a.A[i] = A[i];
    a.T[i] = T[i];
  }
  switch (r) {
    case 8: return launch<8>(X, ldx, M, K, a, nt, scale, s);
    case 16: return launch<16>(X, ldx, M, K, a, nt, scale, s);
    case 32: return launch<32>(X, ldx, M, K, a, nt, scale, s);
    case 64: return launch<64>(X, ldx, M, K, a, nt, scale, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace tidal
