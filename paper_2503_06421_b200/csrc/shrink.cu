// shrink.cu — LoRA shrink T_t = scale * X A_t^T for the targets that share X
// (q,k,v share Xn; gate,up share Xn; o reads O; down reads H).
// A skinny product (r <= 64 per target, <= 3 targets): its cost is one read
// of X [M, K], so the kernel reads X ONCE for all targets and splits K across
// CTAs to put ~4 CTAs on every SM.  Each CTA (64 rows x K/ksplit) accumulates
// with mma.sync m16n8k16 from a 2-stage cp.async ring, writes an fp32 partial
// to a workspace, and the last CTA of each row tile (atomic ticket) reduces
// the partials in a fixed order (deterministic) and stores bf16 T.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"

namespace tidal {
namespace {

constexpr int BM = 64, BK = 32, LD = 40, NTH = 128;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem),
               "r"(valid ? 16 : 0)
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

struct Args {
  const bf16* A[3];
  bf16* T[3];
};

template <int R>
__global__ void __launch_bounds__(NTH) shrink_kernel(const bf16* __restrict__ X, int ldx, int M,
                                                     int K, Args args, int nt, float scale,
                                                     int kchunk, float* __restrict__ ws,
                                                     unsigned int* __restrict__ tickets) {
  extern __shared__ __align__(16) bf16 sm[];
  bf16* xs = sm;                           // [2][BM*LD]
  bf16* as = sm + 2 * BM * LD;             // [2][3*R*LD]
  const int RT = nt * R;
  const int m0 = blockIdx.x * BM;
  const int ks = blockIdx.y, nks = gridDim.y;
  const int kbeg = ks * kchunk, kend = min(K, kbeg + kchunk);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float acc[3][R / 8][4];
#pragma unroll
  for (int t = 0; t < 3; ++t)
#pragma unroll
    for (int i = 0; i < R / 8; ++i) acc[t][i][0] = acc[t][i][1] = acc[t][i][2] = acc[t][i][3] = 0.f;
  const int nk = (kend - kbeg + BK - 1) / BK;
  auto load = [&](int kb, int buf) {
    const int k0 = kbeg + kb * BK;
    for (int c = threadIdx.x; c < BM * 4; c += NTH) {
      const int r = c >> 2, ch = c & 3;
      const int m = m0 + r, k = k0 + ch * 8;
      const bool ok = m < M && k < kend;
      cp_async16(xs + buf * BM * LD + r * LD + ch * 8, ok ? X + (size_t)m * ldx + k : X, ok);
    }
    for (int c = threadIdx.x; c < RT * 4; c += NTH) {
      const int r = c >> 2, ch = c & 3;
      const int t = r / R, rr = r - t * R;
      const int k = k0 + ch * 8;
      const bool ok = k < kend;
      const bf16* A = args.A[t];
      cp_async16(as + buf * 3 * R * LD + r * LD + ch * 8, ok ? A + (size_t)rr * K + k : A, ok);
    }
    cp_commit();
  };
  if (nk > 0) load(0, 0);
  for (int kb = 0; kb < nk; ++kb) {
    const int buf = kb & 1;
    if (kb + 1 < nk) {
      load(kb + 1, buf ^ 1);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const bf16* xb = xs + buf * BM * LD;
    const bf16* ab = as + buf * 3 * R * LD;
#pragma unroll
    for (int kk = 0; kk < BK / 16; ++kk) {
      uint32_t a[4];
      ldsm_x4(a, xb + (warp * 16 + (lane & 15)) * LD + kk * 16 + (lane >> 4) * 8);
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        if (t >= nt) break;
#pragma unroll
        for (int n = 0; n < R / 8; ++n) {
          uint32_t b[2];
          ldsm_x2(b, ab + (t * R + n * 8 + (lane & 7)) * LD + kk * 16 + ((lane >> 3) & 1) * 8);
          mma16816(acc[t][n], a, b);
        }
      }
    }
    __syncthreads();
  }
  // fp32 partial -> workspace [nks][M][RT]
  const int r0 = m0 + warp * 16 + (lane >> 2);
  float* w = ws + (size_t)ks * M * RT;
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    if (t >= nt) break;
#pragma unroll
    for (int n = 0; n < R / 8; ++n) {
      const int c = t * R + n * 8 + 2 * (lane & 3);
      if (r0 < M) *reinterpret_cast<float2*>(w + (size_t)r0 * RT + c) = make_float2(acc[t][n][0], acc[t][n][1]);
      if (r0 + 8 < M)
        *reinterpret_cast<float2*>(w + (size_t)(r0 + 8) * RT + c) = make_float2(acc[t][n][2], acc[t][n][3]);
    }
  }
  __threadfence();
  __syncthreads();
  __shared__ unsigned int last;
  if (threadIdx.x == 0) last = atomicAdd(&tickets[blockIdx.x], 1u) == (unsigned)(nks - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int rows = min(BM, M - m0);
  for (int e = threadIdx.x; e < rows * RT; e += NTH) {
    const int rr = e / RT, c = e - rr * RT;
    const size_t off = (size_t)(m0 + rr) * RT + c;
    float s = 0.f;
    for (int k = 0; k < nks; ++k) s += __ldcg(ws + (size_t)k * M * RT + off);
    const int t = c / R;
    args.T[t][(size_t)(m0 + rr) * R + (c - t * R)] = __float2bfloat16_rn(s * scale);
  }
  if (threadIdx.x == 0) tickets[blockIdx.x] = 0;  // self-cleaning for the next launch
}

template <int R>
cudaError_t launch(const bf16* X, int ldx, int M, int K, const Args& a, int nt, float scale,
                   int ksplit, float* ws, unsigned int* tickets, cudaStream_t s) {
  const int smem = (2 * BM * LD + 2 * 3 * R * LD) * 2;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(shrink_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  int kchunk = (K + ksplit - 1) / ksplit;
  kchunk = (kchunk + BK - 1) / BK * BK;
  const int nks = (K + kchunk - 1) / kchunk;
  dim3 grid((M + BM - 1) / BM, nks);
  shrink_kernel<R><<<grid, NTH, smem, s>>>(X, ldx, M, K, a, nt, scale, kchunk, ws, tickets);
  return cudaGetLastError();
}

}  // namespace

int shrink_ksplit(int M, int K, int num_sms) {
  const int mt = (M + BM - 1) / BM;
  int ks = (4 * num_sms + mt - 1) / mt;
  const int kmax = (K + 255) / 256;   // at least 256 K per CTA
  if (ks > kmax) ks = kmax;
  if (ks > SHRINK_MAX_KSPLIT) ks = SHRINK_MAX_KSPLIT;
  return ks < 1 ? 1 : ks;
}

cudaError_t lora_shrink_launch(const bf16* X, int ldx, int M, int K, const bf16* const* A,
                               bf16* const* T, int nt, int r, float scale, int num_sms,
                               float* ws, unsigned int* tickets, cudaStream_t s) {
  if (nt < 1 || nt > 3) return cudaErrorInvalidValue;
  Args a{};
  for (int i = 0; i < nt; ++i) {
    a.A[i] = A[i];
    a.T[i] = T[i];
  }
  const int ks = shrink_ksplit(M, K, num_sms);
  switch (r) {
    case 8: return launch<8>(X, ldx, M, K, a, nt, scale, ks, ws, tickets, s);
    case 16: return launch<16>(X, ldx, M, K, a, nt, scale, ks, ws, tickets, s);
    case 32: return launch<32>(X, ldx, M, K, a, nt, scale, ks, ws, tickets, s);
    case 64: return launch<64>(X, ldx, M, K, a, nt, scale, ks, ws, tickets, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace tidal
