// attn_tc.cu — causal GQA prefill attention on 5th-gen tensor cores (hd = 128).
//   O_h = softmax(Q_h K_g^T / sqrt(hd) + causal) V_g,   g = h / (H / KV)
// CTA = two adjacent 128-query tiles (A = 2t, B = 2t+1) of one head, which
// share their key range; warp-specialised, ping-pong:
//   warp 0      TMA: Q_A, Q_B once, then K / V^T tiles of 64 keys (3-deep rings)
//   warp 1      tcgen05.mma, interleaving the two tiles: PV_A(j), S_A(j+1),
//               PV_B(j), S_B(j+1) — while softmax A works on S_A the tensor
//               core runs tile B's MMAs and vice versa
//   warps 2..5  softmax of tile A, warps 6..9 of tile B: one query row per
//               thread (TMEM lane = row); P = exp2(S*scale - m) rounded to bf16
//               into a SWIZZLE_128B smem tile (the A operand of PV); running
//               row sum in fp32.  O stays in TMEM; it is rescaled only when a
//               row max grows by more than 2^8 (exact: O and l share the same
//               stale max, P <= 256 cannot overflow); then O / l -> bf16.
// V is consumed as V^T [hd][S] (written transposed by the QKV GEMM epilogue),
// so both MMAs read K-major operands.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"
#include "ptx.cuh"

namespace tidal {
namespace {

constexpr int HD = 128, BQ = 128, BKV = 64, RING = 3;
constexpr int QTILE = BQ * HD * 2;      // 32 KB: [128 q][128 hd] as two 64-wide K-blocks
constexpr int QHALF = QTILE / 2;        // one K-block [128 rows][64]
constexpr int KTILE = BKV * HD * 2;     // 16 KB: [64 keys][128 hd] as two K-blocks
constexpr int KHALF = KTILE / 2;
constexpr int VTILE = HD * BKV * 2;     // 16 KB: V^T [128 hd][64 keys], one K-block
constexpr int PTILE = BQ * BKV * 2;     // 16 KB: P [128 q][64 keys], one K-block
constexpr int OFF_Q = 0;                               // Q_A, Q_B
constexpr int OFF_K = OFF_Q + 2 * QTILE;
constexpr int OFF_V = OFF_K + RING * KTILE;
constexpr int OFF_P = OFF_V + RING * VTILE;            // P_A[2], P_B[2] (double-buffered)
constexpr int OFF_BAR = OFF_P + 4 * PTILE;
constexpr int N_BARS = 1 + 4 * RING + 12;
constexpr int OFF_TMEM = OFF_BAR + N_BARS * 8;
constexpr int SMEM = OFF_TMEM + 16 + 1024;
constexpr int NTH = 320;
// TMEM columns: S_A[2], S_B[2] (64 each: S is double-buffered per tile, so
// S_x(j+1) is computed while softmax x works on S_x(j)), O_A, O_B (128 each)
constexpr uint32_t COL_S = 0, COL_O = 256;

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

__global__ void __launch_bounds__(NTH, 1) attn_tc_kernel(const __grid_constant__ AttnParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const uint32_t sb = ptx::smem_u32(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t bars = sb + OFF_BAR;
  const uint32_t q_full = bars;
  auto k_full = [&](int s) { return bars + 8u * (1 + s); };
  auto k_empty = [&](int s) { return bars + 8u * (1 + RING + s); };
  auto v_full = [&](int s) { return bars + 8u * (1 + 2 * RING + s); };
  auto v_empty = [&](int s) { return bars + 8u * (1 + 3 * RING + s); };
  auto s_full = [&](int x, int b) { return bars + 8u * (1 + 4 * RING + 2 * x + b); };
  // P-full and PV-done barriers per P buffer: softmax may run one tile ahead of
  // the MMA warp, so a single barrier could complete two phases before the
  // waiter looks (parity aliasing); per-buffer barriers cannot.
  auto p_full = [&](int x, int b) { return bars + 8u * (5 + 4 * RING + 2 * x + b); };
  auto pv_done = [&](int x, int b) { return bars + 8u * (9 + 4 * RING + 2 * x + b); };
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + OFF_TMEM);

  const int nq = (p.S + BQ - 1) / BQ;
  const int npair = (nq + 1) / 2;
  const int t = npair - 1 - (int)blockIdx.x;  // heavy (late) pairs first
  const int h = blockIdx.y;
  const int g = h / (p.H / p.KV);
  const int qt[2] = {2 * t, 2 * t + 1};
  // key tiles per query tile (causal): keys [0, (qt+1)*128); tile B may not exist
  const int nt[2] = {2 * (qt[0] + 1), qt[1] < nq ? 2 * (qt[1] + 1) : 0};
  const int nmax = nt[0] > nt[1] ? nt[0] : nt[1];

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&p.q);
    ptx::prefetch_tmap(&p.k);
    ptx::prefetch_tmap(&p.vt);
    ptx::mbar_init(q_full, 1);
    for (int s = 0; s < RING; ++s) {
      ptx::mbar_init(k_full(s), 1);
      ptx::mbar_init(k_empty(s), 1);
      ptx::mbar_init(v_full(s), 1);
      ptx::mbar_init(v_empty(s), 1);
    }
    for (int x = 0; x < 2; ++x) {
      ptx::mbar_init(s_full(x, 0), 1);
      ptx::mbar_init(s_full(x, 1), 1);
      ptx::mbar_init(p_full(x, 0), 128);
      ptx::mbar_init(p_full(x, 1), 128);
      ptx::mbar_init(pv_done(x, 0), 1);
      ptx::mbar_init(pv_done(x, 1), 1);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc(ptx::smem_u32(tmem_holder), 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {
      const int qc = h * HD, kc = (p.H + g) * HD, vr = g * HD;
      ptx::mbar_expect_tx(q_full, (nt[1] ? 2 : 1) * QTILE);
      for (int x = 0; x < 2; ++x) {
        if (!nt[x]) continue;
        const uint32_t qs = sb + OFF_Q + x * QTILE;
        ptx::tma_load_2d(&p.q, qs, q_full, qc, qt[x] * BQ);
        ptx::tma_load_2d(&p.q, qs + QHALF, q_full, qc + 64, qt[x] * BQ);
      }
      for (int j = 0; j < nmax; ++j) {
        const int s = j % RING;
        const uint32_t par = ((j / RING) & 1) ^ 1;
        ptx::mbar_wait(k_empty(s), par);
        ptx::mbar_expect_tx(k_full(s), KTILE);
        const uint32_t ks = sb + OFF_K + s * KTILE;
        ptx::tma_load_2d(&p.k, ks, k_full(s), kc, j * BKV);
        ptx::tma_load_2d(&p.k, ks + KHALF, k_full(s), kc + 64, j * BKV);
        ptx::mbar_wait(v_empty(s), par);
        ptx::mbar_expect_tx(v_full(s), VTILE);
        ptx::tma_load_2d(&p.vt, sb + OFF_V + s * VTILE, v_full(s), j * BKV, vr);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t IDESC_S = ptx::idesc_bf16(128, BKV);
      constexpr uint32_t IDESC_O = ptx::idesc_bf16(128, HD);
      ptx::mbar_wait(q_full, 0);
      auto issue_s = [&](int x, int j) {  // S_x = Q_x K_j^T  (128 x 64, K = 128)
        const int s = j % RING;
        ptx::mbar_wait(k_full(s), (j / RING) & 1);
        ptx::tc_fence_after();
        const uint32_t qs = sb + OFF_Q + x * QTILE, ks = sb + OFF_K + s * KTILE;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          ptx::mma_bf16(tmem + COL_S + (2 * x + (j & 1)) * BKV,
                        ptx::desc_sw128(qs + (kk >> 2) * QHALF) + 2 * (kk & 3),
                        ptx::desc_sw128(ks + (kk >> 2) * KHALF) + 2 * (kk & 3), IDESC_S, kk > 0);
        ptx::mma_commit(s_full(x, j & 1));
      };
      auto issue_pv = [&](int x, int j) {  // O_x += P_x V_j  (128 x 128, K = 64)
        ptx::mbar_wait(p_full(x, j & 1), (j >> 1) & 1);
        ptx::mbar_wait(v_full(j % RING), (j / RING) & 1);
        ptx::tc_fence_after();
        const uint32_t ps = sb + OFF_P + (2 * x + (j & 1)) * PTILE,
                       vs = sb + OFF_V + (j % RING) * VTILE;
#pragma unroll
        for (int kk = 0; kk < BKV / 16; ++kk)
          ptx::mma_bf16(tmem + COL_O + x * HD, ptx::desc_sw128(ps) + 2 * kk,
                        ptx::desc_sw128(vs) + 2 * kk, IDESC_O, (j | kk) != 0);
        ptx::mma_commit(pv_done(x, j & 1));
      };
      // S runs two tiles ahead of PV: S_x(j+2) reuses the S buffer of tile j,
      // which softmax x has released by the time P_x(j) is published.
      for (int jj = 0; jj < 2 && jj < nmax; ++jj) {
        for (int x = 0; x < 2; ++x)
          if (jj < nt[x]) issue_s(x, jj);
        ptx::mma_commit(k_empty(jj % RING));
      }
      for (int j = 0; j < nmax; ++j) {
        for (int x = 0; x < 2; ++x) {
          if (j >= nt[x]) continue;
          issue_pv(x, j);
          if (j + 2 < nt[x]) issue_s(x, j + 2);
        }
        ptx::mma_commit(v_empty(j % RING));
        if (j + 2 < nmax) ptx::mma_commit(k_empty((j + 2) % RING));
      }
    }
    __syncwarp();
  } else {
    // ===================== softmax: warps 2..5 tile A, 6..9 tile B =====================
    const int x = (warp - 2) >> 2;
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int qi = qt[x] * BQ + row;
    const int n = nt[x];
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    const uint32_t o_col = tmem + lane_base + COL_O + x * HD;
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < n; ++j) {
      ptx::mbar_wait(s_full(x, j & 1), (j >> 1) & 1);
      ptx::tc_fence_after();
      const uint32_t s_col = tmem + lane_base + COL_S + (2 * x + (j & 1)) * BKV;
      float v[BKV];
      {
        uint32_t r0[32], r1[32];
        ptx::tmem_ld32(s_col, r0);
        ptx::tmem_ld32(s_col + 32, r1);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          v[i] = __uint_as_float(r0[i]);  // raw scores
          v[32 + i] = __uint_as_float(r1[i]);
        }
      }
      if ((j + 1) * BKV > qt[x] * BQ) {  // tiles reaching the diagonal: causal mask
#pragma unroll
        for (int i = 0; i < BKV; ++i)
          if (j * BKV + i > qi) v[i] = -INFINITY;
      }
      float mr[8];  // 8 independent max chains
#pragma unroll
      for (int k = 0; k < 8; ++k) mr[k] = v[k];
#pragma unroll
      for (int i = 8; i < BKV; ++i) mr[i & 7] = fmaxf(mr[i & 7], v[i]);
      const float mraw = fmaxf(fmaxf(fmaxf(mr[0], mr[1]), fmaxf(mr[2], mr[3])),
                               fmaxf(fmaxf(mr[4], mr[5]), fmaxf(mr[6], mr[7])));
      const float mx = fmaxf(m_used, mraw * p.scale_log2);  // scale > 0: max commutes
      const bool need = mx > m_used + 8.f;
      if (j > 0 && __any_sync(0xffffffffu, need)) {
        ptx::mbar_wait(pv_done(x, (j - 1) & 1), ((j - 1) >> 1) & 1);  // O_x settled
        ptx::tc_fence_after();
        const float corr = need ? exp2f(m_used - mx) : 1.f;
#pragma unroll 1
        for (int c = 0; c < HD / 32; ++c) {
          uint32_t r[32];
          ptx::tmem_ld32(o_col + c * 32, r);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * corr);
          ptx::tmem_st32(o_col + c * 32, r);
        }
        ptx::tmem_st_wait();
        l *= corr;
      }
      if (need) m_used = mx;
      // P buffer j&1 was last read by PV_x(j-2)
      if (j > 1) ptx::mbar_wait(pv_done(x, j & 1), ((j - 2) >> 1) & 1);
      uint8_t* Ps = smem + OFF_P + (2 * x + (j & 1)) * PTILE;
      // P = exp2(s*scale - m) -> bf16, SWIZZLE_128B K-major [128 rows][64 keys]
      float ls[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // independent sum chains
#pragma unroll
      for (int c = 0; c < BKV / 8; ++c) {
        float e[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          e[i] = exp2f(fmaf(v[c * 8 + i], p.scale_log2, -m_used));
          ls[i] += e[i];
        }
        uint4 w;
        w.x = pack_bf16x2(e[0], e[1]);
        w.y = pack_bf16x2(e[2], e[3]);
        w.z = pack_bf16x2(e[4], e[5]);
        w.w = pack_bf16x2(e[6], e[7]);
        *reinterpret_cast<uint4*>(Ps + row * 128 + ((c ^ (row & 7)) << 4)) = w;
      }
      l += ((ls[0] + ls[1]) + (ls[2] + ls[3])) + ((ls[4] + ls[5]) + (ls[6] + ls[7]));
      ptx::fence_proxy_async_smem();
      ptx::tc_fence_before();
      ptx::mbar_arrive(p_full(x, j & 1));
    }
    if (n > 0) {
      // epilogue: O / l -> bf16
      ptx::mbar_wait(pv_done(x, (n - 1) & 1), ((n - 1) >> 1) & 1);
      ptx::tc_fence_after();
      const float inv = 1.f / l;
      bf16* out = p.out + (size_t)qi * p.ldo + h * HD;
#pragma unroll 1
      for (int c = 0; c < HD / 32; ++c) {
        uint32_t r[32];
        ptx::tmem_ld32(o_col + c * 32, r);
        ptx::tmem_ld_wait();
        if (qi < p.S) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            uint4 w;
            w.x = pack_bf16x2(__uint_as_float(r[8 * k + 0]) * inv, __uint_as_float(r[8 * k + 1]) * inv);
            w.y = pack_bf16x2(__uint_as_float(r[8 * k + 2]) * inv, __uint_as_float(r[8 * k + 3]) * inv);
            w.z = pack_bf16x2(__uint_as_float(r[8 * k + 4]) * inv, __uint_as_float(r[8 * k + 5]) * inv);
            w.w = pack_bf16x2(__uint_as_float(r[8 * k + 6]) * inv, __uint_as_float(r[8 * k + 7]) * inv);
            *reinterpret_cast<uint4*>(out + c * 32 + k * 8) = w;
          }
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

}  // namespace

bool attn_tc_params(AttnParams* p, const bf16* qkv, const bf16* vt, int vt_ld, bf16* out, int S,
                    int H, int KV) {
  const int ld = (H + 2 * KV) * HD;
  if (!make_tmap(&p->q, qkv, S, ld, (uint64_t)ld * 2, BQ, 64)) return false;
  if (!make_tmap(&p->k, qkv, S, ld, (uint64_t)ld * 2, BKV, 64)) return false;
  if (!make_tmap(&p->vt, vt, (uint64_t)KV * HD, S, (uint64_t)vt_ld * 2, HD, 64)) return false;
  p->S = S;
  p->H = H;
  p->KV = KV;
  p->scale_log2 = 1.4426950408889634f / sqrtf((float)HD);
  p->out = out;
  p->ldo = H * HD;
  return true;
}

cudaError_t attn_tc_launch(const AttnParams& p, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e =
        cudaFuncSetAttribute(attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int nq = (p.S + BQ - 1) / BQ;
  dim3 grid((nq + 1) / 2, p.H);
  attn_tc_kernel<<<grid, NTH, SMEM, s>>>(p);
  return cudaGetLastError();
}

}  // namespace tidal
