// attn_tc.cu — causal GQA prefill attention on 5th-gen tensor cores (hd = 128).
//   O_h = softmax(Q_h K_g^T / sqrt(hd) + causal) V_g,   g = h / (H / KV)
// CTA = 128 queries of one head; warp-specialised like the GEMM:
//   warp 0      TMA: Q once, then K / V^T tiles of 128 keys (separate rings:
//               K_j is released as soon as S_j is computed, V_j after PV_j)
//   warp 1      tcgen05.mma: S_j = Q K_j^T into TMEM (double-buffered, so
//               S_{j+1} runs while softmax works on S_j), then O += P_j V_j
//               with P_j read straight from TMEM (the "TS" MMA form)
//   warps 2..9  softmax in two column halves: warps 2..5 own keys 0..63 and
//               warps 6..9 keys 64..127 of the same 128 query rows (TMEM lane
//               = row; both halves share a lane quarter), exchanging row
//               maxima through shared memory; P = 2^(S*scale - m) rounded to
//               bf16 and stored to TMEM (tcgen05.st, double-buffered: softmax
//               of tile j+1 writes P_{j+1} while the tensor core runs PV_j);
//               fp32 running row sums.  O lives in TMEM for the whole CTA; it
//               is rescaled (each half its 64 columns) only when a row max
//               grows by more than 2^8 (exact: O and l share the same stale
//               max, P <= 256).
// V is consumed as V^T [hd][S] (written transposed by the QKV GEMM epilogue),
// so the PV MMA's B operand is K-major in shared memory.
// TMEM columns: S_0 [0,128), S_1 [128,256), O [256,384), P_0 [384,448),
// P_1 [448,512) (P: 128 keys as 64 packed bf16x2 columns).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"
#include "launch.cuh"
#include "ptx.cuh"

namespace tidal {
namespace {

constexpr int HD = 128, BQ = 128, BKV = 128;
constexpr int TILE = 128 * 128 * 2;  // 32 KB: any 128 x 128 bf16 tile (two 64-wide K-blocks)
constexpr int HALF = TILE / 2;
constexpr int KST = 2, VST = 3;
constexpr int OFF_Q = 0, OFF_K = OFF_Q + TILE, OFF_V = OFF_K + KST * TILE;
constexpr int OFF_RED = OFF_V + VST * TILE;          // [2 slots][2 halves][128] row maxima
constexpr int OFF_BAR = OFF_RED + 2 * 2 * BQ * 4;
constexpr int N_BARS = 1 + 2 * KST + 2 * VST + 2 + 2 + 2;
constexpr int OFF_TMEM = OFF_BAR + N_BARS * 8;
constexpr int SMEM = OFF_TMEM + 16 + 1024;
constexpr int NSOFT = 256;           // softmax threads
constexpr int NTH = 64 + NSOFT;
constexpr uint32_t COL_S0 = 0, COL_O = 256, COL_P = 384;

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ void softmax_bar() {  // the 8 softmax warps only
  asm volatile("bar.sync 1, %0;" ::"n"(NSOFT) : "memory");
}
__global__ void __launch_bounds__(NTH, 1) attn_tc_kernel(const __grid_constant__ AttnParams p) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned (SWIZZLE_128B); offsetting smem_raw keeps the shared state
  // space visible to the compiler (STS/LDS, not generic ST/LD)
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sb = ptx::smem_u32(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t bars = sb + OFF_BAR;
  const uint32_t q_full = bars;
  auto k_full = [&](int s) { return bars + 8u * (1 + s); };
  auto k_empty = [&](int s) { return bars + 8u * (1 + KST + s); };
  auto v_full = [&](int s) { return bars + 8u * (1 + 2 * KST + s); };
  auto v_empty = [&](int s) { return bars + 8u * (1 + 2 * KST + VST + s); };
  auto s_full = [&](int b) { return bars + 8u * (1 + 2 * KST + 2 * VST + b); };
  // per-P-buffer barriers: softmax runs up to one tile ahead of the PV MMAs, so
  // a single barrier could complete two phases before its waiter looks
  auto p_full = [&](int b) { return bars + 8u * (3 + 2 * KST + 2 * VST + b); };
  auto pv_done = [&](int b) { return bars + 8u * (5 + 2 * KST + 2 * VST + b); };
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + OFF_TMEM);

  const int nq = (p.S + BQ - 1) / BQ;
  const int qt = nq - 1 - (int)blockIdx.x;  // heavy (late) query tiles first
  const int h = blockIdx.y;
  const int g = h / (p.H / p.KV);
  const int q0 = qt * BQ;                   // positions within the sequence
  const int base = blockIdx.z * p.S;        // first row of this sequence (batched prompts)
  const int vbase = blockIdx.z * ((p.S + 63) & ~63);  // its first V^T column (64-aligned)
  const int nkv = qt + 1;                   // causal: key tiles 0..qt (BQ == BKV)

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&p.q);
    ptx::prefetch_tmap(&p.vt);
    ptx::mbar_init(q_full, 1);
    for (int s = 0; s < KST; ++s) {
      ptx::mbar_init(k_full(s), 1);
      ptx::mbar_init(k_empty(s), 1);
    }
    for (int s = 0; s < VST; ++s) {
      ptx::mbar_init(v_full(s), 1);
      ptx::mbar_init(v_empty(s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(s_full(b), 1);
      ptx::mbar_init(p_full(b), NSOFT);
      ptx::mbar_init(pv_done(b), 1);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc(ptx::smem_u32(tmem_holder), 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  ptx::pdl_begin();

  if (warp == 0) {
    if (lane == 0) {
      const int qc = h * HD, kc = (p.H + g) * HD, vr = g * HD;
      ptx::mbar_expect_tx(q_full, TILE);
      ptx::tma_load_2d(&p.q, sb + OFF_Q, q_full, qc, base + q0);
      ptx::tma_load_2d(&p.q, sb + OFF_Q + HALF, q_full, qc + 64, base + q0);
      // in-order issue K_0 V_0 K_1 V_1 ...
      for (int j = 0; j < nkv; ++j) {
        const int s = j % KST, t = j % VST;
        ptx::mbar_wait(k_empty(s), ((j / KST) & 1) ^ 1);
        ptx::mbar_expect_tx(k_full(s), TILE);
        const uint32_t ks = sb + OFF_K + s * TILE;
        ptx::tma_load_2d(&p.q, ks, k_full(s), kc, base + j * BKV);
        ptx::tma_load_2d(&p.q, ks + HALF, k_full(s), kc + 64, base + j * BKV);
        ptx::mbar_wait(v_empty(t), ((j / VST) & 1) ^ 1);
        ptx::mbar_expect_tx(v_full(t), TILE);
        const uint32_t vs = sb + OFF_V + t * TILE;
        ptx::tma_load_2d(&p.vt, vs, v_full(t), vbase + j * BKV, vr);
        ptx::tma_load_2d(&p.vt, vs + HALF, v_full(t), vbase + j * BKV + 64, vr);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t IDESC = ptx::idesc_bf16(128, 128);
      ptx::mbar_wait(q_full, 0);
      auto issue_s = [&](int j) {
        const int s = j % KST;
        ptx::mbar_wait(k_full(s), (j / KST) & 1);
        ptx::tc_fence_after();
        const uint32_t ks = sb + OFF_K + s * TILE;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off = (kk >> 2) * HALF;
          ptx::mma_bf16(tmem + COL_S0 + (j & 1) * 128,
                        ptx::desc_sw128(sb + OFF_Q + off) + 2 * (kk & 3),
                        ptx::desc_sw128(ks + off) + 2 * (kk & 3), IDESC, kk > 0);
        }
        ptx::mma_commit(s_full(j & 1));
        ptx::mma_commit(k_empty(s));
      };
      issue_s(0);
      for (int j = 0; j < nkv; ++j) {
        // S_{j+1} overwrites S buffer (j+1)&1, last read by softmax j-1 (it
        // arrived on p_full(j-1), which this thread observed last iteration)
        if (j + 1 < nkv) issue_s(j + 1);
        const int t = j % VST, b = j & 1;
        ptx::mbar_wait(p_full(b), (j >> 1) & 1);
        ptx::mbar_wait(v_full(t), (j / VST) & 1);
        ptx::tc_fence_after();
        const uint32_t vs = sb + OFF_V + t * TILE;
#pragma unroll
        for (int kk = 0; kk < BKV / 16; ++kk) {
          const uint32_t off = (kk >> 2) * HALF;
          ptx::mma_bf16_ts(tmem + COL_O, tmem + COL_P + b * 64 + kk * 8,
                           ptx::desc_sw128(vs + off) + 2 * (kk & 3), IDESC, (j | kk) != 0);
        }
        ptx::mma_commit(v_empty(t));
        ptx::mma_commit(pv_done(b));
      }
    }
    __syncwarp();
  } else {
    // ===================== softmax: two column halves =====================
    const int half = (warp - 2) >> 2;  // 0: keys 0..63, 1: keys 64..127 of each tile
    const int q = warp & 3;            // TMEM lane quarter (shared by both halves)
    const int row = q * 32 + lane;
    const int qi = q0 + row;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    float* red = reinterpret_cast<float*>(smem + OFF_RED);  // [slot][half][row]
    const uint32_t o_col = tmem + lane_base + COL_O + half * 64;
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < nkv; ++j) {
      const int b = j & 1;
      ptx::mbar_wait(s_full(b), (j >> 1) & 1);
      ptx::tc_fence_after();
      float v[64];
      {
        uint32_t r0[32], r1[32];
        const uint32_t sc = tmem + lane_base + COL_S0 + b * 128 + half * 64;
        ptx::tmem_ld32(sc, r0);
        ptx::tmem_ld32(sc + 32, r1);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          v[i] = __uint_as_float(r0[i]);  // raw scores
          v[32 + i] = __uint_as_float(r1[i]);
        }
      }
      const int key0 = j * BKV + half * 64;
      if (key0 + 63 > q0) {  // reaches the diagonal: causal mask
#pragma unroll
        for (int i = 0; i < 64; ++i)
          if (key0 + i > qi) v[i] = -INFINITY;
      }
      float mr[8];  // 8 independent max chains
#pragma unroll
      for (int k = 0; k < 8; ++k) mr[k] = v[k];
#pragma unroll
      for (int i = 8; i < 64; ++i) mr[i & 7] = fmaxf(mr[i & 7], v[i]);
      float mraw = fmaxf(fmaxf(fmaxf(mr[0], mr[1]), fmaxf(mr[2], mr[3])),
                         fmaxf(fmaxf(mr[4], mr[5]), fmaxf(mr[6], mr[7])));
      // exchange the half-row maxima (double-buffered slot: no WAR hazard)
      float* slot = red + b * 2 * BQ;
      slot[half * BQ + row] = mraw;
      softmax_bar();
      mraw = fmaxf(mraw, slot[(half ^ 1) * BQ + row]);
      const float mx = fmaxf(m_used, mraw * p.scale_log2);  // scale > 0: max commutes
      const bool need = mx > m_used + 8.f;                  // identical in both halves
      if (j > 0 && __any_sync(0xffffffffu, need)) {
        // O settled: PV_{j-1} (and so every earlier PV) has completed
        ptx::mbar_wait(pv_done((j - 1) & 1), ((j - 1) >> 1) & 1);
        ptx::tc_fence_after();
        const float corr = need ? ptx::ex2(m_used - mx) : 1.f;
#pragma unroll 1
        for (int c = 0; c < 2; ++c) {
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
      // P buffer b was last read by PV_{j-2}
      if (j >= 2) ptx::mbar_wait(pv_done(b), ((j - 2) >> 1) & 1);
      // P = 2^(s*scale - m) -> packed bf16 pairs, 32 TMEM columns per half
      float ls[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // independent sum chains
      uint32_t pk[32];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        float e[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          e[i] = ptx::ex2(fmaf(v[c * 8 + i], p.scale_log2, -m_used));
          ls[i] += e[i];
        }
        pk[4 * c + 0] = pack_bf16x2(e[0], e[1]);
        pk[4 * c + 1] = pack_bf16x2(e[2], e[3]);
        pk[4 * c + 2] = pack_bf16x2(e[4], e[5]);
        pk[4 * c + 3] = pack_bf16x2(e[6], e[7]);
      }
      ptx::tc_fence_after();
      ptx::tmem_st32(tmem + lane_base + COL_P + b * 64 + half * 32, pk);
      l += ((ls[0] + ls[1]) + (ls[2] + ls[3])) + ((ls[4] + ls[5]) + (ls[6] + ls[7]));
      ptx::tmem_st_wait();
      ptx::tc_fence_before();
      ptx::mbar_arrive(p_full(b));
    }
    // epilogue: combine the half-row sums, O / l -> bf16 (each half its 64 columns)
    float* lsum = red;  // reuse slot 0 after a barrier (all maxima consumed)
    softmax_bar();
    lsum[half * BQ + row] = l;
    softmax_bar();
    const float inv = 1.f / (l + lsum[(half ^ 1) * BQ + row]);
    ptx::mbar_wait(pv_done((nkv - 1) & 1), ((nkv - 1) >> 1) & 1);
    ptx::tc_fence_after();
    bf16* out = p.out + (size_t)(base + qi) * p.ldo + h * HD + half * 64;
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
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
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

}  // namespace

bool attn_tc_params(AttnParams* p, const bf16* qkv, const bf16* vt, int vt_ld, bf16* out, int S,
                    int H, int KV, int nseq) {
  const int ld = (H + 2 * KV) * HD;
  const uint64_t rows = (uint64_t)S * nseq;
  if (nseq < 1 || nseq > 65535) return false;
  if (!make_tmap(&p->q, qkv, rows, ld, (uint64_t)ld * 2, 128, 64)) return false;
  p->k = p->q;  // K tiles are 128 keys: same box as Q
  // V^T columns: sequence b at b * round_up(S, 64) (the QKV epilogue's layout); one
  // sequence: S columns, keys past S read as zero (out of bounds)
  const uint64_t vcols = nseq > 1 ? (uint64_t)nseq * ((S + 63) & ~63) : (uint64_t)S;
  if (vcols > (uint64_t)vt_ld) return false;
  if (!make_tmap(&p->vt, vt, (uint64_t)KV * HD, vcols, (uint64_t)vt_ld * 2, 128, 64)) return false;
  p->S = S;
  p->nseq = nseq;
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
  dim3 grid((p.S + BQ - 1) / BQ, p.H, p.nseq);
  return launch_k(attn_tc_kernel, grid, dim3(NTH), SMEM, s, 1, p);
}

}  // namespace tidal
