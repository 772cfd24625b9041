// attn_tc.cu — causal GQA prefill attention on 5th-gen tensor cores (hd = 128).
//   O_h = softmax(Q_h K_g^T / sqrt(hd) + causal) V_g,   g = h / (H / KV)
// Two kernels: attn_pp_kernel (below the first one) takes PAIRS of query
// tiles with one softmax warpgroup per tile, so one tile's softmax overlaps
// the other's MMAs; it is used whenever there are enough pairs to fill the
// SMs (attn_tc_launch).  The single-tile kernel first:
// Persistent: one CTA per SM walks a static list of work items (128 queries
// of one head of one sequence), heaviest (latest) query tiles first, in a
// snake order across CTAs; TMEM, barriers and the K/V rings live across
// items, so the next item's Q and K tiles stream in under the current item's
// last tiles and there is no per-item launch, allocation or pipeline fill.
// Warp roles:
//   warp 0      TMA: per item Q once, then K / V^T tiles of 128 keys
//               (separate rings: K_j is released when S_j is computed, V_j
//               after PV_j; the Q buffer after the item's last S MMA)
//   warp 1      tcgen05.mma: S_j = Q K_j^T into TMEM (double-buffered, so
//               S_{j+1} runs while softmax works on S_j), then O += P_j V_j
//               with P_j read straight from TMEM (the "TS" MMA form)
//   warps 2..9  softmax in two column halves: warps 2..5 own keys 0..63 and
//               warps 6..9 keys 64..127 of the same 128 query rows (TMEM lane
//               = row; both halves share a lane quarter), exchanging row
//               maxima through shared memory; P = 2^(S*scale - m) rounded to
//               bf16 and stored to TMEM (tcgen05.st, double-buffered: softmax
//               of tile j+1 writes P_{j+1} while the tensor core runs PV_j);
//               fp32 running row sums.  O lives in TMEM for the whole item;
//               it is rescaled (each half its 64 columns) only when a row max
//               grows by more than 2^8 (exact: O and l share the same stale
//               max, P <= 256).  At an item's end they only publish the row
//               sums (l_ready) and move on to the next item.
//   warps 10..13 epilogue, one row per thread: read O (freeing it for the next
//               item's first PV), O / l -> bf16, store — off the softmax path
//               (measured 64 -> 60 us at 13B, S = 2048).
// All barrier parities derive from per-CTA running counters (items, K/V
// tiles, S/P buffers), never from the per-item tile index.
// V is consumed as V^T [hd][S] (written transposed by the QKV GEMM epilogue),
// so the PV MMA's B operand is K-major in shared memory.
// TMEM columns: S_0 [0,128), S_1 [128,256), O [256,384), P_0 [384,448),
// P_1 [448,512) (P: 128 keys as 64 packed bf16x2 columns).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <queue>
#include <vector>

#include <cstdint>
#include <cstdlib>

#include "kernels.h"
#include "launch.cuh"
#include "ptx.cuh"

namespace tidal {
namespace {

constexpr int HD = 128, BQ = 128, BKV = 128;
constexpr int TILE = 128 * 128 * 2;  // 32 KB: any 128 x 128 bf16 tile (two 64-wide K-blocks)
constexpr int HALF = TILE / 2;
constexpr int KST = 3, VST = 2;
constexpr int OFF_Q = 0, OFF_K = OFF_Q + TILE, OFF_V = OFF_K + KST * TILE;
// Softmax in SPLIT column groups of the 128 keys of a tile (SPLIT = 2: 8
// warps, 64 columns per thread; SPLIT = 4: 16 warps, 32 columns per thread —
// twice the warps per scheduler to hide the per-tile TMEM / barrier latency)
template <int SPLIT>
struct ACfg {
  static constexpr int OFF_RED = OFF_V + VST * TILE;              // [2 slots][SPLIT][128] row maxima
  static constexpr int OFF_LSUM = OFF_RED + 2 * SPLIT * BQ * 4;   // [2 items][SPLIT][128] row sums
  static constexpr int OFF_BAR = OFF_LSUM + 2 * SPLIT * BQ * 4;
  static constexpr int N_BARS = 4 + 2 * KST + 2 * VST + 2 + 2 + 2 + 2;
  static constexpr int OFF_TMEM = OFF_BAR + N_BARS * 8;
  static constexpr int SMEM = OFF_TMEM + 16 + 1024;
  static constexpr int NSOFT = 128 * SPLIT;  // softmax threads
  static constexpr int NEPI = 128;           // epilogue threads: O / l -> bf16, off the softmax path
  static constexpr int NTH = 64 + NSOFT + NEPI;
  static constexpr int COLS = 128 / SPLIT;   // keys per softmax thread
};
constexpr uint32_t COL_S0 = 0, COL_O = 256, COL_P = 384;

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
template <int NSOFT>
__device__ __forceinline__ void softmax_bar() {  // the softmax warps only
  asm volatile("bar.sync 1, %0;" ::"n"(NSOFT) : "memory");
}

struct Item {
  int qt, h, z;
};

// diagnostic timeline (AttnParams::dbg): per CTA, per S/P tile (first 64), 8
// slots: 0 MMA wants S, 1 S issued, 2 softmax sees S, 3 softmax done (P),
// 4 MMA wants PV, 5 PV issued
constexpr int ADBG_TILES = 64;
__device__ __forceinline__ void adbg(const AttnParams& p, int tile, int slot) {
  if (p.dbg && tile < ADBG_TILES) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.dbg[((size_t)blockIdx.x * ADBG_TILES + tile) * 8 + slot] = t;
  }
}
// paired-kernel timeline (same buffer): per CTA, per pair item (first 64), 8
// slots: 0 producer issues Q, 1 MMA wants S(0), 2 MMA issued S_B(0),
// 3 MMA issued PV_A(0) (after o_empty), 4 softmax B sees S(0), 5 softmax B
// stored P(0), 6 MMA issued the item's last PV, 7 epilogue drained O_B
__device__ __forceinline__ void pdbg(const AttnParams& p, int item, int slot) {
  adbg(p, item, slot);
}
// Work item i of this CTA (round-robin rounds, snake order so that the CTAs
// taking the heaviest item of one round take the lightest of the next);
// items are numbered heaviest first: qt = nq-1 .. 0, then head, then sequence.
__device__ __forceinline__ bool item_at(const AttnParams& p, int nq, int round, Item& it) {
  const int G = gridDim.x;
  const int c = blockIdx.x;
  const int idx = round * G + ((round & 1) ? G - 1 - c : c);
  const int per_qt = p.H * p.nseq;
  if (idx >= nq * per_qt) return false;
  const int k = idx / per_qt, rem = idx - k * per_qt;
  it.qt = nq - 1 - k;
  it.h = rem % p.H;
  it.z = rem / p.H;
  return true;
}

template <int SPLIT>
__global__ void __launch_bounds__(ACfg<SPLIT>::NTH, 1) attn_tc_kernel(const __grid_constant__ AttnParams p) {
  using A = ACfg<SPLIT>;
  constexpr int OFF_RED = A::OFF_RED, OFF_LSUM = A::OFF_LSUM, OFF_BAR = A::OFF_BAR,
                OFF_TMEM = A::OFF_TMEM, NSOFT = A::NSOFT, NEPI = A::NEPI, COLS = A::COLS;
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned (SWIZZLE_128B); offsetting smem_raw keeps the shared state
  // space visible to the compiler (STS/LDS, not generic ST/LD)
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sb = ptx::smem_u32(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t bars = sb + OFF_BAR;
  const uint32_t q_full = bars, q_empty = bars + 8, o_empty = bars + 16;
  auto k_full = [&](int s) { return bars + 8u * (4 + s); };
  auto k_empty = [&](int s) { return bars + 8u * (4 + KST + s); };
  auto v_full = [&](int s) { return bars + 8u * (4 + 2 * KST + s); };
  auto v_empty = [&](int s) { return bars + 8u * (4 + 2 * KST + VST + s); };
  auto s_full = [&](int b) { return bars + 8u * (4 + 2 * KST + 2 * VST + b); };
  // per-P-buffer barriers: softmax runs up to one tile ahead of the PV MMAs, so
  // a single barrier could complete two phases before its waiter looks
  auto p_full = [&](int b) { return bars + 8u * (6 + 2 * KST + 2 * VST + b); };
  auto pv_done = [&](int b) { return bars + 8u * (8 + 2 * KST + 2 * VST + b); };
  // the softmax warps publish an item's row sums; the epilogue warps take it
  auto l_ready = [&](int b) { return bars + 8u * (10 + 2 * KST + 2 * VST + b); };
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + OFF_TMEM);

  const int nq = (p.S + BQ - 1) / BQ;
  const int vld = (p.S + 63) & ~63;  // V^T columns per sequence (64-aligned)

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&p.q);
    ptx::prefetch_tmap(&p.vt);
    ptx::mbar_init(q_full, 1);
    ptx::mbar_init(q_empty, 1);
    ptx::mbar_init(o_empty, NEPI);
    for (int b = 0; b < 2; ++b) ptx::mbar_init(l_ready(b), NSOFT);
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

  Item it;
  if (warp == 0) {
    if (lane == 0) {
      int kc = 0, vc = 0;  // K / V tiles issued by this CTA
      for (int i = 0; item_at(p, nq, i, it); ++i) {
        const int g = it.h / (p.H / p.KV);
        const int base = it.z * p.S;
        const int qc = it.h * HD, kcol = (p.H + g) * HD, vr = g * HD;
        // the previous item's S MMAs have consumed Q
        ptx::mbar_wait(q_empty, (i & 1) ^ 1);
        ptx::mbar_expect_tx(q_full, TILE);
        ptx::tma_load_2d(&p.q, sb + OFF_Q, q_full, qc, base + it.qt * BQ);
        ptx::tma_load_2d(&p.q, sb + OFF_Q + HALF, q_full, qc + 64, base + it.qt * BQ);
        // in-order issue K_0 V_0 K_1 V_1 ...
        for (int j = 0; j <= it.qt; ++j, ++kc, ++vc) {
          const int s = kc % KST, t = vc % VST;
          ptx::mbar_wait(k_empty(s), ((kc / KST) & 1) ^ 1);
          ptx::mbar_expect_tx(k_full(s), TILE);
          const uint32_t ks = sb + OFF_K + s * TILE;
          ptx::tma_load_2d(&p.q, ks, k_full(s), kcol, base + j * BKV);
          ptx::tma_load_2d(&p.q, ks + HALF, k_full(s), kcol + 64, base + j * BKV);
          ptx::mbar_wait(v_empty(t), ((vc / VST) & 1) ^ 1);
          ptx::mbar_expect_tx(v_full(t), TILE);
          const uint32_t vs = sb + OFF_V + t * TILE;
          ptx::tma_load_2d(&p.vt, vs, v_full(t), it.z * vld + j * BKV, vr);
          ptx::tma_load_2d(&p.vt, vs + HALF, v_full(t), it.z * vld + j * BKV + 64, vr);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t IDESC = ptx::idesc_bf16(128, 128);
      int kc = 0, vc = 0, gs = 0, gp = 0;  // K / V tiles, S and PV MMAs issued
      auto issue_s = [&]() {
        const int s = kc % KST;
        adbg(p, gs, 0);
        ptx::mbar_wait(k_full(s), (kc / KST) & 1);
        ptx::tc_fence_after();
        adbg(p, gs, 1);
        const uint32_t ks = sb + OFF_K + s * TILE;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off = (kk >> 2) * HALF;
          ptx::mma_bf16(tmem + COL_S0 + (gs & 1) * 128,
                        ptx::desc_sw128(sb + OFF_Q + off) + 2 * (kk & 3),
                        ptx::desc_sw128(ks + off) + 2 * (kk & 3), IDESC, kk > 0);
        }
        ptx::mma_commit(s_full(gs & 1));
        ptx::mma_commit(k_empty(s));
        ++kc;
        ++gs;
      };
      for (int i = 0; item_at(p, nq, i, it); ++i) {
        const int nkv = it.qt + 1;  // causal: key tiles 0..qt (BQ == BKV)
        ptx::mbar_wait(q_full, i & 1);
        ptx::tc_fence_after();
        // S buffer (gs&1) was last read by the softmax of S MMA gs-2, which
        // arrived on p_full before this thread issued PV gs-2
        issue_s();
        for (int j = 0; j < nkv; ++j) {
          if (j + 1 < nkv) issue_s();
          if (j + 1 >= nkv) ptx::mma_commit(q_empty);  // all S MMAs of the item issued
          const int t = vc % VST, b = gp & 1;
          adbg(p, gp, 4);
          ptx::mbar_wait(p_full(b), (gp >> 1) & 1);
          ptx::mbar_wait(v_full(t), (vc / VST) & 1);
          // O of the previous item has been read out by the epilogue
          if (j == 0 && i > 0) ptx::mbar_wait(o_empty, (i - 1) & 1);
          ptx::tc_fence_after();
          adbg(p, gp, 5);
          const uint32_t vs = sb + OFF_V + t * TILE;
#pragma unroll
          for (int kk = 0; kk < BKV / 16; ++kk) {
            const uint32_t off = (kk >> 2) * HALF;
            ptx::mma_bf16_ts(tmem + COL_O, tmem + COL_P + b * 64 + kk * 8,
                             ptx::desc_sw128(vs + off) + 2 * (kk & 3), IDESC, (j | kk) != 0);
          }
          ptx::mma_commit(v_empty(t));
          ptx::mma_commit(pv_done(b));
          ++vc;
          ++gp;
        }
      }
    }
    __syncwarp();
  } else if (warp >= 2 + NSOFT / 32) {
    // ===================== epilogue: O / l -> bf16 =====================
    // one row per thread (TMEM lane quarter = warp & 3), all 128 columns; O is
    // released as soon as it is read, so the next item's PVs and softmax run
    // while these warps normalise and store
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const uint32_t o_row = tmem + ((uint32_t)(q * 32) << 16) + COL_O;
    const float* lsum = reinterpret_cast<const float*>(smem + OFF_LSUM);
    int gt = 0;
    for (int i = 0; item_at(p, nq, i, it); ++i) {
      gt += it.qt + 1;
      const int b = i & 1;
      ptx::mbar_wait(l_ready(b), (i >> 1) & 1);
      float lsum_row = 0.f;
#pragma unroll
      for (int h = 0; h < SPLIT; ++h) lsum_row += lsum[(b * SPLIT + h) * BQ + row];
      const float inv = 1.f / lsum_row;
      ptx::mbar_wait(pv_done((gt - 1) & 1), ((gt - 1) >> 1) & 1);
      ptx::tc_fence_after();
      const int qi = it.qt * BQ + row;
      bf16* out = p.out + (size_t)(it.z * p.S + qi) * p.ldo + it.h * HD;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t r[32];
        ptx::tmem_ld32(o_row + c * 32, r);
        ptx::tmem_ld_wait();
        if (c == 3) {
          ptx::tc_fence_before();
          ptx::mbar_arrive(o_empty);  // O read: the next item's first PV may overwrite it
        }
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
  } else {
    // ===================== softmax: SPLIT column groups =====================
    const int half = (warp - 2) >> 2;  // column group: keys half*COLS .. +COLS of each tile
    const int q = warp & 3;            // TMEM lane quarter (shared by all groups)
    const int row = q * 32 + lane;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    float* red = reinterpret_cast<float*>(smem + OFF_RED);    // [slot][group][row]
    float* lsum = reinterpret_cast<float*>(smem + OFF_LSUM);  // [item&1][group][row]
    const uint32_t o_col = tmem + lane_base + COL_O + half * COLS;
    int gt = 0;  // S/P tiles consumed by this CTA
    for (int i = 0; item_at(p, nq, i, it); ++i) {
      const int q0 = it.qt * BQ, qi = q0 + row;
      const int nkv = it.qt + 1;
      float m_used = -INFINITY, l = 0.f;
      for (int j = 0; j < nkv; ++j, ++gt) {
        const int b = gt & 1;
        ptx::mbar_wait(s_full(b), (gt >> 1) & 1);
        ptx::tc_fence_after();
        if (threadIdx.x == 64) adbg(p, gt, 2);
        float v[COLS];
        {
          const uint32_t sc = tmem + lane_base + COL_S0 + b * 128 + half * COLS;
#pragma unroll
          for (int c0 = 0; c0 < COLS; c0 += 32) {
            uint32_t r0[32];
            ptx::tmem_ld32(sc + c0, r0);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int c = 0; c < 32; ++c) v[c0 + c] = __uint_as_float(r0[c]);  // raw scores
          }
        }
        const int key0 = j * BKV + half * COLS;
        if (key0 + COLS - 1 > q0) {  // reaches the diagonal: causal mask
#pragma unroll
          for (int c = 0; c < COLS; ++c)
            if (key0 + c > qi) v[c] = -INFINITY;
        }
        float mr[8];  // 8 independent max chains
#pragma unroll
        for (int k = 0; k < 8; ++k) mr[k] = v[k];
#pragma unroll
        for (int c = 8; c < COLS; ++c) mr[c & 7] = fmaxf(mr[c & 7], v[c]);
        float mraw = fmaxf(fmaxf(fmaxf(mr[0], mr[1]), fmaxf(mr[2], mr[3])),
                           fmaxf(fmaxf(mr[4], mr[5]), fmaxf(mr[6], mr[7])));
        // exchange the group row maxima (double-buffered slot: no WAR hazard)
        float* slot = red + b * SPLIT * BQ;
        slot[half * BQ + row] = mraw;
        softmax_bar<NSOFT>();
#pragma unroll
        for (int h = 0; h < SPLIT; ++h)
          if (h != half) mraw = fmaxf(mraw, slot[h * BQ + row]);
        const float mx = fmaxf(m_used, mraw * p.scale_log2);  // scale > 0: max commutes
        const bool need = mx > m_used + 8.f;                  // identical in every group
        if (j > 0 && __any_sync(0xffffffffu, need)) {
          // O settled: the previous tile's PV (and so every earlier PV) has completed
          ptx::mbar_wait(pv_done((gt - 1) & 1), ((gt - 1) >> 1) & 1);
          ptx::tc_fence_after();
          const float corr = need ? ptx::ex2(m_used - mx) : 1.f;
#pragma unroll 1
          for (int c = 0; c < COLS / 32; ++c) {
            uint32_t r[32];
            ptx::tmem_ld32(o_col + c * 32, r);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * corr);
            ptx::tmem_st32(o_col + c * 32, r);
          }
          ptx::tmem_st_wait();
          l *= corr;
        }
        if (need) m_used = mx;
        // P buffer b was last read by the PV of tile gt-2
        if (gt >= 2) ptx::mbar_wait(pv_done(b), ((gt - 2) >> 1) & 1);
        // P = 2^(s*scale - m) -> packed bf16 pairs, COLS / 2 TMEM columns per group
        // independent sum chains, two lanes per packed FADD2
        float2 ls2[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
        const float2 sc2 = make_float2(p.scale_log2, p.scale_log2), nm2 = make_float2(-m_used, -m_used);
        uint32_t pk[COLS / 2];
#pragma unroll
        for (int c = 0; c < COLS / 8; ++c) {
          float e[8];
#pragma unroll
          for (int k = 0; k < 8; k += 2) {
            const float2 a = ptx::ffma2(make_float2(v[c * 8 + k], v[c * 8 + k + 1]), sc2, nm2);
            e[k] = ptx::ex2(a.x);
            e[k + 1] = ptx::ex2(a.y);
            ls2[k >> 1] = ptx::fadd2(ls2[k >> 1], make_float2(e[k], e[k + 1]));
          }
          pk[4 * c + 0] = pack_bf16x2(e[0], e[1]);
          pk[4 * c + 1] = pack_bf16x2(e[2], e[3]);
          pk[4 * c + 2] = pack_bf16x2(e[4], e[5]);
          pk[4 * c + 3] = pack_bf16x2(e[6], e[7]);
        }
        ptx::tc_fence_after();
        if constexpr (COLS == 64)
          ptx::tmem_st32(tmem + lane_base + COL_P + b * 64 + half * 32, pk);
        else
          ptx::tmem_st16(tmem + lane_base + COL_P + b * 64 + half * 16, pk);
        l += ((ls2[0].x + ls2[0].y) + (ls2[1].x + ls2[1].y)) +
             ((ls2[2].x + ls2[2].y) + (ls2[3].x + ls2[3].y));
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        ptx::mbar_arrive(p_full(b));
        if (threadIdx.x == 64) adbg(p, gt, 3);
      }
      // hand the row sums to the epilogue warps (double-buffered by item: the
      // epilogue of item i has read them before item i+2's softmax can end)
      lsum[((i & 1) * SPLIT + half) * BQ + row] = l;
      ptx::mbar_arrive(l_ready(i & 1));
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}


// ---------------------------------------------------------------------------
// Two-query-tile ping-pong (the default).  A work item is a PAIR of adjacent
// query tiles of one head, A = qt - 1 and B = qt (A absent for the first tile
// of an odd tile count), sharing every K / V tile they both need.  Two softmax
// warpgroups, one per query tile, each thread owning one query row (all 128
// keys of a tile in registers), so one tile's softmax runs while the tensor
// core works for the other:
//   MMA order per key tile j:  PV_A(j), S_A(j+1), PV_B(j), S_B(j+1)
// S_X and P_X share TMEM columns (P packed bf16 in the first 64 columns of
// S_X): tcgen05.mma executes in issue order, so S_X(j+1) cannot overwrite P_X(j)
// before PV_X(j) has read it, and once S_X(j+1) has landed PV_X(j) — and every
// earlier MMA — is complete, so the softmax may rescale O_X without a wait.
// Warp roles (512 threads, one CTA per SM, registers rebalanced by setmaxnreg):
//   WG0   warp 0 TMA (Q_A, Q_B per item; K / V^T rings), warp 1 MMA issue
//   WG1   softmax of tile A       WG2   softmax of tile B
//   WG3   epilogue: O_X / l -> bf16 rows, off the softmax path
// TMEM columns: S_A/P_A [0,128), S_B/P_B [128,256), O_A [256,384), O_B [384,512).
namespace pp {
constexpr int KST = 2, VST = 2;
constexpr int OFF_Q = 0;  // Q_A, Q_B
constexpr int OFF_K = OFF_Q + 2 * TILE;
constexpr int OFF_V = OFF_K + KST * TILE;
constexpr int OFF_LSUM = OFF_V + VST * TILE;  // [tile X][item parity][128] row sums
constexpr int OFF_BAR = OFF_LSUM + 2 * 2 * BQ * 4;
// q_full[2] q_empty[2] k_full[KST] k_empty[KST] v_full[VST] v_empty[VST]
// s_full[2] p_full[2] o_full[2] o_empty[2] l_ready[2][2]
constexpr int N_BARS = 4 + 2 * KST + 2 * VST + 8 + 4;
constexpr int OFF_TMEM = OFF_BAR + N_BARS * 8;
constexpr int SMEM = OFF_TMEM + 16 + 1024;
constexpr int NTH = 512;
constexpr uint32_t COL_SX = 0, COL_OX = 256;  // + X * 128
}  // namespace pp

__device__ __forceinline__ void setmaxnreg_inc_176() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 176;" ::: "memory");
}
__device__ __forceinline__ void setmaxnreg_dec_112() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 112;" ::: "memory");
}
__device__ __forceinline__ void setmaxnreg_dec_48() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 48;" ::: "memory");
}

// pair item i of this CTA (snake rounds, heaviest pair first): hi tile qb,
// lo tile qb - 1 (< 0: absent)
__device__ __forceinline__ bool pair_at(const AttnParams& p, int nq, int round, Item& it) {
  const int G = gridDim.x;
  const int c = blockIdx.x;
  const int per = p.H * p.nseq;
  const int npair = (nq + 1) / 2;
  int idx;
  if (p.sched) {  // host LPT schedule: this CTA's items, heaviest first
    const int o0 = __ldg(p.sched + c), o1 = __ldg(p.sched + c + 1);
    if (round >= o1 - o0) return false;
    idx = __ldg(p.sched + G + 1 + o0 + round);
  } else {
    idx = round * G + ((round & 1) ? G - 1 - c : c);
    if (idx >= npair * per) return false;
  }
  const int k = idx / per, rem = idx - k * per;
  it.qt = nq - 1 - 2 * k;  // B
  it.h = rem % p.H;
  it.z = rem / p.H;
  return true;
}

__global__ void __launch_bounds__(pp::NTH, 1) attn_pp_kernel(const __grid_constant__ AttnParams p) {
  constexpr int KST = pp::KST, VST = pp::VST, OFF_Q = pp::OFF_Q, OFF_K = pp::OFF_K,
                OFF_V = pp::OFF_V, OFF_LSUM = pp::OFF_LSUM, OFF_BAR = pp::OFF_BAR,
                OFF_TMEM = pp::OFF_TMEM;
  constexpr uint32_t COL_SX = pp::COL_SX, COL_OX = pp::COL_OX;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sb = ptx::smem_u32(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t bars = sb + OFF_BAR;
  auto q_full = [&](int x) { return bars + 8u * x; };
  auto q_empty = [&](int x) { return bars + 8u * (2 + x); };
  auto k_full = [&](int s) { return bars + 8u * (4 + s); };
  auto k_empty = [&](int s) { return bars + 8u * (4 + KST + s); };
  auto v_full = [&](int s) { return bars + 8u * (4 + 2 * KST + s); };
  auto v_empty = [&](int s) { return bars + 8u * (4 + 2 * KST + VST + s); };
  constexpr int B0 = 4 + 2 * KST + 2 * VST;
  auto s_full = [&](int x) { return bars + 8u * (B0 + x); };
  auto p_full = [&](int x) { return bars + 8u * (B0 + 2 + x); };
  auto o_full = [&](int x) { return bars + 8u * (B0 + 4 + x); };
  auto o_empty = [&](int x) { return bars + 8u * (B0 + 6 + x); };
  auto l_ready = [&](int x, int b) { return bars + 8u * (B0 + 8 + 2 * x + b); };
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + OFF_TMEM);

  const int nq = (p.S + BQ - 1) / BQ;
  const int vld = (p.S + 63) & ~63;

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&p.q);
    ptx::prefetch_tmap(&p.vt);
    for (int x = 0; x < 2; ++x) {
      ptx::mbar_init(q_full(x), 1);
      ptx::mbar_init(q_empty(x), 1);
      ptx::mbar_init(s_full(x), 1);
      ptx::mbar_init(p_full(x), 128);
      ptx::mbar_init(o_full(x), 1);
      ptx::mbar_init(o_empty(x), 128);
      ptx::mbar_init(l_ready(x, 0), 128);
      ptx::mbar_init(l_ready(x, 1), 128);
    }
    for (int s = 0; s < KST; ++s) {
      ptx::mbar_init(k_full(s), 1);
      ptx::mbar_init(k_empty(s), 1);
    }
    for (int s = 0; s < VST; ++s) {
      ptx::mbar_init(v_full(s), 1);
      ptx::mbar_init(v_empty(s), 1);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc(ptx::smem_u32(tmem_holder), 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  ptx::pdl_begin();

  const int wg = warp >> 2;
  Item it;
  if (wg == 0) {
    setmaxnreg_dec_112();
    if (warp == 0 && lane == 0) {
      int kc = 0, vc = 0, nx[2] = {0, 0};
      for (int i = 0; pair_at(p, nq, i, it); ++i) {
        const int g = it.h / (p.H / p.KV);
        const int base = it.z * p.S;
        const int qc = it.h * HD, kcol = (p.H + g) * HD, vr = g * HD;
        for (int x = 0; x < 2; ++x) {
          const int qt = it.qt - 1 + x;
          if (qt < 0) continue;
          ptx::mbar_wait(q_empty(x), (nx[x] & 1) ^ 1);
          if (x == 1) pdbg(p, i, 0);
          ptx::mbar_expect_tx(q_full(x), TILE);
          const uint32_t qs = sb + OFF_Q + x * TILE;
          ptx::tma_load_2d(&p.q, qs, q_full(x), qc, base + qt * BQ);
          ptx::tma_load_2d(&p.q, qs + HALF, q_full(x), qc + 64, base + qt * BQ);
          ++nx[x];
        }
        for (int j = 0; j <= it.qt; ++j, ++kc, ++vc) {
          const int s = kc % KST, t = vc % VST;
          ptx::mbar_wait(k_empty(s), ((kc / KST) & 1) ^ 1);
          ptx::mbar_expect_tx(k_full(s), TILE);
          const uint32_t ks = sb + OFF_K + s * TILE;
          ptx::tma_load_2d(&p.q, ks, k_full(s), kcol, base + j * BKV);
          ptx::tma_load_2d(&p.q, ks + HALF, k_full(s), kcol + 64, base + j * BKV);
          ptx::mbar_wait(v_empty(t), ((vc / VST) & 1) ^ 1);
          ptx::mbar_expect_tx(v_full(t), TILE);
          const uint32_t vs = sb + OFF_V + t * TILE;
          ptx::tma_load_2d(&p.vt, vs, v_full(t), it.z * vld + j * BKV, vr);
          ptx::tma_load_2d(&p.vt, vs + HALF, v_full(t), it.z * vld + j * BKV + 64, vr);
        }
      }
    } else if (warp == 1 && lane == 0) {
      constexpr uint32_t IDESC = ptx::idesc_bf16(128, 128);
      int kc = 0, vc = 0;
      int ns[2] = {0, 0}, np[2] = {0, 0}, ni[2] = {0, 0};  // S, PV, items per tile X
      auto issue_s = [&](int x, uint32_t ks) {
        const uint32_t qs = sb + OFF_Q + x * TILE;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off = (kk >> 2) * HALF;
          ptx::mma_bf16(tmem + COL_SX + x * 128, ptx::desc_sw128(qs + off) + 2 * (kk & 3),
                        ptx::desc_sw128(ks + off) + 2 * (kk & 3), IDESC, kk > 0);
        }
        ptx::mma_commit(s_full(x));
        ++ns[x];
      };
      auto issue_pv = [&](int x, uint32_t vs, bool acc) {
#pragma unroll
        for (int kk = 0; kk < BKV / 16; ++kk) {
          const uint32_t off = (kk >> 2) * HALF;
          ptx::mma_bf16_ts(tmem + COL_OX + x * 128, tmem + COL_SX + x * 128 + kk * 8,
                           ptx::desc_sw128(vs + off) + 2 * (kk & 3), IDESC, acc || kk != 0);
        }
        ++np[x];
      };
      // S_A(0) of an item is issued during the previous item's last step (it
      // needs only Q_A and K_0 of the new item, both loaded by then), so softmax
      // A starts the new item while softmax B finishes the old one
      bool a_pre = false;
      static_assert(KST >= 2, "the next item's K_0 needs a free K slot");
      const bool pre_ok = p.variant != 3;  // 3: no cross-item S_A(0) (A/B diagnostic)
      for (int i = 0; pair_at(p, nq, i, it); ++i) {
        const int nb = it.qt + 1, na = it.qt;  // key tiles of B and A (A absent: 0)
        pdbg(p, i, 1);
        // S_A(0), S_B(0) from K_0
        {
          const int s = kc % KST;
          ptx::mbar_wait(k_full(s), (kc / KST) & 1);
          const uint32_t ks = sb + OFF_K + s * TILE;
          if (na > 0 && !a_pre) {
            ptx::mbar_wait(q_full(0), ni[0] & 1);
            ptx::tc_fence_after();
            issue_s(0, ks);
            if (na == 1) ptx::mma_commit(q_empty(0));
          }
          a_pre = false;
          ptx::mbar_wait(q_full(1), ni[1] & 1);
          ptx::tc_fence_after();
          issue_s(1, ks);
          if (nb == 1) ptx::mma_commit(q_empty(1));
          ptx::mma_commit(k_empty(s));
          ++kc;
          pdbg(p, i, 2);
        }
        for (int j = 0; j < nb; ++j) {
          const int t = vc % VST;
          const uint32_t vs = sb + OFF_V + t * TILE;
          ptx::mbar_wait(v_full(t), (vc / VST) & 1);
          const bool more = j + 1 < nb;
          const int s = kc % KST;
          const uint32_t ks = sb + OFF_K + s * TILE;
          if (j < na) {
            ptx::mbar_wait(p_full(0), np[0] & 1);
            if (j == 0 && ni[0] > 0) ptx::mbar_wait(o_empty(0), (ni[0] - 1) & 1);
            ptx::tc_fence_after();
            issue_pv(0, vs, j > 0);
            if (j == 0) pdbg(p, i, 3);
            if (j == na - 1) ptx::mma_commit(o_full(0));
            if (j + 1 < na) {
              ptx::mbar_wait(k_full(s), (kc / KST) & 1);
              ptx::tc_fence_after();
              issue_s(0, ks);
              if (j + 1 == na - 1) ptx::mma_commit(q_empty(0));
            }
          }
          if (!more && pre_ok) {
            Item nx;
            if (pair_at(p, nq, i + 1, nx) && nx.qt > 0) {  // next item's S_A(0)
              const int s2 = kc % KST;
              ptx::mbar_wait(k_full(s2), (kc / KST) & 1);
              ptx::mbar_wait(q_full(0), (ni[0] + (na > 0 ? 1 : 0)) & 1);
              ptx::tc_fence_after();
              issue_s(0, sb + OFF_K + s2 * TILE);
              if (nx.qt == 1) ptx::mma_commit(q_empty(0));
              a_pre = true;
            }
          }
          ptx::mbar_wait(p_full(1), np[1] & 1);
          if (j == 0 && ni[1] > 0) ptx::mbar_wait(o_empty(1), (ni[1] - 1) & 1);
          ptx::tc_fence_after();
          issue_pv(1, vs, j > 0);
          ptx::mma_commit(v_empty(t));
          ++vc;
          if (!more) {
            ptx::mma_commit(o_full(1));
            pdbg(p, i, 6);
          }
          if (more) {
            ptx::mbar_wait(k_full(s), (kc / KST) & 1);
            ptx::tc_fence_after();
            issue_s(1, ks);
            if (j + 1 == nb - 1) ptx::mma_commit(q_empty(1));
            ptx::mma_commit(k_empty(s));
            ++kc;
          }
        }
        if (na > 0) ++ni[0];
        ++ni[1];
      }
    }
    __syncwarp();
  } else if (wg == 3) {
    // ===================== epilogue: O_X / l -> bf16 =====================
    setmaxnreg_dec_48();
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const float* lsum = reinterpret_cast<const float*>(smem + OFF_LSUM);
    int ni[2] = {0, 0};
    for (int i = 0; pair_at(p, nq, i, it); ++i) {
      for (int x = 0; x < 2; ++x) {
        const int qt = it.qt - 1 + x;
        if (qt < 0) continue;
        const int b = ni[x] & 1;
        ptx::mbar_wait(l_ready(x, b), (ni[x] >> 1) & 1);
        const float inv = 1.f / lsum[(x * 2 + b) * BQ + row];
        ptx::mbar_wait(o_full(x), ni[x] & 1);
        ptx::tc_fence_after();
        ++ni[x];
        const int qi = qt * BQ + row;
        const uint32_t o_row = tmem + ((uint32_t)(q * 32) << 16) + COL_OX + x * 128;
        bf16* out = p.out + (size_t)(it.z * p.S + qi) * p.ldo + it.h * HD;
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          uint32_t r[32];
          ptx::tmem_ld32(o_row + c * 32, r);
          ptx::tmem_ld_wait();
          if (c == 3) {
            ptx::tc_fence_before();
            ptx::mbar_arrive(o_empty(x));
            if (x == 1 && threadIdx.x == 3 * 128) pdbg(p, i, 7);
          }
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
  } else {
    // ===================== softmax of tile X (WG1: A, WG2: B) =====================
    setmaxnreg_inc_176();
    const int x = wg - 1;
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    const uint32_t s_col = tmem + lane_base + COL_SX + x * 128;
    const uint32_t o_col = tmem + lane_base + COL_OX + x * 128;
    float* lsum = reinterpret_cast<float*>(smem + OFF_LSUM);
    int gt = 0, ni = 0;
    for (int i = 0; pair_at(p, nq, i, it); ++i) {
      const int qt = it.qt - 1 + x;
      if (qt < 0) continue;
      const int q0 = qt * BQ, qi = q0 + row;
      const int nkv = qt + 1;
      float m_used = -INFINITY, l = 0.f;
      for (int j = 0; j < nkv; ++j, ++gt) {
        ptx::mbar_wait(s_full(x), gt & 1);
        ptx::tc_fence_after();
        if (x == 1 && j == 0 && threadIdx.x == 2 * 128) pdbg(p, i, 4);
        // all 128 scores of the row in registers (one TMEM round trip)
        const bool diag = j == qt;  // the diagonal tile: causal mask key > qi
        const int kq = qi - j * BKV;
        float v[128];
#pragma unroll
        for (int c0 = 0; c0 < 128; c0 += 32) {
          uint32_t r0[32];
          ptx::tmem_ld32(s_col + c0, r0);
#pragma unroll
          for (int c = 0; c < 32; ++c) v[c0 + c] = __uint_as_float(r0[c]);
        }
        ptx::tmem_ld_wait();
        if (diag) {
#pragma unroll
          for (int c = 0; c < 128; ++c)
            if (c > kq) v[c] = -INFINITY;
        }
        // row max with three-input FMNMX3: 63 instructions instead of 127
        float mr[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) mr[k] = v[k];
#pragma unroll
        for (int c = 8; c < 120; c += 2) mr[(c >> 1) & 7] = ptx::fmax3(mr[(c >> 1) & 7], v[c], v[c + 1]);
        mr[0] = ptx::fmax3(mr[0], v[120], v[121]);
        mr[1] = ptx::fmax3(mr[1], v[122], v[123]);
        mr[2] = ptx::fmax3(mr[2], v[124], v[125]);
        mr[3] = ptx::fmax3(mr[3], v[126], v[127]);
        const float mraw = ptx::fmax3(ptx::fmax3(mr[0], mr[1], mr[2]), ptx::fmax3(mr[3], mr[4], mr[5]),
                                      fmaxf(mr[6], mr[7]));
        const float mx = fmaxf(m_used, mraw * p.scale_log2);
        const bool need = mx > m_used + 8.f;
        if (j > 0 && __any_sync(0xffffffffu, need)) {
          // O_X settled: S_X(j) was issued after PV_X(j-1) (in-order tensor pipe)
          const float corr = need ? ptx::ex2(m_used - mx) : 1.f;
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            uint32_t r[32];
            ptx::tmem_ld32(o_col + c * 32, r);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * corr);
            ptx::tmem_st32(o_col + c * 32, r);
          }
          l *= corr;
        }
        if (need) m_used = mx;
        // P = 2^(s*scale - m) -> packed bf16 pairs over the first 64 columns of
        // S_X; chunk c lands on columns [16c, 16c+16), whose scores are in
        // registers already (masked scores are -inf: 2^-inf = 0)
        float2 ls2[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
        const float2 sc2 = make_float2(p.scale_log2, p.scale_log2), nm2 = make_float2(-m_used, -m_used);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t pk[16];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            float e[8];
#pragma unroll
            for (int k = 0; k < 8; k += 2) {
              const float2 a = ptx::ffma2(make_float2(v[c * 32 + u * 8 + k], v[c * 32 + u * 8 + k + 1]), sc2, nm2);
              e[k] = ptx::ex2(a.x);
              e[k + 1] = ptx::ex2(a.y);
              ls2[k >> 1] = ptx::fadd2(ls2[k >> 1], make_float2(e[k], e[k + 1]));
            }
            pk[4 * u + 0] = pack_bf16x2(e[0], e[1]);
            pk[4 * u + 1] = pack_bf16x2(e[2], e[3]);
            pk[4 * u + 2] = pack_bf16x2(e[4], e[5]);
            pk[4 * u + 3] = pack_bf16x2(e[6], e[7]);
          }
          ptx::tmem_st16(s_col + c * 16, pk);
        }
        l += ((ls2[0].x + ls2[0].y) + (ls2[1].x + ls2[1].y)) +
             ((ls2[2].x + ls2[2].y) + (ls2[3].x + ls2[3].y));
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        ptx::mbar_arrive(p_full(x));
        if (x == 1 && j == 0 && threadIdx.x == 2 * 128) pdbg(p, i, 5);
      }
      lsum[(x * 2 + (ni & 1)) * BQ + row] = l;
      ptx::mbar_arrive(l_ready(x, ni & 1));
      ++ni;
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

template <int SPLIT>
static cudaError_t attn_set_attr() {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_tc_kernel<SPLIT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         ACfg<SPLIT>::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  return cudaSuccess;
}

// SPLIT = 2 (8 softmax warps).  SPLIT = 4 (16 warps, 32 keys per thread)
// compiles and is parity-clean but measured slower (13B S = 2048: 68 vs 61
// us; S = 8192: 775 vs 735 us, tools/attn_bench.py): the per-tile softmax is
// not latency-hidden by more warps — the extra row-max exchange and barrier
// of 512 threads cost more than they hide.
// Longest-processing-time schedule of the pair items over the grid: items
// (numbered as pair_at's snake order: k = idx / (H nseq) the pair rank,
// heaviest first) cost their key-tile steps (qt + 1 for B, qt for A) plus ~3
// steps of per-item fill / drain (tools/attn_pp_trace.py: 13B S = 2048 items
// take ~1.4 us per step plus ~3 us at the item boundary); each goes to the
// CTA with the least load so far, so every CTA's list stays heaviest first.
// The static snake order left the last CTA ~15 % behind the mean at S =
// 2048.  One table per (S, H, nseq, grid, device), built once and kept.
static const int* attn_schedule(int nq, int per, int grid) {
  struct Key {
    int nq, per, grid, dev;
    bool operator<(const Key& o) const {
      return nq != o.nq ? nq < o.nq : per != o.per ? per < o.per : grid != o.grid ? grid < o.grid : dev < o.dev;
    }
  };
  static std::mutex mu;
  static std::map<Key, int*> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  const Key key{nq, per, grid, dev};
  auto f = cache.find(key);
  if (f != cache.end()) return f->second;
  const int npair = (nq + 1) / 2, n = npair * per;
  std::vector<std::vector<int>> lists(grid);
  std::vector<long> load(grid, 0);
  // min-heap of (load, cta): ties to the lower CTA index
  std::priority_queue<std::pair<long, int>, std::vector<std::pair<long, int>>,
                      std::greater<std::pair<long, int>>> heap;
  for (int c = 0; c < grid; ++c) heap.push({0, c});
  for (int idx = 0; idx < n; ++idx) {  // already heaviest first
    const int qt = nq - 1 - 2 * (idx / per);
    const long cost = (qt + 1) + qt + 3;
    auto top = heap.top();
    heap.pop();
    lists[top.second].push_back(idx);
    heap.push({top.first + cost, top.second});
  }
  std::vector<int> h(grid + 1 + n);
  int o = 0;
  for (int c = 0; c < grid; ++c) {
    h[c] = o;
    for (int idx : lists[c]) h[grid + 1 + o++] = idx;
  }
  h[grid] = o;
  // may run while the caller's stream is being captured into a CUDA graph:
  // relaxed capture mode for this thread, and the upload on a private
  // non-blocking stream (never the capturing one, never the legacy stream)
  cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
  cudaThreadExchangeStreamCaptureMode(&mode);
  int* d = nullptr;
  cudaStream_t up = nullptr;
  bool ok = cudaMalloc(&d, h.size() * sizeof(int)) == cudaSuccess &&
            cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking) == cudaSuccess &&
            cudaMemcpyAsync(d, h.data(), h.size() * sizeof(int), cudaMemcpyHostToDevice, up) ==
                cudaSuccess &&
            cudaStreamSynchronize(up) == cudaSuccess;
  if (up) cudaStreamDestroy(up);
  cudaThreadExchangeStreamCaptureMode(&mode);
  if (!ok) {
    cudaGetLastError();
    if (d) cudaFree(d);
    return nullptr;  // the kernel falls back to the snake order
  }
  cache[key] = d;
  return d;
}

static cudaError_t attn_pp_launch(const AttnParams& p0, cudaStream_t s, int grid) {
  AttnParams p = p0;
  static const bool lpt_off = [] {
    const char* e = getenv("TIDAL_ATTN_LPT");
    return e && e[0] == '0';
  }();
  p.sched = lpt_off ? nullptr : attn_schedule((p.S + BQ - 1) / BQ, p.H * p.nseq, grid);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_pp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         pp::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  return launch_kt("attn", attn_pp_kernel, dim3(grid), dim3(pp::NTH), pp::SMEM, s, 1, p);
}

cudaError_t attn_tc_launch(const AttnParams& p, cudaStream_t s) {
  constexpr int split = 2;
  cudaError_t ea = attn_set_attr<split>();
  if (ea != cudaSuccess) return ea;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) sms = 148;
  }
  // TIDAL_ATTN=1 / 2 / 3: force single tiles / pairs / pairs without the
  // cross-item S_A(0) (A/B; with TIDAL_ATTN_TRACE, 2 and 3 trace the paired kernel)
  const char* fe = getenv("TIDAL_ATTN");  // read per launch: tests switch it
  const int forced = fe ? atoi(fe) : 0;
  const int variant = p.variant ? p.variant : forced;
  // pairs of query tiles unless there are too few pairs to fill the SMs about
  // 1.25 times (13B, H = 40, tools/attn_bench.py: paired 22.6 / 28.2 / 59.9 /
  // 175 / 638 us against single 20.0 / 32.0 / 64.6 / 205 / 764 us at S = 867 /
  // 1154 / 2048 / 4096 / 8192 — 160 pairs on 148 SMs quantise badly)
  const long pairs = (long)((p.S + BQ - 1) / BQ + 1) / 2 * p.H * p.nseq;
  if (variant == 2 || variant == 3 || (!p.dbg && variant == 0 && 4 * pairs >= 5L * sms)) {
    AttnParams q = p;
    q.variant = variant;  // 3: pairs without the cross-item S_A(0) (A/B)
    return attn_pp_launch(q, s, (int)(pairs < sms ? pairs : sms));
  }
  const long items = (long)((p.S + BQ - 1) / BQ) * p.H * p.nseq;  // persistent: <= one CTA per SM
  const int grid = (int)(items < sms ? items : sms);
  if (grid <= 0) return cudaSuccess;
  return launch_kt("attn", attn_tc_kernel<split>, dim3(grid), dim3(ACfg<split>::NTH),
                   ACfg<split>::SMEM, s, 1, p);
}

}  // namespace tidal
