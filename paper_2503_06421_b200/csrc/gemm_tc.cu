// gemm_tc.cu — the dense contractions of the prefill (QKV, O, gate/up, down)
// on 5th-gen tensor cores: tcgen05.mma with TMEM accumulators, operands staged
// by TMA (SWIZZLE_128B) through a 4-stage mbarrier ring, warp-specialised
// persistent CTAs:
//   warp 0      TMA producer (one elected lane)
//   warp 1      TMEM allocator + MMA issuer (one elected lane)
//   warps 2..5  epilogue: tcgen05.ld -> fused op -> smem transpose -> coalesced st.global
// CG = 2 (the default for M > 128): a CTA pair on the two SMs of a TPC runs
// one 256 x BN tile with tcgen05.mma.cta_group::2 — each CTA stages its 128
// rows of A and its BN/2 rows of B, so per-SM shared-memory operand traffic
// halves; the leader CTA issues the MMA and commits to both CTAs' barriers.
// Two accumulators in TMEM let tile i's epilogue overlap tile i+1's mainloop.
// The LoRA delta of a targeted projection is folded in as a K-extension:
// x W^T + (s x A^T) B^T = [x | T] [W | B]^T, i.e. ceil(r/16) extra UMMA
// K-steps reading T [M, r] and lora_B [n, r] (zero-filled by TMA beyond r).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <mutex>

#include "kernels.h"
#include "launch.cuh"
#include "ptx.cuh"
#include "ptx2.cuh"

namespace tidal {

namespace {

constexpr int BM = GEMM_BM, BN = GEMM_BN, BK = GEMM_BK;
constexpr int A_BYTES = BM * BK * 2;          // 16 KB
constexpr int ROW_BYTES = BK * 2;             // one 64-element K row = 128 B
constexpr int STG_ROW = 144;                  // staging row stride (bytes)
constexpr int STG_WARP = 32 * STG_ROW;
constexpr int SMEM_LIMIT = 227 * 1024;        // max dynamic shared memory per CTA
constexpr int TMEM_COLS = 512;

// Shared-memory layout of one instantiation: a stage holds this CTA's A box
// (128 rows) and its B rows (BNX / CG), so the ring is as deep as 227 KB
// allows (4..8 stages): a CTA-pair 256 x 192 tile streams 28 KB per K-block
// and gets 7 stages (~1.6 us of L2/DRAM latency cover at full MMA rate).
template <int EPI, int BNT, int CG>
struct Cfg {
  static constexpr int BNX = EPI == EPI_SILU ? 256 : BNT;  // MMA N = accumulator columns
  static constexpr int BROWS = BNX / CG;                   // B rows staged by this CTA
  static constexpr int BBYTES = BROWS * ROW_BYTES;
  static constexpr int STAGE = A_BYTES + BBYTES;
  static constexpr int FIXED = 4 * STG_WARP + 16 * 8 + 8 * 4 + 16 + 1024;
  static constexpr int ST_RAW = (SMEM_LIMIT - FIXED) / STAGE;
  static constexpr int STAGES = ST_RAW > 8 ? 8 : ST_RAW;
  static constexpr int OFF_A = 0;
  static constexpr int OFF_B = OFF_A + STAGES * A_BYTES;
  static constexpr int OFF_STG = OFF_B + STAGES * BBYTES;
  static constexpr int OFF_BAR = OFF_STG + 4 * STG_WARP;
  static constexpr int N_BARS = 2 * STAGES + 4;
  static constexpr int OFF_TMEM = OFF_BAR + N_BARS * 8;
  static constexpr int SMEM_BYTES = OFF_TMEM + 16 + 1024;  // + alignment slack
  static_assert(STAGES >= 4 && SMEM_BYTES <= SMEM_LIMIT, "GEMM shared-memory layout");
  static_assert(BBYTES % 1024 == 0, "SWIZZLE_128B stage alignment");
};
constexpr int NTHREADS = 192;

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// Store one 32-column chunk of this thread's row (bf16) via the warp's
// staging buffer so that global stores are row-contiguous.
__device__ __forceinline__ void store_chunk_bf16(const float (&v)[32], uint8_t* stg, int lane,
                                                 bf16* out, int ldo, int row0, int M, int col,
                                                 int nvalid) {
  uint4* st = reinterpret_cast<uint4*>(stg + lane * 80);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    uint4 w;
    w.x = pack_bf16x2(v[8 * k + 0], v[8 * k + 1]);
    w.y = pack_bf16x2(v[8 * k + 2], v[8 * k + 3]);
    w.z = pack_bf16x2(v[8 * k + 4], v[8 * k + 5]);
    w.w = pack_bf16x2(v[8 * k + 6], v[8 * k + 7]);
    st[k] = w;
  }
  __syncwarp();
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    const int r = it * 8 + (lane >> 2), ch = lane & 3;
    const int m = row0 + r;
    const int c = ch * 8;
    if (m < M && c < nvalid) {
      uint4 w = *reinterpret_cast<const uint4*>(stg + r * 80 + ch * 16);
      bf16* dst = out + (size_t)m * ldo + col + c;
      if (c + 8 <= nvalid) {
        *reinterpret_cast<uint4*>(dst) = w;
      } else {
        const bf16* src = reinterpret_cast<const bf16*>(stg + r * 80 + ch * 16);
        for (int e = 0; e < nvalid - c; ++e) dst[e] = src[e];
      }
    }
  }
  __syncwarp();
}

__device__ __forceinline__ void red_add_f32x4(float* dst, float4 a) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(a.x), "f"(a.y),
               "f"(a.z), "f"(a.w)
               : "memory");
}

// out[m, col + j] += v[j]  (fp32 residual), coalesced through staging, as
// L2 reductions (red.global.add.v4.f32): no load round trip in the epilogue.
// One writer per element at a time (split-K parts are ordered by flags), so
// the sum order is fixed and the result deterministic.
__device__ __forceinline__ void add_chunk_f32(const float (&v)[32], uint8_t* stg, int lane,
                                              float* out, int ldo, int row0, int M, int col,
                                              int nvalid) {
  float4* st = reinterpret_cast<float4*>(stg + lane * STG_ROW);
#pragma unroll
  for (int k = 0; k < 8; ++k) st[k] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
  __syncwarp();
  const int ch = lane & 7, c = ch * 4;
#pragma unroll
  for (int it = 0; it < 8; ++it) {
    const int r = it * 4 + (lane >> 3);
    const int m = row0 + r;
    if (m < M && c < nvalid) {
      const float4 a = *reinterpret_cast<const float4*>(stg + r * STG_ROW + ch * 16);
      float* dst = out + (size_t)m * ldo + col + c;
      if (c + 4 <= nvalid) {
        red_add_f32x4(dst, a);
      } else {
        // ragged tail: scalars straight from staging (no local copy of `a`)
        const float* sa = reinterpret_cast<const float*>(stg + r * STG_ROW + ch * 16);
        for (int e = 0; e < nvalid - c; ++e) atomicAdd(dst + e, sa[e]);
      }
    }
  }
  __syncwarp();
}

// out[m, col + j] = v[j]  (fp32 split-K partial), coalesced through staging.
__device__ __forceinline__ void store_chunk_f32(const float (&v)[32], uint8_t* stg, int lane,
                                                float* out, int ldo, int row0, int M, int col,
                                                int nvalid) {
  float4* st = reinterpret_cast<float4*>(stg + lane * STG_ROW);
#pragma unroll
  for (int k = 0; k < 8; ++k) st[k] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
  __syncwarp();
  const int ch = lane & 7, c = ch * 4;
#pragma unroll
  for (int it = 0; it < 8; ++it) {
    const int r = it * 4 + (lane >> 3);
    const int m = row0 + r;
    if (m < M && c < nvalid) {
      const float4 a = *reinterpret_cast<const float4*>(stg + r * STG_ROW + ch * 16);
      float* dst = out + (size_t)m * ldo + col + c;
      if (c + 4 <= nvalid) {
        *reinterpret_cast<float4*>(dst) = a;
      } else {
        const float* s = reinterpret_cast<const float*>(stg + r * STG_ROW + ch * 16);
        for (int e = 0; e < nvalid - c; ++e) dst[e] = s[e];
      }
    }
  }
  __syncwarp();
}

__device__ __forceinline__ void ld_chunk(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  ptx::tmem_ld32(taddr, r);
  ptx::tmem_ld_wait();
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// tile -> (segment, first output column within the segment, first row of the
// cluster tile).  Cluster tiles are n-major so concurrently running tiles share
// the same weight panel (read from HBM once, then from L2).
template <int EPI, int BNT, int CG, int MC>
__device__ __forceinline__ void decode_tile(const GemmParams& p, int tile, int& seg, int& n0,
                                            int& m0) {
  if (EPI == EPI_PARTIAL) {  // tile = ks * m_tiles + m
    seg = 0;
    n0 = 0;
    m0 = (tile % p.m_tiles) * BM;
    return;
  }
  int gn = tile / p.m_tiles;
  m0 = (tile - gn * p.m_tiles) * (BM * CG * MC);  // cluster tile: MC pairs stacked in M
  seg = 0;
  while (seg < p.nseg - 1 && gn >= p.n_tiles[seg]) {
    gn -= p.n_tiles[seg];
    ++seg;
  }
  n0 = gn * (EPI == EPI_SILU ? 128 : BNT);
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// diagnostic timeline (GemmParams::dbg, null in production): per CTA and work
// item, 8 slots: 0 producer start, 1 flag-wait end, 2 first MMA, 3 last commit,
// 4 epilogue start, 5 epilogue end, 6 work id, 7 is_t
constexpr int DBG_ITEMS = 32;
__device__ __forceinline__ void dbg_put(unsigned long long* d, int it, int slot, unsigned long long v) {
  if (d && it < DBG_ITEMS) d[((size_t)blockIdx.x * DBG_ITEMS + it) * 8 + slot] = v;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// One unit of persistent work: a tile, or (EPI_RESID split-K) one K range of
// a tile.  Work w = split * total_tiles + tile, so every split-s part of a
// tile is scheduled after its split-(s-1) part on any CTA (no circular wait).
struct Work {
  int seg, n0, m0;  // m0: first row of this CTA pair
  int kb0, kb1;     // main-loop K blocks [kb0, kb1)
  int lora;         // LoRA K-extension blocks follow (last split only)
  int split, tile;
  int ks;           // split-K parts of this work's tile (1: whole tile)
  int is_t;         // in-GEMM LoRA shrink tile (T = s A lora_A^T for this pair's rows)
};

template <int EPI, int BNT, int CG, int MC>
__device__ __forceinline__ Work decode_work(const GemmParams& p, int w, int pr, int nk,
                                            int nlora) {
  Work r;
  if (EPI == EPI_PARTIAL) {  // w = ks * m_tiles + m
    r.seg = 0;
    r.n0 = 0;
    r.m0 = (w % p.m_tiles) * BM;
    r.kb0 = (w / p.m_tiles) * p.kblocks_per_split;
    r.kb1 = min(nk, r.kb0 + p.kblocks_per_split);
    r.lora = 0;
    r.split = 0;
    r.tile = w;
    r.ks = 1;
    r.is_t = 0;
    return r;
  }
  if (w < 0) {  // T work -w - 1 (see item_work: first on the least loaded units)
    // T tile j in t_ks parts (the K ranges of this GEMM's split-K parts)
    const int tw = -w - 1, tks = p.t_ks > 1 ? p.t_ks : 1;
    const int j = tw / tks;
    r.is_t = 1;
    r.seg = 0;
    r.n0 = 0;
    r.m0 = j * (BM * CG * MC) + pr * BM * CG;
    r.split = tw - j * tks;
    r.ks = tks;
    const int kps = tks > 1 ? p.kblocks_per_split : nk;
    r.kb0 = r.split * kps;
    r.kb1 = min(nk, r.kb0 + kps);
    r.lora = 0;
    r.tile = j;
    return r;
  }
  r.is_t = 0;
  // EPI_RESID split-K: tiles [0, n_full) run whole, the tail tiles in ksplit
  // ordered parts (n_full = 0: every tile split); work = n_full + split * n_tail
  // + tail tile, so part s of a tile is always scheduled after its part s - 1
  int ks = EPI == EPI_RESID && p.ksplit > 1 ? p.ksplit : 1;
  if (ks > 1 && w < p.n_full) {
    ks = 1;
    r.split = 0;
    r.tile = w;
  } else if (ks > 1) {
    const int v = w - p.n_full, ntail = p.total_tiles - p.n_full;
    r.split = v / ntail;
    r.tile = p.n_full + (v - r.split * ntail);
  } else {
    r.split = 0;
    r.tile = w;
  }
  r.ks = ks;
  decode_tile<EPI, BNT, CG, MC>(p, r.tile, r.seg, r.n0, r.m0);
  r.m0 += pr * BM * CG;
  const int kps = ks > 1 ? p.kblocks_per_split : nk;
  r.kb0 = r.split * kps;
  r.kb1 = min(nk, r.kb0 + kps);
  r.lora = (nlora > 0 && p.seg[r.seg].lora && r.split == ks - 1) ? nlora : 0;
  return r;
}

// The i-th work of `unit` (returns false past the end).  T tiles (in-GEMM LoRA
// shrink) come first and go to the units that the round-robin leaves one work
// short (the last units), T tile j to unit nunits - 1 - j (mod nunits); then
// the unit's normal works unit, unit + nunits, ...  Every work a T tile's
// consumers wait for is thus the first work(s) of some unit.  T tiles are
// encoded as negative work ids (-j - 1) for decode_work.
__device__ __forceinline__ bool item_work(const GemmParams& p, int unit, int nunits, int nnorm,
                                          int i, int& w) {
  const int t0 = nunits - 1 - unit;  // this unit's first T work
  const int ntw = p.t_tiles * (p.t_ks > 1 ? p.t_ks : 1);
  const int nt = ntw > t0 ? (ntw - t0 + nunits - 1) / nunits : 0;
  if (i < nt) {
    w = -(t0 + i * nunits) - 1;
    return true;
  }
  w = unit + (i - nt) * nunits;
  return w < nnorm;
}

__device__ __forceinline__ void epi_bar() {  // the 4 epilogue warps of this CTA
  asm volatile("bar.sync 2, 128;" ::: "memory");
}

template <int EPI, int BNT, int CG, int MC>
__global__ void __launch_bounds__(NTHREADS, 1) gemm_tc_kernel(const __grid_constant__ GemmParams p) {
  static_assert(MC == 1 || CG == 2, "multicast clusters are built from CTA pairs");
  using C = Cfg<EPI, BNT, CG>;
  constexpr int BNX = C::BNX, BROWS = C::BROWS, BBYTES = C::BBYTES, STAGES = C::STAGES;
  constexpr int OFF_A = C::OFF_A, OFF_B = C::OFF_B, OFF_STG = C::OFF_STG, OFF_BAR = C::OFF_BAR,
                OFF_TMEM = C::OFF_TMEM;
  constexpr int SILU_LORA_ROWS = 128 / CG;          // per-CTA rows of a gate/up LoRA-B box
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned (SWIZZLE_128B); offsetting smem_raw keeps the shared state
  // space visible to the compiler (STS/LDS, not generic ST/LD)
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sbase = ptx::smem_u32(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // cluster = MC CTA pairs (ranks 2p, 2p+1) stacked along M: they share every
  // B (weight) box, each CTA loading 1/MC of it and multicasting to the
  // same-rank CTA of every pair, so L2->SM operand traffic per MAC drops
  const int crank = CG == 2 ? (int)ptx::cluster_rank() : 0;
  const int rank = crank & 1;   // CTA within its pair
  const int pr = crank >> 1;    // pair within the cluster
  const int unit = (int)blockIdx.x / (CG * MC);
  const int nunits = (int)gridDim.x / (CG * MC);
  const uint16_t mc_mask = (uint16_t)((1u << rank) | (1u << (2 + rank)));
  const uint32_t bar0 = sbase + OFF_BAR;
  auto full_bar = [&](int s) { return bar0 + 8u * s; };
  auto empty_bar = [&](int s) { return bar0 + 8u * (STAGES + s); };
  auto tfull_bar = [&](int a) { return bar0 + 8u * (2 * STAGES + a); };
  auto tempty_bar = [&](int a) { return bar0 + 8u * (2 * STAGES + 2 + a); };
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + OFF_TMEM);

  const int nk = (p.K + BK - 1) / BK;
  const int nlora = p.lora_r > 0 ? (EPI == EPI_SILU ? 2 : 1) : 0;
  const int nwork = EPI == EPI_RESID && p.ksplit > 1
                        ? p.n_full + (p.total_tiles - p.n_full) * p.ksplit
                        : p.total_tiles;  // normal works (T tiles come on top)

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&p.a);
    for (int i = 0; i < 3; ++i)
      if (i < p.nseg || (EPI == EPI_SILU && i < 2)) ptx::prefetch_tmap(&p.b[i]);
    if (p.t_tiles) ptx::prefetch_tmap(&p.la);
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(full_bar(s), CG);  // leader expect_tx + peer arrive
      ptx::mbar_init(empty_bar(s), MC);  // one MMA commit per pair of the cluster
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(tfull_bar(a), 1);
      ptx::mbar_init(tempty_bar(a), 128 * CG);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) {
    if (CG == 2)
      ptx::tmem_alloc_pair(ptx::smem_u32(tmem_holder), TMEM_COLS);
    else
      ptx::tmem_alloc(ptx::smem_u32(tmem_holder), TMEM_COLS);
  }
  ptx::tc_fence_before();
  if (CG == 2)
    ptx::cluster_sync();
  else
    __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  ptx::pdl_begin();  // prologue above overlapped the previous kernel's tail

  if (warp == 0) {
    // ===================== TMA producer (both CTAs) =====================
    if (lane == 0) {
      auto tma = [&](const CUtensorMap* m, uint32_t dst, uint32_t fb, int c0, int c1) {
        if (CG == 2)
          ptx::tma_load_2d_pair(m, dst, fb, c0, c1);
        else
          ptx::tma_load_2d(m, dst, fb, c0, c1);
      };
      // B-side box of `rows` rows at (c0, r0) into dst: with MC pairs, this CTA
      // loads its 1/MC slice and multicasts it to the same-rank CTA of each pair
      auto tmab = [&](const CUtensorMap* m, uint32_t dst, uint32_t fb, int c0, int r0, int rows) {
        if (MC == 1) {
          tma(m, dst, fb, c0, r0);
        } else {
          const int part = rows / MC;
          ptx::tma_load_2d_pair_mc(m, dst + pr * part * ROW_BYTES, fb, c0, r0 + pr * part, mc_mask);
        }
      };
      int stage = 0;
      uint32_t phase = 0;
      bool t_ready = false;  // this CTA has seen every T row block published
      int w;
      for (int it = 0; item_work(p, unit, nunits, nwork, it, w); ++it) {
        const Work wk = decode_work<EPI, BNT, CG, MC>(p, w, pr, nk, nlora);
        const int seg = wk.seg, n0 = wk.n0;
        const int ma = wk.m0 + rank * BM;  // this CTA's A rows
        dbg_put(p.dbg, it, 0, gtimer());
        dbg_put(p.dbg, it, 6, (unsigned long long)(long long)w);
        dbg_put(p.dbg, it, 7, wk.is_t);
        const int nkb = wk.kb1 + wk.lora;
        if (EPI != EPI_PARTIAL && wk.is_t) {
          // T tile: this CTA stages its 128 rows of A and its t_rt_pad / CG rows of
          // the stacked [lora_A_0; lora_A_1; ...], packed K-block-major by
          // lora_pack_kernel so a stage's rows are one contiguous box (padding
          // rows are stale bytes: their accumulator columns are never read)
          const int half = p.t_rt_pad / CG;
          for (int kb = wk.kb0; kb < wk.kb1; ++kb) {
            ptx::mbar_wait(empty_bar(stage), phase ^ 1);
            const uint32_t sa = sbase + OFF_A + stage * A_BYTES;
            const uint32_t sb = sbase + OFF_B + stage * BBYTES;
            const uint32_t fb = full_bar(stage);
            if (rank == 0)
              ptx::mbar_expect_tx(fb, (A_BYTES + half * ROW_BYTES) * CG);
            else
              ptx::mbar_arrive_leader(fb);
            tma(&p.a, sa, fb, kb * BK, ma);
            tma(&p.la, sb, fb, 0, kb * p.t_rt_pad + rank * half);
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
          continue;
        }
        for (int kb = wk.kb0; kb < nkb; ++kb) {
          if (EPI != EPI_PARTIAL && p.t_tiles > 0 && kb == wk.kb1 && !t_ready) {
            // the LoRA K-extension reads T: wait (once per CTA) until every T
            // row block of this launch is published (they run concurrently,
            // first on their units, so one wait costs no more than a per-row one)
            uint32_t n = 0;
            while (ld_acquire(p.t_flags) < p.t_tiles * CG)
              if (++n == (1u << 30)) __trap();
            asm volatile("fence.proxy.async.global;" ::: "memory");
            t_ready = true;
            dbg_put(p.dbg, it, 1, gtimer());
          }
          ptx::mbar_wait(empty_bar(stage), phase ^ 1);
          const uint32_t sa = sbase + OFF_A + stage * A_BYTES;
          const uint32_t sb = sbase + OFF_B + stage * BBYTES;
          const uint32_t fb = full_bar(stage);
          int bytes;  // this CTA's bytes for the stage
          if (EPI == EPI_PARTIAL) {
            bytes = A_BYTES + p.nseg * p.src_rows * ROW_BYTES;
          } else if (kb < wk.kb1) {
            bytes = A_BYTES + BBYTES;
          } else {
            bytes = A_BYTES + (EPI == EPI_SILU ? SILU_LORA_ROWS : BROWS) * ROW_BYTES;
          }
          if (rank == 0)
            ptx::mbar_expect_tx(fb, bytes * CG);
          else
            ptx::mbar_arrive_leader(fb);
          if (EPI == EPI_PARTIAL) {
            tma(&p.a, sa, fb, kb * BK, ma);
            for (int s = 0; s < p.nseg; ++s)
              tma(&p.b[s], sb + s * p.src_rows * ROW_BYTES, fb, kb * BK, 0);
          } else if (kb < wk.kb1) {
            tma(&p.a, sa, fb, kb * BK, ma);
            if (EPI == EPI_SILU) {
              if (CG == 2) {
                tmab(&p.b[rank], sb, fb, kb * BK, n0, 128);  // rank 0: gate rows, rank 1: up rows
              } else {
                tma(&p.b[0], sb, fb, kb * BK, n0);
                tma(&p.b[1], sb + 128 * ROW_BYTES, fb, kb * BK, n0);
              }
            } else {
              tmab(&p.b[seg], sb, fb, kb * BK, n0 + rank * BROWS, BROWS);
            }
          } else {
            const int j = kb - wk.kb1;  // LoRA stage: EPI_SILU j=0 gate, j=1 up
            tma(&p.ta[EPI == EPI_SILU ? j : seg], sa, fb, 0, ma);
            if (EPI == EPI_SILU)
              tmab(&p.tb[j], sb, fb, 0, n0 + rank * SILU_LORA_ROWS, SILU_LORA_ROWS);
            else
              tmab(&p.tb[seg], sb, fb, 0, n0 + rank * BROWS, BROWS);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ===================== MMA issuer (leader CTA) =====================
    if (rank == 0) {  // whole warp: uniform control flow, one elected lane issues
      constexpr uint32_t IDESC = ptx::idesc_bf16(BM * CG, BNX);
      constexpr uint32_t IDESC_HALF = ptx::idesc_bf16(BM * CG, 128);
      const uint32_t IDESC_T = ptx::idesc_bf16(BM * CG, p.t_rt_pad > 0 ? p.t_rt_pad : 16);
      const int nmma_lora = (p.lora_r + 15) / 16;
      auto mma = [&](uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
        ptx::mma_bf16_ws<CG>(d, a, b, id, acc);
      };
      auto commit = [&](uint32_t bar) {  // this pair's two CTAs
        if (CG == 2)
          ptx::mma_commit_mask_ws(bar, (uint16_t)(3u << (2 * pr)));
        else
          ptx::mma_commit_ws(bar);
      };
      auto commit_stage = [&](uint32_t bar) {  // a stage slot is shared by all pairs
        if (MC == 2)
          ptx::mma_commit_mask_ws(bar, (uint16_t)0xF);
        else
          commit(bar);
      };
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int w;
      for (int it = 0; item_work(p, unit, nunits, nwork, it, w); ++it) {
        const Work wk = decode_work<EPI, BNT, CG, MC>(p, w, pr, nk, nlora);
        const int kb0 = wk.kb0, nkb = wk.kb1 + wk.lora;
        bool first_mma = true;
        ptx::mbar_wait(tempty_bar(acc), acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BNX;
        for (int kb = kb0; kb < nkb; ++kb) {
          ptx::mbar_wait(full_bar(stage), phase);
          ptx::tc_fence_after();
          if (first_mma && lane == 0) dbg_put(p.dbg, it, 2, gtimer());
          first_mma = false;
          const uint64_t adesc = ptx::desc_sw128(sbase + OFF_A + stage * A_BYTES);
          const uint64_t bdesc = ptx::desc_sw128(sbase + OFF_B + stage * BBYTES);
          if (EPI != EPI_PARTIAL && wk.is_t) {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              mma(d_tmem, adesc + 2 * k, bdesc + 2 * k, IDESC_T, ((kb - kb0) | k) != 0);
          } else if (EPI == EPI_PARTIAL || kb < wk.kb1) {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              mma(d_tmem, adesc + 2 * k, bdesc + 2 * k, IDESC, ((kb - kb0) | k) != 0);
          } else if (EPI == EPI_SILU) {
            const int j = kb - wk.kb1;
            for (int k = 0; k < nmma_lora; ++k)
              mma(d_tmem + j * 128, adesc + 2 * k, bdesc + 2 * k, IDESC_HALF, 1);
          } else {
            for (int k = 0; k < nmma_lora; ++k) mma(d_tmem, adesc + 2 * k, bdesc + 2 * k, IDESC, 1);
          }
          commit_stage(empty_bar(stage));
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        commit(tfull_bar(acc));
        if (lane == 0) dbg_put(p.dbg, it, 3, gtimer());
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
    __syncwarp();
  } else {
    // ===================== epilogue (warps 2..5, both CTAs) =====================
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    uint8_t* stg = smem + OFF_STG + (warp - 2) * STG_WARP;
    int acc = 0;
    uint32_t acc_phase = 0;
    int wi;
    for (int it = 0; item_work(p, unit, nunits, nwork, it, wi); ++it) {
      const Work wk = decode_work<EPI, BNT, CG, MC>(p, wi, pr, nk, nlora);
      const int tile = wk.tile, n0 = wk.n0, m0 = wk.m0;
      const GemmSeg sg = p.seg[wk.seg];
      ptx::mbar_wait(tfull_bar(acc), acc_phase);
      ptx::tc_fence_after();
      if (threadIdx.x == 64) dbg_put(p.dbg, it, 4, gtimer());
      const uint32_t tacc = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BNX;
      const int row0 = m0 + rank * BM + q * 32;
      const int m = row0 + lane;
      float v[32], w[32];
      if (EPI != EPI_PARTIAL && wk.is_t) {
        // T_t[m, j] = bf16(s * acc[m, t * r + j]); with t_ks K parts each part
        // leaves its fp32 partial in t_ws and the last to arrive sums all parts
        // in part order (deterministic) before rounding.  8-column groups never
        // straddle targets (r % 8 == 0); each thread owns one row.
        const int rt = p.t_nt * p.t_r, tks = wk.ks;
        const int prow = rank * BM + q * 32 + lane;  // row within the pair tile
        float* ws = p.t_ws + (size_t)(wk.tile * tks) * (BM * CG) * p.t_rt_pad;
        volatile int* bcast = reinterpret_cast<volatile int*>(smem + OFF_TMEM + 8);
        bool last = true;
        if (tks > 1) {
#pragma unroll 1
          for (int j = 0; j * 32 < rt; ++j) {
            ld_chunk(tacc + j * 32, v);
            float* dst = ws + ((size_t)wk.split * (BM * CG) + prow) * p.t_rt_pad + j * 32;
#pragma unroll
            for (int g = 0; g < 8; ++g)
              if (j * 32 + g * 4 < rt)
                *reinterpret_cast<float4*>(dst + g * 4) =
                    make_float4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3]);
          }
          __threadfence();
          epi_bar();
          if (threadIdx.x == 64) {
            const int old = atomicAdd(p.t_flags + 1 + wk.tile * CG + rank, 1);
            *bcast = old;
          }
          epi_bar();
          last = *bcast == tks - 1;
          if (last) __threadfence();  // acquire the other parts' partials
        }
        if (last) {
#pragma unroll 1
          for (int j = 0; j * 32 < rt; ++j) {
            if (tks > 1) {
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = 0.f;
              for (int s2 = 0; s2 < tks; ++s2) {
                const float* src = ws + ((size_t)s2 * (BM * CG) + prow) * p.t_rt_pad + j * 32;
#pragma unroll
                for (int g = 0; g < 8; ++g)
                  if (j * 32 + g * 4 < rt) {
                    const float4 a = __ldcg(reinterpret_cast<const float4*>(src + g * 4));
                    v[4 * g] += a.x;
                    v[4 * g + 1] += a.y;
                    v[4 * g + 2] += a.z;
                    v[4 * g + 3] += a.w;
                  }
              }
            } else {
              ld_chunk(tacc + j * 32, v);
            }
            if (m < p.M) {
#pragma unroll
              for (int g = 0; g < 4; ++g) {
                const int c0 = j * 32 + g * 8;
                if (c0 < rt) {
                  const int t = c0 / p.t_r;
                  uint4 o;
                  o.x = pack_bf16x2(p.t_scale * v[8 * g + 0], p.t_scale * v[8 * g + 1]);
                  o.y = pack_bf16x2(p.t_scale * v[8 * g + 2], p.t_scale * v[8 * g + 3]);
                  o.z = pack_bf16x2(p.t_scale * v[8 * g + 4], p.t_scale * v[8 * g + 5]);
                  o.w = pack_bf16x2(p.t_scale * v[8 * g + 6], p.t_scale * v[8 * g + 7]);
                  *reinterpret_cast<uint4*>(p.t_out[t] + (size_t)m * p.t_r + (c0 - t * p.t_r)) = o;
                }
              }
            }
          }
          // publish: T stores visible (generic and async proxy) before the count
          __threadfence();
          asm volatile("fence.proxy.async.global;" ::: "memory");
          epi_bar();
          if (threadIdx.x == 64) atomicAdd(p.t_flags, 1);
        }
      } else if (EPI == EPI_PARTIAL) {
        const int ks = tile / p.m_tiles;
        const int ncols = p.nseg * p.src_rows;
        float* out = reinterpret_cast<float*>(p.out) + (size_t)ks * p.M * p.ldo;
#pragma unroll 1
        for (int j = 0; j * 32 < ncols; ++j) {
          ld_chunk(tacc + j * 32, v);
          store_chunk_f32(v, stg, lane, out, p.ldo, row0, p.M, j * 32, ncols - j * 32);
        }
      } else if (EPI == EPI_SILU) {
        const int ncols = min(128, sg.n - n0);
#pragma unroll 1
        for (int j = 0; j < 4; ++j) {
          if (j * 32 >= ncols) break;
          ld_chunk(tacc + j * 32, v);          // gate
          ld_chunk(tacc + 128 + j * 32, w);    // up
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float g = v[i];
            v[i] = g * ptx::rcp(1.0f + ptx::ex2(-1.4426950408889634f * g)) * w[i];
          }
          store_chunk_bf16(v, stg, lane, reinterpret_cast<bf16*>(p.out), p.ldo, row0, p.M,
                           sg.out_col + n0 + j * 32, ncols - j * 32);
        }
      } else if (EPI == EPI_RESID) {
        const int ncols = min(BNT, sg.n - n0);
        const int ks = wk.ks;
        int* flag = ks > 1 ? p.flags + (tile * MC + pr) * CG + rank : nullptr;
        if (ks > 1 && wk.split > 0) {
          // split s adds after split s-1 of this tile half has landed
          if (threadIdx.x == 64) {
            uint32_t n = 0;
            while (ld_acquire(flag) != wk.split)
              if (++n == (1u << 30)) __trap();
          }
          epi_bar();
        }
#pragma unroll 1
        for (int j = 0; j < BNT / 32; ++j) {
          if (j * 32 >= ncols) break;
          ld_chunk(tacc + j * 32, v);
          add_chunk_f32(v, stg, lane, reinterpret_cast<float*>(p.out), p.ldo, row0, p.M,
                        sg.out_col + n0 + j * 32, ncols - j * 32);
        }
        if (ks > 1) {
          __threadfence();  // this thread's reductions are performed before the flag
          epi_bar();
          if (threadIdx.x == 64) st_release(flag, wk.split + 1 < ks ? wk.split + 1 : 0);
        }
      } else if (EPI == EPI_ROPE && sg.rope) {
        // rotate-half RoPE: the (cos, sin) of this row's position and a
        // 32-pair column block are loaded once and reused by every head of the
        // tile; the loads are issued before the TMEM reads so their latency
        // overlaps them (the table loads were the epilogue's main stall)
        const int hd = p.head_dim, half = hd >> 1;
        const int ncols = min(BNT, sg.n - n0);
        const int pos = p.seq_len ? m % p.seq_len : m;  // batched prompts restart at 0
        bf16* out = reinterpret_cast<bf16*>(p.out);
#pragma unroll 1
        for (int j = 0; j * 32 < half; ++j) {
          float2 cs[32];
          if (m < p.M) {
            const float2* src = p.rope + (size_t)pos * half + j * 32;
#pragma unroll
            for (int i = 0; i < 32; ++i) cs[i] = __ldg(src + i);
          }
#pragma unroll 1
          for (int h = 0; h * hd < ncols; ++h) {
            const int c1 = h * hd + j * 32, c2 = c1 + half;
            ld_chunk(tacc + c1, v);
            ld_chunk(tacc + c2, w);
            if (m < p.M) {
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                const float x1 = v[i], x2 = w[i];
                v[i] = x1 * cs[i].x - x2 * cs[i].y;
                w[i] = x2 * cs[i].x + x1 * cs[i].y;
              }
            }
            store_chunk_bf16(v, stg, lane, out, p.ldo, row0, p.M, sg.out_col + n0 + c1, 32);
            store_chunk_bf16(w, stg, lane, out, p.ldo, row0, p.M, sg.out_col + n0 + c2, 32);
            if (sg.out2) {
              store_chunk_bf16(v, stg, lane, sg.out2, sg.ldo2, row0, p.M, n0 + c1, 32);
              store_chunk_bf16(w, stg, lane, sg.out2, sg.ldo2, row0, p.M, n0 + c2, 32);
            }
          }
        }
      } else {
        const int ncols = min(BNT, sg.n - n0);
#pragma unroll 1
        for (int j = 0; j < BNT / 32; ++j) {
          if (j * 32 >= ncols) break;
          ld_chunk(tacc + j * 32, v);
          store_chunk_bf16(v, stg, lane, reinterpret_cast<bf16*>(p.out), p.ldo, row0, p.M,
                           sg.out_col + n0 + j * 32, ncols - j * 32);
          if (EPI == EPI_ROPE && sg.out2)
            store_chunk_bf16(v, stg, lane, sg.out2, sg.ldo2, row0, p.M, n0 + j * 32, ncols - j * 32);
          if (EPI == EPI_ROPE && sg.vt && m < p.M) {
            // V^T for the tcgen05 attention: lanes are consecutive tokens -> coalesced.
            // Batched prompts: sequence b's keys start at column b * round_up(seq_len, 64),
            // so every TMA box of V^T starts 16-B aligned; the last row of a sequence
            // also zeroes its padding columns (masked keys must hold finite values).
            int vcol = m, pad = 0;
            if (p.seq_len) {
              const int sb = m / p.seq_len, pos = m - sb * p.seq_len;
              const int lp = (p.seq_len + 63) & ~63;
              vcol = sb * lp + pos;
              if (pos == p.seq_len - 1) pad = lp - p.seq_len;
            }
            bf16* dst = p.vt + (size_t)(n0 + j * 32) * p.vt_ld + vcol;
            const int nv = min(32, ncols - j * 32);
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (i < nv) dst[(size_t)i * p.vt_ld] = __float2bfloat16_rn(v[i]);
            if (pad) {
#pragma unroll 1
              for (int i = 0; i < nv; ++i)
                for (int c = 1; c <= pad; ++c) dst[(size_t)i * p.vt_ld + c] = __float2bfloat16_rn(0.f);
            }
          }
        }
      }
      if (threadIdx.x == 64) dbg_put(p.dbg, it, 5, gtimer());
      ptx::tc_fence_before();
      if (CG == 2)
        ptx::mbar_arrive_leader(tempty_bar(acc));
      else
        ptx::mbar_arrive(tempty_bar(acc));
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  ptx::tc_fence_before();
  if (CG == 2)
    ptx::cluster_sync();
  else
    __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    if (CG == 2)
      ptx::tmem_dealloc_pair(tmem_base, TMEM_COLS);
    else
      ptx::tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn g_encode = nullptr;
std::once_flag g_once;

template <int EPI, int BNT, int CG, int MC = 1>
cudaError_t launch_t(const GemmParams& p, int num_sms, cudaStream_t s) {
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tc_kernel<EPI, BNT, CG, MC>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Cfg<EPI, BNT, CG>::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  const int units = gemm_units(CG, MC, num_sms);
  const int works = (EPI == EPI_RESID && p.ksplit > 1
                         ? p.n_full + (p.total_tiles - p.n_full) * p.ksplit
                         : p.total_tiles) +
                    (EPI == EPI_PARTIAL ? 0 : p.t_tiles * (p.t_ks > 1 ? p.t_ks : 1));
  const int grid = (works < units ? works : units) * CG * MC;
  if (grid <= 0) return cudaSuccess;
  return launch_kt(EPI == EPI_PARTIAL ? "shrink" : "gemm", gemm_tc_kernel<EPI, BNT, CG, MC>, dim3(grid), dim3(NTHREADS),
                  Cfg<EPI, BNT, CG>::SMEM_BYTES, s, CG * MC, p);
}

template <int EPI, int BNT>
cudaError_t launch_cg(const GemmParams& p, int num_sms, cudaStream_t s) {
  if (p.cg == 2 && p.mc == 2) return launch_t<EPI, BNT, 2, 2>(p, num_sms, s);
  if (p.cg == 2) return launch_t<EPI, BNT, 2>(p, num_sms, s);
  return launch_t<EPI, BNT, 1>(p, num_sms, s);
}

}  // namespace

int gemm_pick_cg(int M) { return M > GEMM_BM ? 2 : 1; }

// Concurrently resident clusters of cg * mc CTAs (one CTA per SM): a
// persistent grid larger than this would serialise whole clusters.
int gemm_units(int cg, int mc, int num_sms) {
  if (mc == 1) return num_sms / cg;
  static int cached = -1;
  if (cached < 0) {
    int n = 0;
    auto k = gemm_tc_kernel<EPI_RESID, 192, 2, 2>;
    constexpr int smem = Cfg<EPI_RESID, 192, 2>::SMEM_BYTES;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = 4;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.gridDim = dim3(num_sms / 4 * 4);
    cfg.blockDim = dim3(NTHREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess ||
        cudaOccupancyMaxActiveClusters(&n, k, &cfg) != cudaSuccess)
      n = 0;
    cudaGetLastError();
    cached = n;
  }
  return cached;
}

// Two CTA pairs per cluster sharing the weight boxes (TMA multicast): opt-in
// (TIDAL_GEMM_MC=2).  Measured at the 13B shapes it cuts L2->SM sectors by
// 20-25% but only 33 four-CTA clusters are co-resident (132 of 148 SMs), and
// per-SM tensor activity did not rise, so the pair-only grid is faster.
int gemm_pick_mc(int M, int num_sms) {
  static const bool on = [] {
    const char* e = getenv("TIDAL_GEMM_MC");
    return e && e[0] == '2';
  }();
  if (!on || gemm_pick_cg(M) != 2 || M <= 2 * GEMM_BM) return 1;
  return gemm_units(2, 2, num_sms) > 0 ? 2 : 1;
}

int gemm_m_tiles(int M, int cg, int mc) { return (M + BM * cg * mc - 1) / (BM * cg * mc); }

int gemm_pick_bn(int epi, int M, const int* seg_n, int nseg, int num_sms, int* cg_out) {
  const int cg0 = gemm_pick_cg(M);
  int best = 256, best_cg = cg0;
  double best_cost = 1e30;
  for (int cg = cg0; cg >= (cg_out ? 1 : cg0); --cg) {
    const int mc = cg == 2 ? gemm_pick_mc(M, num_sms) : 1;
    const int mt = gemm_m_tiles(M, cg, mc);
    const int units = gemm_units(cg, mc, num_sms);
    static const int cands[] = {256, 192, 128};
    for (int bn : cands) {
      if (epi == EPI_SILU && bn != 128) continue;
      if (epi == EPI_ROPE && bn == 192) continue;  // RoPE tiles must hold whole heads
      long tiles = 0;
      for (int s = 0; s < nseg; ++s) tiles += (long)mt * ((seg_n[s] + bn - 1) / bn);
      const long waves = (tiles + units - 1) / units;
      // 128-wide tiles pay ~15% more per MAC (A-operand smem traffic per MMA
      // doubles); single-CTA tiles ~10% (each CTA loads its whole B tile)
      const double cost = (double)waves * bn * (bn == 128 ? 1.15 : 1.0) *
                          (cg == 1 && cg0 == 2 ? 1.1 : 1.0);
      if (cost < best_cost - 1e-9) {
        best_cost = cost;
        best = bn;
        best_cg = cg;
      }
    }
  }
  if (cg_out) *cg_out = best_cg;
  return best;
}

// Residual (row-parallel) GEMMs: choose the CTA group, the N-tile width and
// the ordered split-K jointly.  Cost of a plan, in K-block times of a pair
// tile (~0.39 us at 13B): rounds x (K-blocks per part + ~11 K-blocks of
// per-part epilogue / hand-off), plus the ordered epilogue chain when the
// parts of a tile run in the same round; a K-block of a 192-wide pair tile
// costs as much as a 256-wide one (tools/gemm_bench.py --resid-sweep: O 256 x
// 2-3 parts 84-86 us, 192 x 1 part 97-127 us); single-CTA tiles (cg = 1, M =
// 128 rows) give the same per-SM rate.  Short prompts thereby split K until
// the works fill the SMs (13B S = 256: down 20 pair tiles x 3 parts instead
// of 54 whole-K single-CTA tiles on 54 SMs).
void gemm_plan_resid(int M, int N, int K, int num_sms, int* bn_out, int* ks_out, int* cg_out,
                     bool allow_split, int* nfull_out) {
  if (nfull_out) *nfull_out = 0;
  const int cg0 = gemm_pick_cg(M);
  const int nk = (K + BK - 1) / BK;
  static const int split_env = [] {
    const char* e = getenv("TIDAL_RESID_SPLIT");  // 0: no split-K; 3: also tail splits
    return e ? e[0] - '0' : 2;
  }();
  const bool split_ok = allow_split && split_env != 0;
  const bool tail_ok = nfull_out != nullptr && split_env == 3 && split_ok;
  static const int cands[] = {256, 192, 128};
  double best = 1e30;
  int bb = 256, bk = 1, bf = 0, bc = cg0;
  for (int cg = cg0; cg >= (cg_out ? 1 : cg0); --cg) {
    const int mc = cg == 2 ? gemm_pick_mc(M, num_sms) : 1;
    const long mt = gemm_m_tiles(M, cg, mc);
    const long units = gemm_units(cg, mc, num_sms);
    for (int bn : cands) {
      const long tiles = mt * ((N + bn - 1) / bn);
      if (tiles * mc * cg > GEMM_MAX_FLAGS) continue;
      // with one or two M tiles the K-block rate is bound by each SM's operand
      // stream (A + B bytes), not the MMA: a 192-wide K-block then costs ~0.75
      // of a 256-wide one (13B S = 256: O 192 x 2 parts 25.5-26 us vs 256 x 3
      // 33.5 us; down 192 x 2 45.7-46.4 us vs 256 x 3 51.6-51.7 us; at 0.8 the
      // 2 % hysteresis below kept down at 256 x 3, profiles/short_r02.txt)
      const bool stream_bound = M <= 2 * BM * 2;
      const double kb_cost = (bn == 128 ? 0.75 : (bn == 192 && stream_bound ? 0.75 : 1.0)) *
                             (cg == 1 ? 1.03 : 1.0);
      for (int ks = 1; ks <= (split_ok ? 8 : 1) && ks <= nk; ++ks) {
        const int kps = (nk + ks - 1) / ks;
        const int ks_eff = (nk + kps - 1) / kps;  // every part non-empty
        if (ks_eff != ks) continue;
        const long rounds = (tiles * ks + units - 1) / units;
        const double chain = rounds < ks ? 11.0 * (ks - 1) : 0.0;
        const double cost = ((double)rounds * (kps + 11) + chain) * kb_cost;
        if (cost < best * 0.98) {  // prefer fewer parts / the pair unless clearly better
          best = cost;
          bb = bn;
          bk = ks;
          bf = 0;
          bc = cg;
        }
      }
      // (b) opt-in (TIDAL_RESID_SPLIT=3): whole tiles for the full waves, the
      // last partial wave's tiles in ordered parts.  Measured slower than (a):
      // the parts of one tile run concurrently, so their ordered epilogues
      // serialise (O 256-wide: 92-116 us against 84 us uniform).
      const long full = tiles / units, tail = tiles - full * units;
      if (tail_ok && cg == cg0 && full >= 1 && tail > 0) {
        int ks = (int)(units / tail);
        ks = ks > 8 ? 8 : (ks > nk ? nk : ks);
        if (ks >= 2) {
          const int kps = (nk + ks - 1) / ks;
          const int ks_eff = (nk + kps - 1) / kps;
          const double cost = ((double)full * (nk + 11) + (kps + 11) + 11.0 * (ks - 1)) * kb_cost;
          if (cost < best * 0.98) {
            best = cost;
            bb = bn;
            bk = ks_eff;
            bf = (int)(full * units);
            bc = cg;
          }
        }
      }
    }
  }
  *bn_out = bb;
  *ks_out = bk;
  if (cg_out) *cg_out = bc;
  if (nfull_out) *nfull_out = bf;
}

int gemm_b_box(int epi, int bn, int cg, int mc) { return (epi == EPI_SILU ? 128 : bn / cg) / mc; }
int gemm_tb_box(int epi, int bn, int cg, int mc) {
  return (epi == EPI_SILU ? 128 / cg : bn / cg) / mc;
}

bool tma_init() {
  std::call_once(g_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<EncodeTiledFn>(fn);
  });
  return g_encode != nullptr;
}

bool make_tmap(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols,
               uint64_t row_stride_bytes, uint32_t box_rows, uint32_t box_cols) {
  if (!tma_init()) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

cudaError_t gemm_launch(const GemmParams& p0, int epi, int num_sms, cudaStream_t s) {
  const GemmParams& p = p0;
  switch (epi) {
    case EPI_STORE:
      if (p.bn == 192) return launch_cg<EPI_STORE, 192>(p, num_sms, s);
      if (p.bn == 128) return launch_cg<EPI_STORE, 128>(p, num_sms, s);
      return launch_cg<EPI_STORE, 256>(p, num_sms, s);
    case EPI_ROPE:
      if (p.bn == 128) return launch_cg<EPI_ROPE, 128>(p, num_sms, s);
      return launch_cg<EPI_ROPE, 256>(p, num_sms, s);
    case EPI_SILU: return launch_cg<EPI_SILU, 128>(p, num_sms, s);
    case EPI_RESID:
      if (p.bn == 192) return launch_cg<EPI_RESID, 192>(p, num_sms, s);
      if (p.bn == 128) return launch_cg<EPI_RESID, 128>(p, num_sms, s);
      return launch_cg<EPI_RESID, 256>(p, num_sms, s);
    case EPI_PARTIAL:  // split-K shrink: single-CTA tiles
      if (p.bn == 64) return launch_t<EPI_PARTIAL, 64, 1>(p, num_sms, s);
      if (p.bn == 128) return launch_t<EPI_PARTIAL, 128, 1>(p, num_sms, s);
      return launch_t<EPI_PARTIAL, 192, 1>(p, num_sms, s);
  }
  return cudaErrorInvalidValue;
}

// ---------------------------------------------------------------------------
// lora_A packing for the in-GEMM T tiles: lora_A_t [r, K] (adapter arena) ->
// pack[(kb * rt_pad + row0_t + j) * 64 + c] for K-block kb, so the T tile's
// B operand for one K-block is a single contiguous box of rt_pad rows.
// ---------------------------------------------------------------------------
namespace {
__global__ void lora_pack_kernel(const LoraPackArgs a) {
  ptx::pdl_begin();
  const int sgi = blockIdx.y;
  const bf16* __restrict__ src = a.src[sgi];
  const int K = a.K[sgi], r = a.r;
  const int chunks = r * (K / 8);  // 16-byte chunks of this lora_A
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < chunks; i += gridDim.x * blockDim.x) {
    const int j = i / (K / 8), c = i - j * (K / 8);
    const int kb = c >> 3, w = c & 7;
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(src + (size_t)j * K) + c);
    reinterpret_cast<uint4*>(a.dst[sgi])[((size_t)kb * a.rtp[sgi] + a.row0[sgi] + j) * 8 + w] = v;
  }
}
}  // namespace

cudaError_t lora_pack_launch(const LoraPackArgs& a, int num_sms, cudaStream_t s) {
  if (a.n <= 0) return cudaSuccess;
  return launch_k(lora_pack_kernel, dim3(num_sms, a.n), dim3(256), 0, s, 1, a);
}

// ---------------------------------------------------------------------------
// LoRA shrink on tensor cores: split-K EPI_PARTIAL GEMM + fixed-order reduce.
// ---------------------------------------------------------------------------
namespace {
__global__ void shrink_reduce_kernel(const float* __restrict__ ws, int ksplit, int M, int RT, int r,
                                     bf16* T0, bf16* T1, bf16* T2, float scale) {
  ptx::pdl_begin();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= M * RT) return;
  // all parts' loads in flight at once, then summed in part order (deterministic)
  float pv[SHRINK_MAX_SPLIT];
#pragma unroll
  for (int k = 0; k < SHRINK_MAX_SPLIT; ++k)
    if (k < ksplit) pv[k] = __ldcs(ws + (size_t)k * M * RT + e);
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < SHRINK_MAX_SPLIT; ++k)
    if (k < ksplit) s += pv[k];
  const int m = e / RT, c = e - m * RT, t = c / r;
  bf16* T = t == 0 ? T0 : (t == 1 ? T1 : T2);
  T[(size_t)m * r + (c - t * r)] = __float2bfloat16_rn(s * scale);
}
}  // namespace

bool shrink_plan(ShrinkPlan* sp, const bf16* X, int M, int K, const bf16* const* A, bf16* const* T,
                 int nt, int r, float* ws, int num_sms) {
  memset(sp, 0, sizeof *sp);
  GemmParams& g = sp->g;
  const int RT = nt * r;
  if (nt < 1 || nt > 3 || RT > 192 || r % 8) return false;
  g.bn = RT <= 64 ? 64 : (RT <= 128 ? 128 : 192);
  g.cg = 1;
  if (!make_tmap(&g.a, X, M, K, (uint64_t)K * 2, 128, 64)) return false;
  for (int s = 0; s < nt; ++s)
    if (!make_tmap(&g.b[s], A[s], r, K, (uint64_t)K * 2, r, 64)) return false;
  g.nseg = nt;
  g.src_rows = r;
  g.M = M;
  g.K = K;
  g.m_tiles = (M + BM - 1) / BM;
  g.n_tiles[0] = 1;
  g.seg[0].n = RT;
  const int nk = (K + BK - 1) / BK;
  int ks = num_sms / g.m_tiles;
  ks = ks < 1 ? 1 : (ks > SHRINK_MAX_SPLIT ? SHRINK_MAX_SPLIT : ks);
  g.kblocks_per_split = (nk + ks - 1) / ks;
  g.ksplit = (nk + g.kblocks_per_split - 1) / g.kblocks_per_split;  // every split non-empty
  g.total_tiles = g.m_tiles * g.ksplit;
  g.out = ws;
  g.ldo = RT;
  sp->M = M;
  sp->RT = RT;
  sp->r = r;
  sp->nt = nt;
  for (int s = 0; s < nt; ++s) sp->T[s] = T[s];
  sp->ws = ws;
  return true;
}

// A8 kernel pre-load for the LoRA shrink kernels, which the adapter-less warm
// forward at template creation does not launch (lazy loading would otherwise
// load them inside the first adapter invocation's TTFT window).
void shrink_preload() {
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, gemm_tc_kernel<EPI_PARTIAL, 64, 1, 1>);
  cudaFuncGetAttributes(&fa, gemm_tc_kernel<EPI_PARTIAL, 128, 1, 1>);
  cudaFuncGetAttributes(&fa, gemm_tc_kernel<EPI_PARTIAL, 192, 1, 1>);
  cudaFuncGetAttributes(&fa, shrink_reduce_kernel);
  cudaGetLastError();
}

cudaError_t shrink_run(const ShrinkPlan& sp, float scale, int num_sms, cudaStream_t s) {
  cudaError_t e = gemm_launch(sp.g, EPI_PARTIAL, num_sms, s);
  if (e != cudaSuccess) return e;
  const int n = sp.M * sp.RT;
  return launch_kt("reduce", shrink_reduce_kernel, dim3((n + 255) / 256), dim3(256), 0, s, 1, sp.ws,
                  sp.g.ksplit, sp.M, sp.RT, sp.r, sp.T[0], sp.T[1], sp.T[2], scale);
}

}  // namespace tidal
