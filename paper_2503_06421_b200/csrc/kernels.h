// kernels.h — device kernels of the prefill path (sm_100a), host launchers.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace tidal {

using bf16 = __nv_bfloat16;

// ------------------------------------------------------------------------
// tcgen05 GEMM  C[M, N] = A[M, K] . W[N, K]^T  (+ LoRA K-extension), fused
// epilogues.  A and W are bf16, K-major ("TN"), fed by TMA (SWIZZLE_128B)
// into a 4-stage mbarrier ring; accumulators live in TMEM (2 x 256 columns,
// double-buffered so the epilogue of tile i overlaps the mainloop of i+1);
// persistent grid of one CTA per SM.
// ------------------------------------------------------------------------
enum GemmEpi : int {
  EPI_STORE = 0,  // out bf16 [M, ldo] at out_col
  EPI_ROPE = 1,   // as STORE, rotate-half RoPE on segments with rope=1 (q, k)
  EPI_SILU = 2,   // W = [gate ; up] paired 128-row tiles: out = silu(g) * u (bf16)
  EPI_RESID = 3,  // out fp32 [M, ldo]: out += acc (residual stream)
  EPI_PARTIAL = 4 // split-K partial sums: out fp32 [ksplit][M][ldo] = acc; the B tile
                  // stacks nseg sources of src_rows rows each (LoRA shrink: A_q;A_k;A_v)
};

constexpr int GEMM_BM = 128, GEMM_BN = 256, GEMM_BK = 64, GEMM_STAGES = 4;

struct GemmSeg {
  int n;        // rows of this weight segment (output columns)
  int out_col;  // first output column
  int lora;     // LoRA K-extension present for this segment
  int rope;     // EPI_ROPE: rotate this segment
  int vt;       // EPI_ROPE: also store this segment transposed into GemmParams::vt
  bf16* out2;   // EPI_ROPE (nullable): also store this segment row-major [M, n] (ld ldo2):
  int ldo2;     //   the decode KV cache capturing K (after RoPE) and V during the prefill
};

struct alignas(64) GemmParams {
  CUtensorMap a;       // A [M, K], box {64, 128}
  CUtensorMap b[3];    // W segment [n, K], box {64, 256} (EPI_SILU: b[0]=gate, b[1]=up, box {64,128})
  CUtensorMap ta[3];   // T [M, r] (LoRA shrink output, scale folded), box {64, 128}
  CUtensorMap tb[3];   // lora_B [n, r], box {64, 256} (EPI_SILU: {64, 128})
  GemmSeg seg[3];
  int nseg;
  int M, K;
  int lora_r;          // 0: no LoRA
  int m_tiles;
  int n_tiles[3];
  int total_tiles;
  void* out;
  int ldo;
  const float2* rope;  // [S, head_dim/2] (cos, sin)
  int head_dim;
  int seq_len;         // EPI_ROPE: position = row % seq_len (batched prompts); 0: position = row
  int bn;              // N tile: 256 | 192 | 128 (EPI_SILU: 128 output cols = 256 acc cols)
  bf16* vt;            // V^T [n_vt][vt_ld] for the tcgen05 attention (segments with vt=1)
  int vt_ld;
  int ksplit, kblocks_per_split, src_rows;  // EPI_PARTIAL / EPI_RESID split-K
  int n_full;          // EPI_RESID with ksplit > 1: tiles [0, n_full) run whole, the rest
                       // in ksplit ordered parts (0: every tile split)
  int cg;              // 1: single-CTA 128-row tiles; 2: CTA pair, 256-row tiles (cta_group::2)
  int mc;              // cg == 2: CTA pairs per cluster sharing W boxes (1 or 2; 0 = 1)
  int* flags;          // EPI_RESID with ksplit > 1: per (tile, CTA) split counters, all 0
                       // between launches (GEMM_MAX_FLAGS ints); parts add in split order
  // In-GEMM LoRA shrink ("T tiles", t_tiles > 0): the first works of the
  // persistent grid (on the least loaded units) compute T_t = bf16(t_scale *
  // A x lora_A_t^T) for the t_nt targets sharing this GEMM's input A (stacked:
  // t_nt * t_r columns, MMA N = t_rt_pad) into t_out[t] [M, t_r], one tile per
  // m-tile, in t_ks K parts (t_ks > 1: the GEMM's own split-K ranges; fp32
  // partials in t_ws, the last part to arrive folds them in part order).
  // t_flags[0] counts published 128-row blocks; the LoRA K-extension of every
  // other tile waits (once per CTA) for all t_tiles * cg of them;
  // t_flags[1 + tile * cg + rank] count arrived parts.  All zeroed once per
  // forward.  Requires every CTA of the grid to be able to run (persistent
  // grid <= SMs, no co-located grids).  lora_A comes packed K-block-major.
  CUtensorMap la;      // packed lora_A [nk * t_rt_pad rows, 64 cols], box {64, t_rt_pad / cg}
  bf16* t_out[3];
  int t_tiles, t_ks, t_nt, t_r, t_rt_pad;
  float t_scale;
  int* t_flags;
  float* t_ws;         // t_ks > 1: [t_tiles][t_ks][128 * cg rows][t_rt_pad] fp32 partials
  unsigned long long* dbg;  // diagnostic per-work timeline (TIDAL_GEMM_TRACE); null in production
};
// lora_A of up to 7 targets (one layer) -> the packed T-tile layout:
// dst[sgi][(kb * rtp + row0 + j) * 64 + c] = src[sgi][j * K + kb * 64 + c].
struct LoraPackArgs {
  const bf16* src[7];
  bf16* dst[7];
  int K[7], row0[7], rtp[7];
  int n, r;
};
cudaError_t lora_pack_launch(const LoraPackArgs& a, int num_sms, cudaStream_t s);

// CTA-group size for an M-row GEMM, and the TMA box rows of the W and lora_B
// maps a CTA loads for (epi, bn, cg).
int gemm_pick_cg(int M);
// 2: clusters of two CTA pairs stacked in M sharing the W boxes by TMA multicast
int gemm_pick_mc(int M, int num_sms);
int gemm_units(int cg, int mc, int num_sms);  // resident clusters of cg * mc CTAs
int gemm_m_tiles(int M, int cg, int mc);      // M tiles of 128 * cg * mc rows
int gemm_b_box(int epi, int bn, int cg, int mc = 1);
// EPI_RESID: N-tile width and ordered split-K parts (GemmParams::ksplit and
// kblocks_per_split = ceil(nk / ks)) for an M x N x K residual GEMM.
constexpr int GEMM_MAX_FLAGS = 16384;
// cg_out (optional): also choose the CTA group — single-CTA tiles when they fit
// one wave and pair tiles would not (short prompts); else the pair default.
// allow_split = false: one part only (no CTA waits on another CTA's flag —
// required when several persistent grids may share the device).
// nfull_out (optional): allow a tail split — tiles [0, *nfull_out) whole, the
// rest in ks parts (GemmParams::n_full); without it every tile has ks parts.
void gemm_plan_resid(int M, int N, int K, int num_sms, int* bn, int* ks, int* cg_out = nullptr,
                     bool allow_split = true, int* nfull_out = nullptr);
int gemm_tb_box(int epi, int bn, int cg, int mc = 1);

// LoRA shrink on tensor cores: T_t = bf16(scale * X A_t^T) for nt targets
// sharing X, as a split-K EPI_PARTIAL GEMM into ws plus a fixed-order reduce.
struct ShrinkPlan {
  GemmParams g;
  int M, RT, r, nt;
  bf16* T[3];
  float* ws;
};
bool shrink_plan(ShrinkPlan* sp, const bf16* X, int M, int K, const bf16* const* A, bf16* const* T,
                 int nt, int r, float* ws, int num_sms);
cudaError_t shrink_run(const ShrinkPlan& sp, float scale, int num_sms, cudaStream_t s);
void shrink_preload();  // load the shrink kernels (template creation, A8)
constexpr int SHRINK_MAX_SPLIT = 16;

// tcgen05 causal attention (hd = 128): Q/K from QKV [S, (H+2KV)*128], V from
// V^T [KV*128][vt_ld] (written by the QKV epilogue).
struct alignas(64) AttnParams {
  CUtensorMap q;    // over QKV, box {64 cols, 128 rows}
  CUtensorMap k;    // over QKV, box {64 cols, 64 rows}
  CUtensorMap vt;   // over V^T, box {64 keys, 128 rows}
  int S, H, KV;     // S: tokens per sequence
  int nseq;         // sequences of S tokens each, stacked along the rows (grid.z)
  float scale_log2;
  bf16* out;
  int ldo;
  unsigned long long* dbg;  // diagnostic per-tile timeline (TIDAL_ATTN_TRACE); null in production
  int variant;  // 0: by size (pairs of query tiles when >= 2 rounds), 1: single tiles, 2: pairs
  const int* sched;  // paired kernel (set by attn_tc_launch): per-CTA pair-item lists,
                     // [G + 1] offsets then the item indices (host LPT schedule)
};
bool attn_tc_params(AttnParams* p, const bf16* qkv, const bf16* vt, int vt_ld, bf16* out, int S,
                    int H, int KV, int nseq = 1);
cudaError_t attn_tc_launch(const AttnParams& p, cudaStream_t s);

// N-tile width minimising (waves x tile width) on num_sms SMs; the W/lora_B
// tensor maps must use box rows = the returned value (128 for EPI_SILU).
// cg_out (optional): choose the CTA group too (pairs pay less shared-memory
// traffic per MAC; single CTAs double the tile count for short prompts).
int gemm_pick_bn(int epi, int M, const int* seg_n, int nseg, int num_sms, int* cg_out = nullptr);

// Host helpers (gemm_tc.cu).
bool tma_init();  // resolve cuTensorMapEncodeTiled through the runtime
// 2-D bf16 tensor map: rows x cols, row stride in bytes, box {box_cols, box_rows}, SW128.
bool make_tmap(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols,
               uint64_t row_stride_bytes, uint32_t box_rows, uint32_t box_cols);
cudaError_t gemm_launch(const GemmParams& p, int epi, int num_sms, cudaStream_t s);

// ------------------------------------------------------------------------
// SIMT / legacy-MMA kernels (kernels.cu, attention.cu)
// ------------------------------------------------------------------------
// X[s, :] = fp32(E[tok[s] - row0, :]) for tokens in [row0, row0+rows), else 0 (vocab shard).
// key_reset (nullable): n_keys keys zeroed by the kernel — the packed argmax keys of this forward.
cudaError_t embed_launch(const int32_t* tok, const bf16* E, float* X, int S, int d, int row0,
                         int rows, cudaStream_t s, unsigned long long* key_reset = nullptr,
                         int n_keys = 1);
// Y = bf16(g * x * rsqrt(mean(x^2) + eps)), one row per CTA.
cudaError_t rmsnorm_launch(const float* X, const bf16* g, bf16* Y, int S, int d, float eps,
                           cudaStream_t s);
// Causal GQA prefill attention over QKV [nseq * S, (H + 2 KV) hd] -> O [nseq * S, H hd],
// each sequence of S rows attending only to itself.
cudaError_t attention_launch(const bf16* qkv, bf16* O, int S, int H, int KV, int hd,
                             cudaStream_t s, int nseq = 1);
// For each of nseq rows X_last + b * x_stride: final RMSNorm, logits[b * ldl + v]
// = W[v] . h (fp32), and the packed argmax key (orderable(logit) << 32 | ~v)
// max-reduced into key[b] (preset to 0).  W is read once for all rows.
constexpr int HEAD_MAX_ROWS = 8;
cudaError_t head_launch(const float* X_last, size_t x_stride, int nseq, const bf16* g, const bf16* W,
                        int V, int d, float eps, float* logits, int ldl, unsigned long long* key,
                        int vocab_offset, int num_sms, cudaStream_t s);
// ------------------------------------------------------------------------
// Decode continuation (decode.cu): one token per step, all HBM-bound GEMVs.
// ------------------------------------------------------------------------
struct DecodeState {           // device-resident, read by every kernel of a step
  unsigned long long key;      // packed argmax of the last step (the next input token)
  int step;                    // decode steps started
  int pos;                     // position of the token fed in the current step
  int pos0;                    // prompt length (position of the first decoded input)
  int pad;
};
constexpr int DEC_TSPLIT = 2;      // K parts of the decode LoRA shrink (CTAs per 8 rows)
constexpr int DEC_TSTRIDE = 7 * 64;  // floats between parts: T[part][target][j]
struct DecShrink {             // T_t[j] = scale * A_t[j, :] . x   (t < nt <= 3, j < r)
  const bf16* A[3];
  float* T[3];                 // target t's slot; part q at T[t] + q * DEC_TSTRIDE
  int nt, r;
};
enum DecMode { DEC_QKV = 0, DEC_GU = 1, DEC_RESID = 2 };
struct DecGemv {
  // input: RMSNorm(X) * g (X fp32, g bf16) when X is set, else the bf16 vector xin
  const float* X;
  const bf16* g;
  const bf16* xin;
  float eps;
  int K;                       // input length
  int N;                       // output rows (DEC_RESID) / per-segment rows
  int npairs;                  // row pairs (one per warp iteration)
  const bf16* W[3];            // QKV: Wq, Wk, Wv; GU: Wgate, Wup; RESID: W
  const bf16* B[3];            // LoRA B per segment [rows, r] (nullable)
  const float* T[3];           // LoRA shrink outputs per segment (nullable; DEC_TSPLIT parts)
  int r;
  // QKV
  int nq, nkv, hd;
  const float2* rope;          // [positions][hd/2] (cos, sin)
  bf16* q;                     // [nq]
  bf16 *kc, *vc;               // this layer's cache rows [cap][nkv]
  const DecodeState* st;
  // GU
  bf16* h;                     // [F]
  // RESID
  float* Xout;                 // [N] += W . x
  // the LoRA shrink of this GEMV's input, computed by the first nsh CTAs of
  // the launch (0: none); T[seg] above point into sh.T's slots
  DecShrink sh;
  float sh_scale;
  int nsh;
  int* sh_cnt;                 // monotonic count of finished shrink CTAs (0 at decode start)
  int split;                   // DEC_RESID (set by dec_gemv_launch): a "pair" is one row's two
                               // K halves, so twice as many warps stream the (short) matrix
};
inline int dec_shrink_ctas(int nt, int r) { return ((nt * r + 7) / 8) * DEC_TSPLIT; }
struct DecAttn {
  const bf16* q;               // [H hd]
  const bf16 *kc, *vc;         // this layer's cache [cap][ldkv]
  int ldkv, H, KV, hd;
  float scale_log2;
  const DecodeState* st;       // keys 0 .. st->pos
  float* part;                 // [H][chunks][2 + 128] partial (max, sum, o)
  int* cnt;                    // [H] chunks finished (0 at rest)
  bf16* out;                   // [H hd]
};
cudaError_t dec_embed_launch(DecodeState* st, const bf16* E, float* X, int d, int32_t* toks_out,
                             cudaStream_t s);
cudaError_t dec_finish_launch(DecodeState* st, int32_t* toks_out, cudaStream_t s);
cudaError_t dec_save_logits_launch(const DecodeState* st, const float* logits, float* all, int V,
                                   cudaStream_t s);
cudaError_t dec_gemv_launch(const DecGemv& p, int mode, int num_sms, cudaStream_t s);
cudaError_t dec_attn_launch(const DecAttn& a, int max_keys, cudaStream_t s);

// TP bf16 allreduce option: Pb = bf16(P) before, X += Pb after the allreduce.
cudaError_t tp_pack_bf16_launch(const float* P, bf16* Pb, size_t n, int num_sms, cudaStream_t s);
cudaError_t tp_add_bf16_launch(const bf16* Pb, float* X, size_t n, int num_sms, cudaStream_t s);

// Debug / invariants.
cudaError_t poison_launch(void* p, size_t bytes, cudaStream_t s);           // bf16 NaN 0x7FC0
cudaError_t checksum_launch(const void* p, size_t bytes, unsigned long long* out, cudaStream_t s);
cudaError_t scrub_launch(void* p, size_t bytes, cudaStream_t s);
cudaError_t nan_check_launch(const float* x, int n, int* flag, cudaStream_t s);

}  // namespace tidal
