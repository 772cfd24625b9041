// runtime.cu — the op launcher: walks the canonical op sequence (plan.h R1),
// waits on the copy-stream events of the transfer groups each op reads
// (§5.2 "injects synchronization events"), and enqueues the
// fused kernels for that op.  The same launcher serves the traced first run
// (a Recorder captures first-read order as ops execute) and every invocation.
#include <cuda_runtime.h>
#include <sched.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <mutex>
#include <unordered_map>

#include "runtime.h"

namespace tidal {

[[noreturn]] void fail(int code, const std::string& msg) { throw Error{code, msg}; }

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    if (e == cudaErrorMemoryAllocation) fail(2, std::string(what) + ": " + cudaGetErrorString(e));
    fail(3, std::string(what) + ": " + cudaGetErrorString(e));
  }
}

namespace {
struct DevAllocator {
  DevAllocFn alloc = nullptr;
  DevFreeFn free_ = nullptr;
  void* ctx = nullptr;
  int device = -1;
};
std::mutex g_alloc_mu;
DevAllocator g_alloc;                                // the current hook (alloc == null: cudaMalloc)
std::unordered_map<void*, DevAllocator> g_owned;     // blocks that came from a hook
}  // namespace

void set_device_allocator(DevAllocFn alloc, DevFreeFn free_, void* ctx) {
  std::lock_guard<std::mutex> lk(g_alloc_mu);
  g_alloc.alloc = alloc;
  g_alloc.free_ = free_;
  g_alloc.ctx = ctx;
}

bool device_allocator_set() {
  std::lock_guard<std::mutex> lk(g_alloc_mu);
  return g_alloc.alloc != nullptr;
}

void* dev_alloc(size_t bytes, int device, const char* what) {
  DevAllocator a;
  {
    std::lock_guard<std::mutex> lk(g_alloc_mu);
    a = g_alloc;
  }
  bytes = bytes ? bytes : 16;
  if (!a.alloc) {
    void* q = nullptr;
    cuda_check(cudaMalloc(&q, bytes), what);
    return q;
  }
  void* q = a.alloc(bytes, device, a.ctx);
  if (!q) fail(2, std::string(what) + ": the caller's allocator returned NULL");
  a.device = device;
  std::lock_guard<std::mutex> lk(g_alloc_mu);
  g_owned[q] = a;
  return q;
}

void dev_free(void* p) {
  if (!p) return;
  DevAllocator a;
  {
    std::lock_guard<std::mutex> lk(g_alloc_mu);
    auto it = g_owned.find(p);
    if (it == g_owned.end()) {
      a.alloc = nullptr;
    } else {
      a = it->second;
      g_owned.erase(it);
    }
  }
  if (a.free_)
    a.free_(p, a.device, a.ctx);
  else if (!a.alloc)
    cudaFree(p);
}

template <typename T>
static void dalloc(T*& p, size_t bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  p = reinterpret_cast<T*>(dev_alloc(bytes, dev, "device allocation (activations)"));
}

void Exec::init(int dev, const ModelShape& shape, float eps_, float theta_, int world_, int rank_,
                int max_tok) {
  device = dev;
  m = shape;
  eps = eps_;
  theta = theta_;
  world = world_;
  rank = rank_;
  max_tokens = max_tok;
  cuda_check(cudaSetDevice(device), "cudaSetDevice");
  cuda_check(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, device), "SM count");
  if (!tma_init()) fail(3, "cuTensorMapEncodeTiled unavailable (driver too old?)");
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  cuda_check(cudaStreamCreateWithPriority(&compute, cudaStreamNonBlocking, lo), "stream");
  cuda_check(cudaStreamCreateWithPriority(&copy, cudaStreamNonBlocking, hi), "stream");
  const size_t S = (size_t)max_tokens;
  const int hd = m.head_dim();
  const size_t nq = (size_t)m.n_heads * hd / world, nkv = (size_t)m.n_kv_heads * hd / world;
  dalloc(X, S * m.d_model * 4);
  dalloc(Xn, S * m.d_model * 2);
  dalloc(QKV, S * (nq + 2 * nkv) * 2);
  dalloc(O, S * nq * 2);
  dalloc(Hb, S * (size_t)(m.d_ff / world) * 2);
  for (int t = 0; t < kNumTargets; ++t) dalloc(T[t], S * 64 * 2);
  dalloc(logits, (size_t)kMaxBatch * m.vocab * 4);
  dalloc(key, 8 * kMaxBatch);
  dalloc(tok, S * 4);
  // split-K partials of the stand-alone LoRA shrink, or of split T tiles
  // ([m-tiles][<= 8 parts][256 rows][<= 64 columns], rows rounded up to a tile)
  dalloc(shrink_ws, std::max((size_t)SHRINK_MAX_SPLIT * S * 192, (S + 256) * 8 * 64) * 4);
  dalloc(gemm_flags, GEMM_MAX_FLAGS * sizeof(int));
  dalloc(zero_b, (size_t)(m.d_ff / world) * 64 * 2);
  cuda_check(cudaMemset(zero_b, 0, (size_t)(m.d_ff / world) * 64 * 2), "memset zero lora_B");
  {
    // packed lora_A of the in-GEMM T tiles: per layer room for rank 64 x
    // (3 q/k/v, 1 o, 2 gate/up, 1 down) K-block-major; zeroed once so the
    // K-tail columns of a last partial K-block (never written) stay 0
    auto r64 = [](size_t k) { return (k + 63) / 64 * 64; };  // whole K-blocks
    const size_t nqr = (size_t)m.n_heads * m.head_dim() / world;
    pack_stride = (size_t)(192 + 128) * r64(m.d_model) + (size_t)64 * r64(nqr) +
                  (size_t)64 * r64(m.d_ff / world);
    dalloc(lora_pack, (size_t)m.n_layers * pack_stride * 2);
    cuda_check(cudaMemset(lora_pack, 0, (size_t)m.n_layers * pack_stride * 2), "memset lora pack");
  }
  tflag_stride = (int)((S + 127) / 128 + 4);
  dalloc(tflags, (size_t)m.n_layers * 4 * tflag_stride * sizeof(int));
  {
    const char* e = getenv("TIDAL_FUSED_SHRINK");  // 0: stand-alone shrink launches (A/B)
    fuse_shrink = !(e && e[0] == '0');
  }
  cuda_check(cudaMemset(gemm_flags, 0, GEMM_MAX_FLAGS * sizeof(int)), "memset flags");
  // V^T: batched prompts pad each sequence to 64 columns (<= 63 per prompt)
  vt_ld = (int)((S + 63) / 64 * 64 + 64 * (size_t)kMaxBatch);
  dalloc(Vt, nkv * (size_t)vt_ld * 2);
  cuda_check(cudaMemset(Vt, 0, nkv * (size_t)vt_ld * 2), "memset V^T");  // padding stays finite
  if (world > 1) {  // bf16 allreduce option (allocated up front: the option may be set any time)
    dalloc(P32, S * m.d_model * 4);
    dalloc(Pb, S * m.d_model * 2);
  }
  build_rope((int)S);
  cuda_check(cudaHostAlloc((void**)&h_tok, S * 4 + 16, cudaHostAllocDefault), "pinned tokens");
  cuda_check(cudaHostAlloc((void**)&h_logits, (size_t)kMaxBatch * m.vocab * 4 + 16,
                           cudaHostAllocDefault),
             "pinned logits");
  cuda_check(cudaHostAlloc((void**)&h_key, 8 * kMaxBatch, cudaHostAllocDefault), "pinned key");
}

// RoPE table: angle = pos * theta^(-2i/hd), cos/sin in double, stored fp32
void Exec::build_rope(int rows) {
  const int hd = m.head_dim();
  std::vector<float2> cs((size_t)rows * (hd / 2));
  for (size_t p = 0; p < (size_t)rows; ++p)
    for (int i = 0; i < hd / 2; ++i) {
      const double inv = std::pow((double)theta, -(2.0 * i) / hd);
      const double ang = (double)p * inv;
      cs[p * (hd / 2) + i] = make_float2((float)std::cos(ang), (float)std::sin(ang));
    }
  if (rope) dev_free(rope);
  rope = nullptr;
  dalloc(rope, cs.size() * sizeof(float2));
  cuda_check(cudaMemcpy(rope, cs.data(), cs.size() * sizeof(float2), cudaMemcpyHostToDevice),
             "rope upload");
}

// KV cache [L][max_tokens + max_new][nkv] for K and V, decode scratch and the
// RoPE table extended to the decoded positions.  Launch parameters are rebuilt
// (the QKV epilogue now also stores K and V into the cache).
void Exec::enable_decode(int max_new) {
  if (world != 1) fail(1, "decode with tensor parallelism is not implemented");
  if (max_new < 1) fail(1, "max_new_tokens must be >= 1");
  cuda_check(cudaSetDevice(device), "cudaSetDevice");
  cuda_check(cudaStreamSynchronize(compute), "sync");
  Decode& D = dec;
  void* ptrs[] = {D.kc, D.vc, D.q, D.att, D.h, D.T, D.part, D.cnt, D.shcnt, D.st, D.toks,
                  D.logits_all};
  for (void* p : ptrs) dev_free(p);
  if (D.gexec) cudaGraphExecDestroy(D.gexec);
  D = Decode();
  const int hd = m.head_dim();
  const size_t nq = (size_t)m.n_heads * hd, nkv = (size_t)m.n_kv_heads * hd;
  D.max_new = max_new;
  D.cap = max_tokens + max_new;
  dalloc(D.kc, (size_t)m.n_layers * D.cap * nkv * 2);
  dalloc(D.vc, (size_t)m.n_layers * D.cap * nkv * 2);
  dalloc(D.q, nq * 2);
  dalloc(D.att, nq * 2);
  dalloc(D.h, (size_t)m.d_ff * 2);
  dalloc(D.T, (size_t)DEC_TSPLIT * DEC_TSTRIDE * 4);
  dalloc(D.part, (size_t)m.n_heads * ((D.cap + 127) / 128) * 130 * 4);
  dalloc(D.cnt, (size_t)m.n_heads * 4);
  dalloc(D.shcnt, (size_t)m.n_layers * 4 * 4);
  cuda_check(cudaMemset(D.cnt, 0, (size_t)m.n_heads * 4), "memset");
  dalloc(D.st, sizeof(DecodeState));
  dalloc(D.toks, (size_t)max_new * 4);
  dalloc(D.logits_all, (size_t)max_new * m.vocab * 4);
  build_rope(D.cap);
  cache.clear();
}

void Exec::dbg_dump() {
  if (!dbg_pending || !dbg_trace) return;
  dbg_pending = false;
  std::vector<unsigned long long> h((size_t)num_sms * 32 * 8);
  if (cudaMemcpy(h.data(), dbg_trace, h.size() * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return;
  const char* path = getenv("TIDAL_GEMM_TRACE_FILE");
  FILE* f = fopen(path ? path : "gemm_trace.bin", "wb");
  if (!f) return;
  fwrite(h.data(), 8, h.size(), f);
  fclose(f);
}

void Exec::destroy() {
  if (device < 0) return;
  cudaSetDevice(device);
  if (compute) cudaStreamSynchronize(compute);
  if (copy) cudaStreamSynchronize(copy);
  void* ptrs[] = {X, Xn, QKV, O, Hb, logits, key, tok, rope, Vt, shrink_ws, gemm_flags, P32, Pb, tflags,
                  zero_b, dbg_trace, lora_pack,
                  dec.kc, dec.vc, dec.q, dec.att, dec.h, dec.T, dec.part, dec.cnt, dec.shcnt, dec.st,
                  dec.toks,
                  dec.logits_all};
  if (dec.gexec) cudaGraphExecDestroy(dec.gexec);
  for (void* p : ptrs) dev_free(p);
  for (int t = 0; t < kNumTargets; ++t) dev_free(T[t]);
  if (h_tok) cudaFreeHost(h_tok);
  if (h_logits) cudaFreeHost(h_logits);
  if (h_key) cudaFreeHost(h_key);
  if (compute) cudaStreamDestroy(compute);
  if (copy) cudaStreamDestroy(copy);
  device = -1;
}

static void tmap(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols,
                 uint32_t box_rows) {
  if (!make_tmap(m, base, rows, cols, cols * 2, box_rows, 64))
    fail(3, "cuTensorMapEncodeTiled failed (rows=" + std::to_string(rows) +
                " cols=" + std::to_string(cols) + ")");
}

const std::vector<LayerLaunch>& Exec::layer_params(const TensorTable& tt, int S, int nseq,
                                                   const void* akey, uint64_t gen) {
  auto k = std::make_tuple(S, nseq, tt.lora_rank, tt.lora_mask, akey, gen);
  auto it = cache.find(k);
  if (it != cache.end()) return it->second;
  const int L = m.n_layers, d = m.d_model, hd = m.head_dim();
  const int nq = m.n_heads * hd / world, nkv = m.n_kv_heads * hd / world;
  const int F = m.d_ff / world;
  const int r = tt.lora_rank;
  std::vector<LayerLaunch> v(L);
  for (int l = 0; l < L; ++l) {
    LayerLaunch& ll = v[l];
    int cur = 0;  // which GEMM's tensor maps are being built (ids recorded per GEMM)
    auto W = [&](int id) {
      ll.ids[cur].push_back(id);
      return wptr[id];
    };
    // ---- QKV + RoPE ----
    GemmParams& q = ll.qkv;
    memset(&q, 0, sizeof q);
    tmap(&q.a, Xn, S, d, 128);
    const int segn[3] = {nq, nkv, nkv};
    const int tg[3] = {T_Q, T_K, T_V};
    int col = 0;
    q.lora_r = 0;
    q.total_tiles = 0;
    q.bn = gemm_pick_bn(EPI_ROPE, S, segn, 3, num_sms, &q.cg);
    q.mc = q.cg == 2 ? gemm_pick_mc(S, num_sms) : 1;
    const int qmt = gemm_m_tiles(S, q.cg, q.mc);
    for (int s = 0; s < 3; ++s) {
      q.seg[s].n = segn[s];
      q.seg[s].out_col = col;
      q.seg[s].rope = s < 2;
      col += segn[s];
      tmap(&q.b[s], W(tt.proj[l][tg[s]]), segn[s], d, gemm_b_box(EPI_ROPE, q.bn, q.cg, q.mc));
      const int la = tt.lora_a[l][tg[s]];
      q.seg[s].lora = la >= 0;
      if (la >= 0) {
        q.lora_r = r;
        tmap(&q.ta[s], T[tg[s]], S, r, 128);
        tmap(&q.tb[s], W(tt.lora_b[l][tg[s]]), segn[s], r, gemm_tb_box(EPI_ROPE, q.bn, q.cg, q.mc));
      }
      q.n_tiles[s] = (segn[s] + q.bn - 1) / q.bn;
      q.total_tiles += q.n_tiles[s] * qmt;
    }
    q.nseg = 3;
    q.seg[2].vt = hd == 128;  // V^T for the tcgen05 attention
    if (dec.kc && nseq == 1) {  // decode enabled: K (after RoPE) and V into the cache
      q.seg[1].out2 = dec.kc + (size_t)l * dec.cap * nkv;
      q.seg[1].ldo2 = nkv;
      q.seg[2].out2 = dec.vc + (size_t)l * dec.cap * nkv;
      q.seg[2].ldo2 = nkv;
    }
    q.vt = Vt;
    q.vt_ld = vt_ld;
    q.M = S;
    q.K = d;
    q.m_tiles = qmt;
    q.out = QKV;
    q.ldo = nq + 2 * nkv;
    q.rope = rope;
    q.head_dim = hd;
    q.seq_len = nseq > 1 ? S / nseq : 0;
    // ---- O (+ residual) ----
    cur = 1;
    GemmParams& o = ll.o;
    memset(&o, 0, sizeof o);
    int ks = 1;
    gemm_plan_resid(S, d, nq, num_sms, &o.bn, &ks, &o.cg, !colocated, &o.n_full);
    o.ksplit = ks;
    o.kblocks_per_split = ((nq + GEMM_BK - 1) / GEMM_BK + ks - 1) / ks;
    o.flags = gemm_flags;
    o.mc = o.cg == 2 ? gemm_pick_mc(S, num_sms) : 1;
    const int omt = gemm_m_tiles(S, o.cg, o.mc);
    tmap(&o.a, O, S, nq, 128);
    tmap(&o.b[0], W(tt.proj[l][T_O]), d, nq, gemm_b_box(EPI_RESID, o.bn, o.cg, o.mc));
    o.seg[0].n = d;
    o.seg[0].lora = tt.lora_a[l][T_O] >= 0;
    if (o.seg[0].lora) {
      o.lora_r = r;
      tmap(&o.ta[0], T[T_O], S, r, 128);
      tmap(&o.tb[0], W(tt.lora_b[l][T_O]), d, r, gemm_tb_box(EPI_RESID, o.bn, o.cg, o.mc));
    }
    o.nseg = 1;
    o.M = S;
    o.K = nq;
    o.m_tiles = omt;
    o.n_tiles[0] = (d + o.bn - 1) / o.bn;
    o.total_tiles = o.n_tiles[0] * omt;
    o.out = X;
    o.ldo = d;
    // ---- gate/up + SiLU*mul ----
    cur = 2;
    GemmParams& g = ll.gu;
    memset(&g, 0, sizeof g);
    {
      const int fn = F;
      g.bn = gemm_pick_bn(EPI_SILU, S, &fn, 1, num_sms, &g.cg);
    }
    g.mc = g.cg == 2 ? gemm_pick_mc(S, num_sms) : 1;
    const int gmt = gemm_m_tiles(S, g.cg, g.mc);
    tmap(&g.a, Xn, S, d, 128);
    tmap(&g.b[0], W(tt.proj[l][T_GATE]), F, d, gemm_b_box(EPI_SILU, 128, g.cg, g.mc));
    tmap(&g.b[1], W(tt.proj[l][T_UP]), F, d, gemm_b_box(EPI_SILU, 128, g.cg, g.mc));
    g.seg[0].n = F;
    {
      // the paired gate/up tile has one LoRA K-extension per half; a target the
      // adapter leaves out gets an all-zero lora_B box (its T is any finite T)
      const bool lg = tt.lora_a[l][T_GATE] >= 0, lu = tt.lora_a[l][T_UP] >= 0;
      g.seg[0].lora = lg || lu;
      if (lg || lu) {
        g.lora_r = r;
        const int tbb = gemm_tb_box(EPI_SILU, 128, g.cg, g.mc);
        tmap(&g.ta[0], T[lg ? T_GATE : T_UP], S, r, 128);
        tmap(&g.ta[1], T[lu ? T_UP : T_GATE], S, r, 128);
        tmap(&g.tb[0], lg ? W(tt.lora_b[l][T_GATE]) : zero_b, F, r, tbb);
        tmap(&g.tb[1], lu ? W(tt.lora_b[l][T_UP]) : zero_b, F, r, tbb);
      }
    }
    g.nseg = 1;
    g.bn = 128;
    g.M = S;
    g.K = d;
    g.m_tiles = gmt;
    g.n_tiles[0] = (F + 127) / 128;
    g.total_tiles = g.n_tiles[0] * gmt;
    g.out = Hb;
    g.ldo = F;
    // ---- down (+ residual) ----
    cur = 3;
    GemmParams& dn = ll.down;
    memset(&dn, 0, sizeof dn);
    gemm_plan_resid(S, d, F, num_sms, &dn.bn, &ks, &dn.cg, !colocated, &dn.n_full);
    dn.ksplit = ks;
    dn.kblocks_per_split = ((F + GEMM_BK - 1) / GEMM_BK + ks - 1) / ks;
    dn.flags = gemm_flags;
    dn.mc = dn.cg == 2 ? gemm_pick_mc(S, num_sms) : 1;
    const int dmt = gemm_m_tiles(S, dn.cg, dn.mc);
    tmap(&dn.a, Hb, S, F, 128);
    tmap(&dn.b[0], W(tt.proj[l][T_DOWN]), d, F, gemm_b_box(EPI_RESID, dn.bn, dn.cg, dn.mc));
    dn.seg[0].n = d;
    dn.seg[0].lora = tt.lora_a[l][T_DOWN] >= 0;
    if (dn.seg[0].lora) {
      dn.lora_r = r;
      tmap(&dn.ta[0], T[T_DOWN], S, r, 128);
      tmap(&dn.tb[0], W(tt.lora_b[l][T_DOWN]), d, r, gemm_tb_box(EPI_RESID, dn.bn, dn.cg, dn.mc));
    }
    dn.nseg = 1;
    dn.M = S;
    dn.K = F;
    dn.m_tiles = dmt;
    dn.n_tiles[0] = (d + dn.bn - 1) / dn.bn;
    dn.total_tiles = dn.n_tiles[0] * dmt;
    dn.out = X;
    dn.ldo = d;
    // ---- LoRA shrinks (T = s x A^T) for the targets sharing each input ----
    if (r) {
      const std::initializer_list<int> groups[4] = {{T_Q, T_K, T_V}, {T_O}, {T_GATE, T_UP}, {T_DOWN}};
      const bf16* inputs[4] = {Xn, O, Xn, Hb};
      const int kdim[4] = {d, nq, d, F};
      GemmParams* gp[4] = {&ll.qkv, &ll.o, &ll.gu, &ll.down};
      for (int gi = 0; gi < 4; ++gi) {
        cur = gi;
        const bf16* A[3];
        bf16* Tt[3];
        int n = 0;
        for (int t : groups[gi])
          if (tt.lora_a[l][t] >= 0) {
            A[n] = reinterpret_cast<const bf16*>(W(tt.lora_a[l][t]));
            Tt[n] = T[t];
            ++n;
          }
        if (!n) continue;
        // in-GEMM T tiles when the stacked lora_A fits one accumulator buffer and
        // no other grid can share the device (a T-tile wait needs its producer CTA)
        GemmParams& g = *gp[gi];
        const int bnx = gi == 2 ? 256 : g.bn;
        const int rt_pad = (n * r + 15) / 16 * 16;
        if (fuse_shrink && !colocated && g.mc <= 1 && rt_pad <= bnx) {
          // packed lora_A region of this (layer, GEMM): room for rank 64 x 3
          // targets, so the offsets do not depend on the adapter
          if (!lora_pack) fail(3, "packed lora_A buffer missing");
          auto r64 = [](size_t k) { return (k + 63) / 64 * 64; };  // whole K-blocks
          const size_t goff = gi == 0 ? 0
                              : gi == 1 ? (size_t)192 * r64(d)
                              : gi == 2 ? (size_t)192 * r64(d) + (size_t)64 * r64(nq)
                                        : (size_t)320 * r64(d) + (size_t)64 * r64(nq);
          bf16* dst = lora_pack + (size_t)l * pack_stride + goff;
          const int nk = (kdim[gi] + GEMM_BK - 1) / GEMM_BK;
          if (!make_tmap(&g.la, dst, (uint64_t)nk * rt_pad, 64, 128, rt_pad / g.cg, 64))
            fail(3, "packed lora_A tensor map");
          for (int s2 = 0; s2 < n; ++s2) {
            g.t_out[s2] = Tt[s2];
            LoraPackArgs& pa = ll.pack;
            pa.src[pa.n] = A[s2];
            pa.dst[pa.n] = dst;
            pa.K[pa.n] = kdim[gi];
            pa.row0[pa.n] = s2 * r;
            pa.rtp[pa.n] = rt_pad;
            pa.r = r;
            ++pa.n;
          }
          for (int t : groups[gi])
            if (tt.lora_a[l][t] >= 0) ll.pack_ids.push_back(tt.lora_a[l][t]);
          g.t_nt = n;
          g.t_r = r;
          g.t_rt_pad = rt_pad;
          g.t_tiles = g.m_tiles;
          // split GEMMs: the T tile in the same K parts (a whole-K T tile would
          // take ks part-times on its unit)
          g.t_ks = (gi == 1 || gi == 3) && g.ksplit > 1 ? g.ksplit : 1;
          g.t_ws = shrink_ws;
          g.t_flags = tflags + (size_t)(4 * l + gi) * tflag_stride;
          continue;
        }
        if (!shrink_plan(&ll.sh[gi], inputs[gi], S, kdim[gi], A, Tt, n, r, shrink_ws, num_sms))
          fail(3, "shrink tensor maps");
        ll.has_sh[gi] = 1;
      }
    }
  }
  if (cache.size() > 64) cache.clear();
  return cache.emplace(k, std::move(v)).first->second;
}

const char* const kKernelClassNames[KC_COUNT] = {
    "embed", "rmsnorm", "lora_shrink", "gemm_qkv_rope", "attention", "gemm_o_resid",
    "gemm_gate_up_silu", "gemm_down_resid", "head_argmax", "allreduce"};

int Exec::prof_begin() {
  const size_t i = prof_pending.size();
  while (prof_ev.size() < 2 * (i + 1)) {
    cudaEvent_t e;
    cuda_check(cudaEventCreate(&e), "cudaEventCreate(profile)");
    prof_ev.push_back(e);
  }
  cuda_check(cudaEventRecord(prof_ev[2 * i], compute), "event");
  prof_pending.push_back({-1, (int)i, 0, 0});
  return (int)i;
}

void Exec::prof_end(int cls, int ev, double flops, double bytes) {
  cuda_check(cudaEventRecord(prof_ev[2 * ev + 1], compute), "event");
  prof_pending[ev] = {cls, ev, flops, bytes};
}

void Exec::prof_collect() {
  if (prof_tot.size() < KC_COUNT) prof_tot.resize(KC_COUNT);
  for (const ProfRec& p : prof_pending) {
    if (p.cls < 0) continue;
    float ms = 0;
    cuda_check(cudaEventElapsedTime(&ms, prof_ev[2 * p.ev], prof_ev[2 * p.ev + 1]), "elapsed");
    ProfTot& t = prof_tot[p.cls];
    t.ms += ms;
    t.flops += p.flops;
    t.bytes += p.bytes;
    t.launches += 1;
  }
  prof_pending.clear();
}

cudaError_t Exec::attention_tc(int S, int nseq, cudaStream_t s) {
  auto it = attn_cache.find({S, nseq});
  if (it == attn_cache.end()) {
    AttnParams p;
    memset(&p, 0, sizeof p);
    if (!attn_tc_params(&p, QKV, Vt, vt_ld, O, S / nseq, m.n_heads / world, m.n_kv_heads / world,
                        nseq))
      fail(3, "attention tensor maps");
    // TIDAL_ATTN=1 / 2 pins the single-tile / paired kernel for this template (A/B, tests)
    if (const char* v = getenv("TIDAL_ATTN")) p.variant = atoi(v);
    it = attn_cache.emplace(std::make_pair(S, nseq), p).first;
  }
  return attn_tc_launch(it->second, s);
}

enum OpKind {
  OP_EMBED, OP_ATTN_NORM, OP_QKV, OP_ROPE, OP_ATTN, OP_O, OP_MLP_NORM, OP_GU, OP_ACT, OP_DOWN,
  OP_FNORM, OP_HEAD, OP_ARGMAX, OP_EMBED_AR, OP_ATTN_AR, OP_MLP_AR, OP_LOGITS_AG
};

static int op_kind(const std::string& n) {
  static const std::map<std::string, int> k = {
      {"embed", OP_EMBED}, {"attn_norm", OP_ATTN_NORM}, {"qkv_proj", OP_QKV}, {"rope", OP_ROPE},
      {"attention", OP_ATTN}, {"o_proj", OP_O}, {"mlp_norm", OP_MLP_NORM},
      {"gate_up_proj", OP_GU}, {"act_mul", OP_ACT}, {"down_proj", OP_DOWN},
      {"final_norm", OP_FNORM}, {"lm_head", OP_HEAD}, {"argmax", OP_ARGMAX},
      {"embed_allreduce", OP_EMBED_AR}, {"attn_allreduce", OP_ATTN_AR},
      {"mlp_allreduce", OP_MLP_AR}, {"logits_allgather", OP_LOGITS_AG}};
  auto it = k.find(n);
  if (it == k.end()) fail(1, "unknown op " + n);
  return it->second;
}

// TP collectives (comm.cu); no-ops when world == 1.
void tp_allreduce_f32(Exec& ex, Comm* comm, float* buf, size_t n);
void tp_allreduce_bf16(Exec& ex, Comm* comm, bf16* buf, size_t n);
void tp_argmax_reduce(Exec& ex, Comm* comm, unsigned long long* key, int nseq);
void tp_allgather_logits(Exec& ex, Comm* comm, int nseq);

void run_forward(Exec& ex, const RunArgs& a) {
  const TensorTable& tt = *a.tt;
  const ModelShape& m = ex.m;
  const int S = a.S, d = m.d_model, hd = m.head_dim();
  const int nq = m.n_heads * hd / ex.world;
  const int F = m.d_ff / ex.world;
  const int Vl = m.vocab / ex.world;
  const int r = tt.lora_rank;
  const int B = a.nseq, Ls = S / B;  // B prompts of Ls tokens
  if (B < 1 || B > kMaxBatch || Ls * B != S) fail(1, "bad batch shape");
  const auto& LP = ex.layer_params(tt, S, B, a.akey, a.gen);
  cudaStream_t st = ex.compute;
  int waited = -1;
  // event pair around a launch: every launch (profile_all) or the GEMMs only
  auto P0 = [&](int cls = -1) {
    if (!ex.profile) return -1;
    if (!ex.profile_all && cls < 0) return -1;
    return ex.prof_begin();
  };
  auto K = [&](int cls, int ev, double fl, double by, cudaError_t e, const char* what) {
    cuda_check(e, what);
    ++ex.launches;
    if (ev >= 0) ex.prof_end(cls, ev, fl, by);
  };
  const double Sd = S;
  // LoRA shrink gi (0 qkv, 1 o, 2 gate_up, 3 down): split-K tcgen05 GEMM + reduce
  auto shrink = [&](const bf16* X, int ldx, int Kd, int l, int gi) {
    (void)X;
    (void)ldx;
    if (!LP[l].has_sh[gi]) return;
    const ShrinkPlan& sp = LP[l].sh[gi];
    const int e0 = P0();
    K(KC_SHRINK, e0, 2.0 * Sd * Kd * sp.RT, 2.0 * (Sd * Kd + (double)sp.RT * (Kd + Sd)),
      shrink_run(sp, a.lora_scale, ex.num_sms, st), "lora_shrink");
    ++ex.launches;  // shrink_run launches two kernels (GEMM + reduce)
  };
  auto lora_n = [&](int l, std::initializer_list<int> ts) {
    double n = 0;
    for (int t : ts)
      if (tt.lora_a[l][t] >= 0) n += tt.t[tt.lora_b[l][t]].rows;
    return n;
  };
  const int nkv = m.n_kv_heads * hd / ex.world;
  // row-parallel GEMMs under TP: rank 0 adds its partial sum to the residual,
  // the others start from zero (the allreduce then sums residual + partials);
  // with the bf16 allreduce every rank's partial goes to P32 instead
  const bool bf16_ar = ex.world > 1 && ex.ar_bf16;
  // GEMM launch; with in-GEMM T tiles the invocation's LoRA scale goes into a
  // copy of the cached parameters
  // diagnostic: TIDAL_GEMM_TRACE=<layer>,<gemm 0 qkv|1 o|2 gu|3 down> records a
  // per-work timeline of that one launch (dumped by the invoke after it syncs)
  static const int trace_sel = [] {
    const char* e = getenv("TIDAL_GEMM_TRACE");
    int l = -1, g = 0;
    if (e && sscanf(e, "%d,%d", &l, &g) >= 1 && l >= 0) return l * 4 + g;
    return -1;
  }();
  int cur_gemm = -1;
  auto launch = [&](const GemmParams& g, int epi, float* out_override = nullptr) {
    const bool tr = trace_sel >= 0 && cur_gemm == trace_sel;
    if (!g.t_tiles && !out_override && !tr) return gemm_launch(g, epi, ex.num_sms, st);
    GemmParams p = g;
    p.t_scale = a.lora_scale;
    if (out_override) p.out = out_override;
    if (tr) {
      const size_t nb = (size_t)ex.num_sms * 32 * 8 * 8;
      if (!ex.dbg_trace)
        ex.dbg_trace = reinterpret_cast<unsigned long long*>(dev_alloc(nb, ex.device, "trace"));
      cuda_check(cudaMemsetAsync(ex.dbg_trace, 0, nb, st), "memset trace");
      p.dbg = ex.dbg_trace;
      ex.dbg_pending = true;
    }
    return gemm_launch(p, epi, ex.num_sms, st);
  };
  auto resid_gemm = [&](const GemmParams& g) {
    if (bf16_ar) {
      cuda_check(cudaMemsetAsync(ex.P32, 0, (size_t)S * d * 4, st), "memset partial");
      return launch(g, EPI_RESID, ex.P32);
    }
    if (ex.world > 1 && ex.rank != 0)
      cuda_check(cudaMemsetAsync(ex.X, 0, (size_t)S * d * 4, st), "memset partial");
    return launch(g, EPI_RESID);
  };
  // the T-ready flags of the in-GEMM LoRA shrinks start at 0 in every forward
  if (r) {
    bool fused = false;
    for (const LayerLaunch& ll : LP) fused |= ll.qkv.t_tiles || ll.o.t_tiles || ll.gu.t_tiles || ll.down.t_tiles;
    if (fused)
      cuda_check(cudaMemsetAsync(ex.tflags, 0, (size_t)m.n_layers * 4 * ex.tflag_stride * sizeof(int), st),
                 "memset T flags");
  }
  const std::vector<Op>& ops = *a.ops;
  for (size_t k = 0; k < ops.size(); ++k) {
    const Op& op = ops[k];
    // lax tracing: the ids behind this op's kernel arguments (below)
    auto rec = [&](std::initializer_list<int> ids) {
      if (a.rec)
        for (int id : ids) a.rec->use((int)k, id, tt.n_base);
    };
    if (a.barriers && !(*a.barriers)[k].empty()) {
      // the copy stream is FIFO: waiting on the needed group copied last covers
      // all of them (waited = copy position already covered)
      int g = -1, gp = -1;
      for (int x : (*a.barriers)[k]) {
        if (x == a.skip_group) continue;
        const int pos = a.copy_pos ? (*a.copy_pos)[x] : x;
        if (pos > gp) {
          gp = pos;
          g = x;
        }
      }
      if (gp > waited) {
        cuda_check(cudaStreamWaitEvent(st, (*a.events)[g], 0), "cudaStreamWaitEvent");
        waited = gp;
      }
    }
    if (a.tl_op) cuda_check(cudaEventRecord((*a.tl_op)[k], st), "timeline event");
    const int l = op.layer;
    auto Wp = [&](int id) { return reinterpret_cast<const bf16*>(ex.wptr[id]); };
    switch (op_kind(op.name)) {
      case OP_EMBED:
        rec({tt.embed});
        {
          const int e0 = P0();
          K(KC_EMBED, e0, 0, Sd * d * 6, embed_launch(ex.tok, Wp(tt.embed), ex.X, S, d, ex.rank * Vl, Vl, st, ex.key, B),
            "embed");
        }
        break;
      case OP_EMBED_AR:
      case OP_ATTN_AR:
      case OP_MLP_AR:
        {
          const int e0 = P0();
          const size_t n = (size_t)S * d;
          if (bf16_ar && op_kind(op.name) != OP_EMBED_AR) {
            // C1/C2 in bf16: the partial sum (P32, no residual) is rounded once,
            // reduced in bf16 and added to the fp32 residual stream
            cuda_check(tp_pack_bf16_launch(ex.P32, ex.Pb, n, ex.num_sms, st), "tp pack");
            tp_allreduce_bf16(ex, a.comm, ex.Pb, n);
            cuda_check(tp_add_bf16_launch(ex.Pb, ex.X, n, ex.num_sms, st), "tp add");
            ex.launches += 2;
            if (e0 >= 0) ex.prof_end(KC_ALLREDUCE, e0, 0, Sd * d * 2);
          } else {
            tp_allreduce_f32(ex, a.comm, ex.X, n);
            if (e0 >= 0) ex.prof_end(KC_ALLREDUCE, e0, 0, Sd * d * 4);
          }
        }
        break;
      case OP_ATTN_NORM:
        rec({tt.norm1[l]});
        {
          const int e0 = P0();
          K(KC_RMSNORM, e0, 0, Sd * d * 6 + 2.0 * d,
            rmsnorm_launch(ex.X, Wp(tt.norm1[l]), ex.Xn, S, d, ex.eps, st), "rmsnorm");
        }
        break;
      case OP_QKV:
        if (a.rec) a.rec->use((int)k, LP[l].ids[0], tt.n_base);
        cur_gemm = 4 * l + 0;
        if (LP[l].pack.n) {
          // pack this layer's lora_A (all fused GEMMs) once its adapter bytes
          // landed: the groups of those tensors (one group under per_layer)
          if (a.barriers && a.group_of) {
            int gp = -1, g = -1;
            for (int id : LP[l].pack_ids) {
              const int x = (*a.group_of)[id];
              if (x < 0 || x == a.skip_group) continue;
              const int pos = a.copy_pos ? (*a.copy_pos)[x] : x;
              if (pos > gp) {
                gp = pos;
                g = x;
              }
            }
            if (gp > waited) {
              cuda_check(cudaStreamWaitEvent(st, (*a.events)[g], 0), "cudaStreamWaitEvent");
              waited = gp;
            }
          }
          const int e0 = P0();
          K(KC_SHRINK, e0, 0, 4.0 * LP[l].pack.n * LP[l].pack.r * d,
            lora_pack_launch(LP[l].pack, ex.num_sms, st), "lora_pack");
        }
        shrink(ex.Xn, d, d, l, 0);
        {
          const double n = nq + 2.0 * nkv;
          const int e0 = P0(KC_GEMM_QKV);
          K(KC_GEMM_QKV, e0, 2.0 * Sd * (n * d + r * lora_n(l, {T_Q, T_K, T_V})),
            2.0 * (n * d + Sd * d + Sd * n), launch(LP[l].qkv, EPI_ROPE),
            "gemm_qkv");
        }
        break;
      case OP_ROPE:  // fused into the QKV epilogue
        break;
      case OP_ATTN:
        {
          const int e0 = P0();
          K(KC_ATTN, e0, 2.0 * hd * ((double)m.n_heads / ex.world) * Sd * (Ls + 1.0),
            2.0 * Sd * (2.0 * nq + 2.0 * nkv),
            hd == 128 ? ex.attention_tc(S, B, st)
                      : attention_launch(ex.QKV, ex.O, Ls, m.n_heads / ex.world,
                                         m.n_kv_heads / ex.world, hd, st, B),
            "attention");
        }
        break;
      case OP_O:
        if (a.rec) a.rec->use((int)k, LP[l].ids[1], tt.n_base);
        cur_gemm = 4 * l + 1;
        shrink(ex.O, nq, nq, l, 1);
        {
          const int e0 = P0(KC_GEMM_O);
          K(KC_GEMM_O, e0, 2.0 * Sd * d * ((double)nq + r * lora_n(l, {T_O}) / d),
            2.0 * ((double)d * nq + Sd * nq) + 8.0 * Sd * d,
            resid_gemm(LP[l].o), "gemm_o");
        }
        break;
      case OP_MLP_NORM:
        rec({tt.norm2[l]});
        {
          const int e0 = P0();
          K(KC_RMSNORM, e0, 0, Sd * d * 6 + 2.0 * d,
            rmsnorm_launch(ex.X, Wp(tt.norm2[l]), ex.Xn, S, d, ex.eps, st), "rmsnorm");
        }
        break;
      case OP_GU:
        if (a.rec) a.rec->use((int)k, LP[l].ids[2], tt.n_base);
        cur_gemm = 4 * l + 2;
        shrink(ex.Xn, d, d, l, 2);
        {
          const int e0 = P0(KC_GEMM_GU);
          K(KC_GEMM_GU, e0, 2.0 * Sd * (2.0 * F * d + r * lora_n(l, {T_GATE, T_UP})),
            2.0 * (2.0 * F * d + Sd * d + Sd * F), launch(LP[l].gu, EPI_SILU),
            "gemm_gate_up");
        }
        break;
      case OP_ACT:  // fused into the gate/up epilogue
        break;
      case OP_DOWN:
        if (a.rec) a.rec->use((int)k, LP[l].ids[3], tt.n_base);
        cur_gemm = 4 * l + 3;
        shrink(ex.Hb, F, F, l, 3);
        {
          const int e0 = P0(KC_GEMM_DOWN);
          K(KC_GEMM_DOWN, e0, 2.0 * Sd * ((double)d * F + r * lora_n(l, {T_DOWN})),
            2.0 * ((double)d * F + Sd * F) + 8.0 * Sd * d,
            resid_gemm(LP[l].down), "gemm_down");
        }
        break;
      case OP_FNORM:  // fused into the head kernel (fp32 last-row norm)
        break;
      case OP_HEAD:  // the argmax key was zeroed by the embed kernel of this forward
        rec({tt.fnorm, tt.head});  // final_norm is fused into the head kernel
        {
          const int e0 = P0();
          // logits layout [world][B][Vl]: this rank's slices contiguous for the allgather
          K(KC_HEAD, e0, 2.0 * B * Vl * d, 2.0 * Vl * d + 4.0 * B * Vl,
            head_launch(ex.X + (size_t)(Ls - 1) * d, (size_t)Ls * d, B, Wp(tt.fnorm), Wp(tt.head),
                        Vl, d, ex.eps, ex.logits + (size_t)ex.rank * B * Vl, Vl, ex.key,
                        ex.rank * Vl, ex.num_sms, st),
            "head");
        }
        break;
      case OP_LOGITS_AG:
        tp_allgather_logits(ex, a.comm, B);
        break;
      case OP_ARGMAX:  // fused: atomicMax of packed keys in the head kernel
        tp_argmax_reduce(ex, a.comm, ex.key, B);
        break;
    }
  }
}

// ---------------- decode continuation ----------------
// One step = embed, L x (shrink?, QKV, attention, shrink?, O, shrink?, GU,
// shrink?, down), head (+ logits save): a fixed launch sequence over device
// state, captured once per (adapter, scale, logits) as a CUDA graph.
static void enqueue_decode_step(Exec& ex, const TensorTable& tt, float lora_scale,
                                bool want_logits) {
  const ModelShape& m = ex.m;
  Exec::Decode& D = ex.dec;
  cudaStream_t s = ex.compute;
  const int L = m.n_layers, d = m.d_model, hd = m.head_dim(), F = m.d_ff;
  if ((D.cap + 127) / 128 > 128) fail(1, "decode cache longer than 16384 positions");
  const int nq = m.n_heads * hd, nkv = m.n_kv_heads * hd;
  const int r = tt.lora_rank;
  auto W = [&](int id) { return id >= 0 ? reinterpret_cast<const bf16*>(ex.wptr[id]) : nullptr; };
  auto la = [&](int l, int t) { return r ? W(tt.lora_a[l][t]) : nullptr; };
  auto lb = [&](int l, int t) { return r ? W(tt.lora_b[l][t]) : nullptr; };
  float* T = D.T;  // [7][64]
  auto Tp = [&](int t) { return T + 64 * t; };
  cuda_check(dec_embed_launch(D.st, W(tt.embed), ex.X, d, D.toks, s), "dec_embed");
  ++ex.launches;
  // the LoRA shrink of a GEMV's input rides in the GEMV's launch (first CTAs)
  auto shrink = [&](DecGemv& gv, int l, int which, std::initializer_list<int> ts) {
    DecShrink& a = gv.sh;
    memset(&a, 0, sizeof a);
    for (int t : ts)
      if (la(l, t)) {
        a.A[a.nt] = la(l, t);
        a.T[a.nt] = Tp(t);
        ++a.nt;
      }
    a.r = r;
    gv.nsh = a.nt ? dec_shrink_ctas(a.nt, r) : 0;
    gv.sh_scale = lora_scale;
    gv.sh_cnt = D.shcnt + 4 * l + which;
    gv.st = D.st;
  };
  for (int l = 0; l < L; ++l) {
    const bf16 *g1 = W(tt.norm1[l]), *g2 = W(tt.norm2[l]);
    bf16* kc = D.kc + (size_t)l * D.cap * nkv;
    bf16* vc = D.vc + (size_t)l * D.cap * nkv;
    // ---- attention block ----
    DecGemv g;
    memset(&g, 0, sizeof g);
    shrink(g, l, 0, {T_Q, T_K, T_V});
    g.X = ex.X;
    g.g = g1;
    g.eps = ex.eps;
    g.K = d;
    g.npairs = (nq + 2 * nkv) / 2;
    const int tq[3] = {T_Q, T_K, T_V};
    for (int i = 0; i < 3; ++i) {
      g.W[i] = W(tt.proj[l][tq[i]]);
      g.B[i] = lb(l, tq[i]);
      g.T[i] = g.B[i] ? Tp(tq[i]) : nullptr;
    }
    g.r = r;
    g.nq = nq;
    g.nkv = nkv;
    g.hd = hd;
    g.rope = ex.rope;
    g.q = D.q;
    g.kc = kc;
    g.vc = vc;
    g.st = D.st;
    cuda_check(dec_gemv_launch(g, DEC_QKV, ex.num_sms, s), "dec_qkv");
    DecAttn at;
    memset(&at, 0, sizeof at);
    at.q = D.q;
    at.kc = kc;
    at.vc = vc;
    at.ldkv = nkv;
    at.H = m.n_heads;
    at.KV = m.n_kv_heads;
    at.hd = hd;
    at.scale_log2 = 1.4426950408889634f / sqrtf((float)hd);
    at.st = D.st;
    at.part = D.part;
    at.cnt = D.cnt;
    at.out = D.att;
    cuda_check(dec_attn_launch(at, D.cap, s), "dec_attn");
    DecGemv o;
    memset(&o, 0, sizeof o);
    shrink(o, l, 1, {T_O});
    o.xin = D.att;
    o.K = nq;
    o.N = d;
    o.npairs = (d + 1) / 2;
    o.W[0] = W(tt.proj[l][T_O]);
    o.B[0] = lb(l, T_O);
    o.T[0] = o.B[0] ? Tp(T_O) : nullptr;
    o.r = r;
    o.Xout = ex.X;
    cuda_check(dec_gemv_launch(o, DEC_RESID, ex.num_sms, s), "dec_o");
    // ---- MLP block ----
    DecGemv gu;
    memset(&gu, 0, sizeof gu);
    shrink(gu, l, 2, {T_GATE, T_UP});
    gu.X = ex.X;
    gu.g = g2;
    gu.eps = ex.eps;
    gu.K = d;
    gu.npairs = F;
    gu.W[0] = W(tt.proj[l][T_GATE]);
    gu.W[1] = W(tt.proj[l][T_UP]);
    gu.B[0] = lb(l, T_GATE);
    gu.B[1] = lb(l, T_UP);
    gu.T[0] = gu.B[0] ? Tp(T_GATE) : nullptr;
    gu.T[1] = gu.B[1] ? Tp(T_UP) : nullptr;
    gu.r = r;
    gu.h = D.h;
    cuda_check(dec_gemv_launch(gu, DEC_GU, ex.num_sms, s), "dec_gu");
    DecGemv dn;
    memset(&dn, 0, sizeof dn);
    shrink(dn, l, 3, {T_DOWN});
    dn.xin = D.h;
    dn.K = F;
    dn.N = d;
    dn.npairs = (d + 1) / 2;
    dn.W[0] = W(tt.proj[l][T_DOWN]);
    dn.B[0] = lb(l, T_DOWN);
    dn.T[0] = dn.B[0] ? Tp(T_DOWN) : nullptr;
    dn.r = r;
    dn.Xout = ex.X;
    cuda_check(dec_gemv_launch(dn, DEC_RESID, ex.num_sms, s), "dec_down");
    ex.launches += 5;  // qkv, attention (+ in-kernel combine), o, gu, down
  }
  cuda_check(head_launch(ex.X, 0, 1, W(tt.fnorm), W(tt.head), m.vocab, d, ex.eps, ex.logits,
                         m.vocab, &D.st->key, 0, ex.num_sms, s),
             "dec_head");
  ++ex.launches;
  if (want_logits) {
    cuda_check(dec_save_logits_launch(D.st, ex.logits, D.logits_all, m.vocab, s), "dec_logits");
    ++ex.launches;
  }
}

void run_decode(Exec& ex, const TensorTable& tt, int n_steps, float lora_scale, const void* akey,
                uint64_t gen, bool want_logits) {
  Exec::Decode& D = ex.dec;
  if (!D.kc) fail(1, "decode not enabled on this template (tidal_template_enable_decode)");
  if (D.prompt_len <= 0) fail(1, "decode must follow a single-prompt prefill on this template");
  if (D.prompt_akey != akey || D.prompt_gen != gen)
    fail(1, "decode must use the adapter (and template state) of the preceding prefill");
  if (n_steps < 1 || n_steps > D.max_new || D.prompt_len + n_steps > D.cap)
    fail(1, "n_steps out of range (1..max_new_tokens, prompt + steps <= cache rows)");
  cudaStream_t s = ex.compute;
  // device state: the prefill's argmax key is the first decode input
  DecodeState init;
  memset(&init, 0, sizeof init);
  init.pos0 = D.prompt_len;
  cuda_check(cudaMemcpyAsync(D.st, &init, sizeof init, cudaMemcpyHostToDevice, s), "state");
  cuda_check(cudaMemcpyAsync(&D.st->key, ex.key, 8, cudaMemcpyDeviceToDevice, s), "state key");
  cuda_check(cudaMemsetAsync(D.shcnt, 0, 4ull * 4 * ex.m.n_layers, s), "shrink counters");
  const auto gkey = std::make_tuple(akey, gen, tt.lora_rank, tt.lora_mask, lora_scale,
                                    want_logits ? 1 : 0);
  if (!D.gexec || D.gkey != gkey) {
    if (D.gexec) cudaGraphExecDestroy(D.gexec);
    D.gexec = nullptr;
    cudaGraph_t graph = nullptr;
    const int l0 = ex.launches;
    cuda_check(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "begin capture");
    try {
      enqueue_decode_step(ex, tt, lora_scale, want_logits);
    } catch (...) {
      cudaStreamEndCapture(s, &graph);
      if (graph) cudaGraphDestroy(graph);
      throw;
    }
    cuda_check(cudaStreamEndCapture(s, &graph), "end capture");
    cuda_check(cudaGraphInstantiate(&D.gexec, graph, 0), "graph instantiate");
    cudaGraphDestroy(graph);
    D.gkey = gkey;
    D.launches_per_step = ex.launches - l0;
    ex.launches = l0;
  }
  for (int i = 0; i < n_steps; ++i) cuda_check(cudaGraphLaunch(D.gexec, s), "graph launch");
  cuda_check(dec_finish_launch(D.st, D.toks, s), "dec_finish");
  ex.launches += n_steps * D.launches_per_step + 1;
}

// ---------------- NUMA binding ----------------
static bool parse_cpulist(const std::string& s, cpu_set_t* set) {
  CPU_ZERO(set);
  std::stringstream ss(s);
  std::string part;
  bool any = false;
  while (std::getline(ss, part, ',')) {
    int a = 0, b = 0;
    if (sscanf(part.c_str(), "%d-%d", &a, &b) == 2) {
    } else if (sscanf(part.c_str(), "%d", &a) == 1) {
      b = a;
    } else {
      continue;
    }
    for (int c = a; c <= b && c < CPU_SETSIZE; ++c) {
      CPU_SET(c, set);
      any = true;
    }
  }
  return any;
}

NumaGuard::NumaGuard(int device) {
  static_assert(sizeof(cpu_set_t) <= sizeof(saved), "cpu_set_t too large");
  char bus[32] = {0};
  if (cudaDeviceGetPCIBusId(bus, sizeof bus, device) != cudaSuccess) return;
  for (char* c = bus; *c; ++c) *c = (char)tolower(*c);
  std::ifstream f(std::string("/sys/bus/pci/devices/") + bus + "/local_cpulist");
  std::string line;
  if (!f || !std::getline(f, line)) return;
  cpu_set_t want, avail;
  if (!parse_cpulist(line, &want)) return;
  if (sched_getaffinity(0, sizeof(cpu_set_t), reinterpret_cast<cpu_set_t*>(saved)) != 0) return;
  CPU_AND(&avail, &want, reinterpret_cast<cpu_set_t*>(saved));
  if (CPU_COUNT(&avail) == 0) return;
  if (sched_setaffinity(0, sizeof(cpu_set_t), &avail) == 0) active = true;
}

NumaGuard::~NumaGuard() {
  if (active) sched_setaffinity(0, sizeof(cpu_set_t), reinterpret_cast<cpu_set_t*>(saved));
}

}  // namespace tidal
