// runtime.h — device execution context and the op launcher.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "kernels.h"
#include "plan.h"

namespace tidal {

struct Status {
  int code = 0;
  std::string msg;
};
struct Error {
  int code;
  std::string msg;
};
[[noreturn]] void fail(int code, const std::string& msg);
void cuda_check(cudaError_t e, const char* what);

// Device memory of templates (layout buffer when not on CUDA VMM, activations,
// adapter arena, scratch): through the caller's allocator when one is set
// (tidal_set_device_allocator), else cudaMalloc.  dev_free returns a block to
// whichever allocator produced it.  Allocation failure -> TIDAL_ERR_OOM.
typedef void* (*DevAllocFn)(size_t bytes, int device, void* ctx);
typedef void (*DevFreeFn)(void* ptr, int device, void* ctx);
void set_device_allocator(DevAllocFn alloc, DevFreeFn free_, void* ctx);
bool device_allocator_set();
void* dev_alloc(size_t bytes, int device, const char* what);
void dev_free(void* p);

// Per-layer launch parameters, cached per (prompt length, adapter layout).
struct LayerLaunch {
  GemmParams qkv, o, gu, down;
  ShrinkPlan sh[4];  // LoRA shrink feeding qkv / o / gate_up / down
  int has_sh[4] = {0, 0, 0, 0};
  std::vector<int> ids[4];    // weight ids behind the qkv / o / gate_up / down tensor maps
  LoraPackArgs pack = {};     // lora_A of the GEMMs with in-GEMM T tiles (packed per layer)
  std::vector<int> pack_ids;  // their tensor ids (the packing waits for their groups)
};

// Device execution context: streams, activation arena, rope table, the fork
// pointer table (tensor id -> device address) and a launch-parameter cache.
constexpr int kMaxBatch = 64;  // prompts per invocation (logits / argmax buffers)

struct Exec {
  int device = -1, num_sms = 148;
  ModelShape m;
  float eps = 1e-5f, theta = 1e4f;
  int world = 1, rank = 0;
  int max_tokens = 0;
  cudaStream_t compute = nullptr, copy = nullptr;
  // activations
  float* X = nullptr;
  bf16 *Xn = nullptr, *QKV = nullptr, *O = nullptr, *Hb = nullptr;
  bf16* T[kNumTargets] = {};
  float* logits = nullptr;
  unsigned long long* key = nullptr;
  int32_t* tok = nullptr;
  float2* rope = nullptr;
  float* shrink_ws = nullptr;  // split-K partials of the LoRA shrink
  int* gemm_flags = nullptr;   // ordered split-K counters of the residual GEMMs (all 0 at rest)
  // in-GEMM LoRA shrink: per (layer, GEMM) a row-block array of T-ready flags,
  // zeroed at the start of every forward; tflag_stride ints per GEMM
  int* tflags = nullptr;
  int tflag_stride = 0;
  bool fuse_shrink = true;
  bf16* zero_b = nullptr;
  bf16* lora_pack = nullptr;   // packed lora_A of the in-GEMM T tiles, [L][per-layer stride]
  size_t pack_stride = 0;
  unsigned long long* dbg_trace = nullptr;  // TIDAL_GEMM_TRACE diagnostic timeline
  bool dbg_pending = false;
  void dbg_dump();                          // after the invocation synchronised      // [F / world][64] zeros: lora_B of an untargeted gate or up half     // T tiles inside the GEMMs (else split-K shrink + reduce launches)
  bf16* Vt = nullptr;  // V^T [KV*hd][vt_ld] (tcgen05 attention, hd = 128)
  // TP: row-parallel partial sums for the bf16 allreduce option (C1/C2 in
  // bf16): the GEMM adds into P32 (zeroed), P32 -> Pb, allreduce(Pb), X += Pb
  bool ar_bf16 = false;
  bool colocated = false;  // TP ranks share this GPU (Comm::colocated)
  float* P32 = nullptr;
  bf16* Pb = nullptr;
  int vt_ld = 0;
  std::map<std::pair<int, int>, AttnParams> attn_cache;  // per (rows, prompts)
  // decode continuation (decode.cu): KV cache filled by the prefill's QKV
  // epilogue, per-step scratch, device state, and the captured step graph
  struct Decode {
    int max_new = 0, cap = 0;         // cache rows per layer = max_tokens + max_new
    bf16 *kc = nullptr, *vc = nullptr;  // [L][cap][nkv]
    bf16 *q = nullptr, *att = nullptr, *h = nullptr;
    float* T = nullptr;               // [DEC_TSPLIT][7][64] LoRA shrink parts
    float* part = nullptr;            // attention chunk partials
    int* cnt = nullptr;               // attention chunks finished per head (0 at rest)
    int* shcnt = nullptr;             // [L][4] fused-shrink CTA counts (reset per decode)
    DecodeState* st = nullptr;
    int32_t* toks = nullptr;          // [max_new]
    float* logits_all = nullptr;      // [max_new][V]
    int prompt_len = 0;               // rows of the cache valid (last single-prompt prefill)
    const void* prompt_akey = nullptr;
    uint64_t prompt_adapter = 0;      // serial of the prefill's adapter (0: none)
    uint64_t prompt_gen = 0;
    cudaGraphExec_t gexec = nullptr;
    int launches_per_step = 0;
    std::tuple<const void*, uint64_t, int, uint32_t, float, int> gkey;
  } dec;
  // pinned host staging
  int32_t* h_tok = nullptr;
  float* h_logits = nullptr;
  unsigned long long* h_key = nullptr;
  // fork pointer table
  std::vector<void*> wptr;
  // cache: (S, lora_rank, mask, adapter arena base) -> per-layer params
  std::map<std::tuple<int, int, int, uint32_t, const void*, uint64_t>, std::vector<LayerLaunch>> cache;
  int launches = 0;
  // per-kernel-class timing (TIDAL_DEBUG_PROFILE): event pairs on the compute
  // stream around every launch, plus each launch's algorithmic flops/bytes
  bool profile = false, profile_all = false;
  std::vector<cudaEvent_t> prof_ev;
  struct ProfRec {
    int cls;
    int ev;
    double flops, bytes;
  };
  std::vector<ProfRec> prof_pending;
  struct ProfTot {
    double ms = 0, flops = 0, bytes = 0;
    long launches = 0;
  };
  std::vector<ProfTot> prof_tot;
  int prof_begin();                               // returns event-pair index, records start
  void prof_end(int cls, int ev, double flops, double bytes);
  void prof_collect();                            // after the stream synchronised

  void init(int device, const ModelShape& m, float eps, float theta, int world, int rank,
            int max_tokens);
  void enable_decode(int max_new);
  void build_rope(int rows);
  void destroy();
  const std::vector<LayerLaunch>& layer_params(const TensorTable& tt, int S, int nseq,
                                               const void* akey, uint64_t gen);
  cudaError_t attention_tc(int S, int nseq, cudaStream_t s);
};

enum KernelClass {
  KC_EMBED, KC_RMSNORM, KC_SHRINK, KC_GEMM_QKV, KC_ATTN, KC_GEMM_O, KC_GEMM_GU, KC_GEMM_DOWN,
  KC_HEAD, KC_ALLREDUCE, KC_COUNT
};
extern const char* const kKernelClassNames[KC_COUNT];

// Lax tracing: first-read order of the weights the launcher actually hands to
// its kernels (the ids behind every kernel argument / tensor map), recorded
// as the kernels are enqueued — not the planner's read lists, so tidal_trace
// can check the two against each other.
struct Recorder {
  std::vector<char> seen;
  std::vector<std::pair<int, int>> access;
  void use(int k, int id, int n_base) {
    if (id >= 0 && id < n_base && !seen[id]) {
      seen[id] = 1;
      access.emplace_back(id, k);
    }
  }
  void use(int k, const std::vector<int>& ids, int n_base) {
    for (int id : ids) use(k, id, n_base);
  }
};

// TP collectives (comm.cu), enqueued on `s`; every rank calls them in the same
// order with the same sizes.  allgather_f32: buf holds world slices of n
// floats, this rank's slice filled in place.
struct Comm {
  int world = 1, rank = 0, device = 0;
  // ranks may share a GPU (LocalComm): kernels whose CTAs wait on other CTAs
  // of the same grid (ordered split-K, in-GEMM LoRA T tiles) are not used,
  // since two ranks' persistent grids may each be only partly resident
  bool colocated = false;
  virtual ~Comm() {}
  virtual void allreduce_f32(float* buf, size_t n, cudaStream_t s) = 0;
  virtual void allreduce_bf16(bf16* buf, size_t n, cudaStream_t s) = 0;
  virtual void max_u64(unsigned long long* key, size_t n, cudaStream_t s) = 0;
  virtual void allgather_f32(float* buf, size_t n, cudaStream_t s) = 0;
};

struct RunArgs {
  const TensorTable* tt = nullptr;
  const std::vector<Op>* ops = nullptr;
  const std::vector<std::vector<int>>* barriers = nullptr;  // nullable
  const std::vector<cudaEvent_t>* events = nullptr;         // per group
  const std::vector<int>* copy_pos = nullptr;               // position of each group in the copy stream
  const std::vector<int>* group_of = nullptr;               // per tensor id: its transfer group (-1: resident)
  const std::vector<cudaEvent_t>* tl_op = nullptr;          // timeline: an event at each op start
  int skip_group = -1;                                       // fault injection
  int S = 0;     // total rows: nseq prompts of S / nseq tokens each
  int nseq = 1;
  float lora_scale = 1.f;
  const void* akey = nullptr;
  uint64_t gen = 0;
  Recorder* rec = nullptr;
  Comm* comm = nullptr;  // TP communicator (nullable when world == 1)
};

// Enqueue the forward for one prompt on exec.compute (tokens already in exec.tok).
void run_forward(Exec& ex, const RunArgs& a);

// Greedy decode of n_steps tokens continuing the last single-prompt prefill
// (whose argmax key is in ex.key[0]); all weights must be on the device.
// Tokens (and, if want_logits, [n_steps][V] logits) are left in ex.dec.toks /
// ex.dec.logits_all; returns after enqueueing (compute stream).
void run_decode(Exec& ex, const TensorTable& tt, int n_steps, float lora_scale, const void* akey,
                uint64_t gen, bool want_logits);

// Template device memory on CUDA VMM (vmm.cu): one virtual range backed by
// equal physical chunks with POSIX-fd handles; the first n_shared chunks may
// be imported read-only from another process's template.
struct VmmBuf {
  CUdeviceptr va = 0;
  size_t size = 0, chunk = 0;
  std::vector<CUmemGenericAllocationHandle> h;
  int n_shared = 0, device = -1;
};
bool vmm_available();
void vmm_alloc(VmmBuf& b, size_t bytes, int device, const int* fds, int n_shared);
void vmm_free(VmmBuf& b);
int vmm_export_fd(const VmmBuf& b, size_t chunk);

// NUMA: bind the calling thread to the CPUs local to `device` (restored by the guard).
struct NumaGuard {
  bool active = false;
  unsigned char saved[128];
  explicit NumaGuard(int device);
  ~NumaGuard();
};

}  // namespace tidal
