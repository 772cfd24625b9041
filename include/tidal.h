/* tidal.h — C-ABI of the B200-native Tidal template-start prefill library.
 *
 * The calls follow the paper's problem statement (§3 "Invocation
 * workflow", lines 356-367): trace a first run, build a function template
 * with some weights GPU-resident, attach a dynamic component (LoRA adapter),
 * then invoke: non-resident weights stream from a pinned host pool in traced
 * access order while prefill runs, gated by per-group CUDA events.
 *
 *   tidal_trace           lax inference tracing -> weight access order
 *                         (§4.1)
 *   tidal_template_create access-ordered layout, resident prefix (budget or
 *                         Eq. 1), pinned pool, transfer
 *                         groups (§6), kernel pre-load (§5.1)
 *   tidal_attach_lora     bind a dynamic adapter (§5.2)
 *   tidal_invoke_prefill  adaptive fork + overlapped streaming + prefill,
 *                         returns last-position logits and the first token
 *                         (§5.2)
 *
 * Conventions (all entry points):
 *   - Every function returns tidal_status and never throws across the ABI;
 *     on a non-OK status tidal_last_error() returns a thread-local message.
 *   - Handles are opaque; each *_create has a NULL-safe *_destroy.
 *   - Inputs are BORROWED for the duration stated on each call; outputs are
 *     caller-owned buffers.  Dumps use the two-call pattern: pass cap=0 to
 *     learn *needed, then call again with a buffer of that size.
 *   - Pointers named host_* are host memory; dev_* are device memory of the
 *     template's device.  Sizes are in bytes unless named n_*.
 *   - One invoke in flight per template (the streaming arena is per template).
 *   - There is no CPU fallback: every compute step runs in this library's
 *     sm_100a kernels; a build without them fails at load time.
 *   - device = -1 selects DRY mode for tidal_trace / tidal_template_create:
 *     the planner runs on the host only (no GPU, no pool), so traces and plans
 *     can be checked on a CPU-only box.  A dry template cannot be invoked.
 */
#ifndef TIDAL_H
#define TIDAL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  TIDAL_OK = 0,
  TIDAL_ERR_INVALID = 1,    /* bad argument (NULL, out of range, wrong mode) */
  TIDAL_ERR_OOM = 2,        /* device or pinned-host allocation failed; never silent eviction */
  TIDAL_ERR_CUDA = 3,       /* CUDA runtime/driver error */
  TIDAL_ERR_NCCL = 4,       /* collective error (tensor-parallel ranks) */
  TIDAL_ERR_STRUCTURE = 5,  /* weights/adapter do not match the model structure:
                               template invalidation */
  TIDAL_ERR_RESIDENCY = 6,  /* debug checker: an op read a group that had not landed */
  TIDAL_ERR_COW = 7,        /* template bytes changed (copy-on-write invariant) */
  TIDAL_ERR_BUFSZ = 8,      /* caller buffer too small (see *needed) */
  TIDAL_ERR_NUMERIC = 9     /* NaN in the logits (argmax undefined, reading A5) */
} tidal_status;

const char* tidal_last_error(void);
const char* tidal_version(void);

/* Llama-style decoder shape.  head_dim = d_model / n_heads (64 or 128). */
typedef struct {
  int n_layers, d_model, n_heads, n_kv_heads, d_ff, vocab;
  float rope_theta; /* 1e4 Llama-2 shapes, 5e5 Llama-3 */
  float rms_eps;    /* 1e-5 (reading A1) */
  int tie_embeddings;
} tidal_model_config;

/* One weight tensor, bf16, row-major in the HF shape ([out,in] for linears).
 * Either host_bf16 (borrowed, any host memory) or fill (called synchronously
 * by tidal_trace/tidal_template_create to write exactly `bytes` into dst,
 * e.g. straight into the pinned pool) must be set. */
typedef void (*tidal_fill_fn)(void* dst, size_t bytes, int tensor_index, void* ctx);
typedef struct {
  const char* name;      /* canonical HF name (R0), e.g. model.layers.3.mlp.up_proj.weight */
  const void* host_bf16; /* nullable if fill != NULL */
  size_t bytes;          /* must equal 2 * prod(rank-local shape) */
} tidal_host_tensor;

typedef struct tidal_model tidal_model;
typedef struct tidal_trace_rec tidal_trace_rec; /* handle returned by tidal_trace */
typedef struct tidal_template tidal_template;
typedef struct tidal_adapter tidal_adapter;
typedef struct tidal_comm tidal_comm;

/* Describe a model.  `w[0..n)` must be exactly the R0 tensor set for the
 * (rank-local) shapes; missing/extra/mis-sized -> TIDAL_ERR_STRUCTURE.
 * `checkpoint` names the source (provenance of INIT lines).  `fill`/`ctx`
 * are optional (see tidal_host_tensor).  world/rank: tensor-parallel shard
 * this model holds (1/0 for a single GPU).  Everything is borrowed until the
 * last tidal_trace / tidal_template_create that uses the model returns. */
tidal_status tidal_model_create(const tidal_model_config* cfg, const tidal_host_tensor* w, int n,
                                const char* checkpoint, tidal_fill_fn fill, void* fill_ctx,
                                int world, int rank, tidal_model** out);
void tidal_model_destroy(tidal_model* m);

/* SPEC trace_inference: run the model once and record the
 * order in which weights are first read (aliases collapse; never-read at the
 * tail) and the kernel set.  device >= 0: a real first run on that GPU — all
 * weights copied in registration order, then the forward (the
 * load-then-infer "PyTorch-pin" path); its logits/token/
 * timing are returned through the optional outputs.  device = -1: dry. */
tidal_status tidal_trace(tidal_model* m, const int32_t* host_tokens, int n_tokens, int device,
                             float* host_logits_out /*[vocab], nullable*/,
                             int32_t* host_token_out /*nullable*/,
                             double* cold_ttft_ms_out /*nullable*/, tidal_trace_rec** out);
void tidal_trace_destroy(tidal_trace_rec* t);
/* INIT <name> <fnv1a64(provenance)> <bytes> lines in registration order, then
 * ACCESS <k> <name> <op>#<op-ordinal> in access order. */
tidal_status tidal_trace_dump(const tidal_trace_rec* t, char* buf, size_t cap, size_t* needed);

enum { TIDAL_GROUPS_PER_LAYER = 0, TIDAL_GROUPS_MAX_TRANSFERS = 1, TIDAL_GROUPS_PER_TENSOR = 2 };

typedef struct {
  uint64_t resident_bytes; /* budget, rounded DOWN to whole weights; UINT64_MAX = all */
  int eq1;                 /* 1: resident = Eq. 1's M_prefetch = max(M - floor(T*B), 0),
                              rounded UP to whole weights */
  double t_ttft_s;         /* Eq. 1 T_TTFT: measured warm TTFT (seconds) */
  double b_pcie_Bps;       /* Eq. 1 B_PCIe: measured H2D bytes/s */
  int group_policy;        /* TIDAL_GROUPS_* (default per_layer) */
  int max_transfers;       /* for TIDAL_GROUPS_MAX_TRANSFERS (paper: 1200 -> 300) */
  int max_tokens;          /* largest prompt the activation arena must hold */
  int device;              /* CUDA device, or -1 for DRY (planner only) */
  tidal_comm* comm;        /* NULL for one GPU */
} tidal_template_opts;

/* SPEC generate_template: layout = static weights in access
 * order (256-B aligned offsets), resident prefix, pinned host pool holding the
 * whole image in layout order (NUMA-local to the device), one device buffer in
 * layout order whose prefix is the read-only template and whose suffix is the
 * streaming arena, one-time H2D of the prefix, events, eager kernel load and
 * warm launches (A4/A8).  `trace` and the model are borrowed for the call. */
tidal_status tidal_template_create(tidal_model* m, const tidal_trace_rec* t,
                                   const tidal_template_opts* opts, tidal_template** out);
/* Adapt the template size in place ("dynamically adapts this value",
 * PAPER.md line 576): re-plans the resident prefix from opts (resident_bytes
 * or eq1 fields; other fields ignored) and copies any newly resident bytes. */
tidal_status tidal_template_resize(tidal_template* tpl, const tidal_template_opts* opts);
/* Keep-alive of a dynamic function (§5.2 "Keep-alive of dynamic
 * function", lines 579-587): after an invocation every streamed weight is
 * already on the device, so the whole layout is marked resident (no copy) and
 * later invocations stream only their dynamic adapter.  Fails with
 * TIDAL_ERR_INVALID if the streaming arena does not hold valid weights (no
 * successful invoke since a fault-injection run). */
tidal_status tidal_template_keep_alive(tidal_template* tpl);
/* Loading-order ablation (§7.4): copy the transfer
 * groups in traced access order (default), reverse order, or registration
 * (initialisation) order.  Barriers stay correct in every order: each op waits
 * on the needed group that is copied last. */
enum { TIDAL_ORDER_TRACED = 0, TIDAL_ORDER_REVERSE = 1, TIDAL_ORDER_REGISTRATION = 2 };
tidal_status tidal_set_load_order(tidal_template* tpl, int order);
void tidal_template_destroy(tidal_template* tpl);

/* Canonical adapter layout for (rank, target_mask): tensors in adapter access
 * order, 256-B aligned.  Fills up to `cap` slots; *n = number of tensors,
 * *total_bytes = buffer size.  Slot names point into library memory valid
 * until the template is destroyed. */
typedef struct { const char* name; uint64_t offset; uint64_t bytes; int rows, cols; } tidal_slot;
tidal_status tidal_adapter_layout(const tidal_template* tpl, int rank, uint32_t target_mask,
                                  tidal_slot* slots, int cap, int* n, uint64_t* total_bytes);

/* A LoRA adapter: A [r,in], B [out,r] per targeted module (bit i of
 * target_mask: q,k,v,o,gate,up,down).  host_pinned holds the canonical layout
 * (tidal_adapter_layout) in page-locked memory (tidal_host_alloc); it is
 * borrowed until tidal_adapter_destroy and must not change while an invoke is
 * in flight.  Dynamic by construction: never resident in the template
 * (SPEC.md:236).  Host-only work (validation + plan), inside the TTFT window. */
typedef struct {
  int rank;               /* 8..64, multiple of 8 */
  float scale;            /* alpha / r */
  uint32_t target_mask;   /* 0x7F = all 7 projections */
  const void* host_pinned;
  uint64_t bytes;
  const char* checkpoint; /* provenance, e.g. "adapter:3" */
} tidal_lora_desc;
tidal_status tidal_attach_lora(tidal_template* tpl, const tidal_lora_desc* d, tidal_adapter** out);
void tidal_adapter_destroy(tidal_adapter* a);

/* ACTION / GROUP / BARRIER / BYTES lines
 * for this template with the given adapter (nullable). */
tidal_status tidal_plan_dump(const tidal_template* tpl, const tidal_adapter* a, char* buf,
                             size_t cap, size_t* needed);

typedef struct {
  double ttft_host_ms;      /* host clock: invoke entry -> token on host */
  double device_ms;         /* device events: first H2D/compute -> logits D2H done */
  double h2d_first_ms, h2d_last_ms;      /* relative to the invoke's start event */
  double compute_first_ms, compute_last_ms;
  uint64_t bytes_streamed, bytes_resident, bytes_adapter;
  int n_copies;
  int n_kernels;            /* kernels this library launched for the invoke */
} tidal_stats;

/* Run the first-token prefill.  host_tokens[0..n_tokens) in [0, vocab),
 * 1 <= n_tokens <= max_tokens.  Synchronous: returns after the token (and the
 * logits, if host_logits_out != NULL, [vocab] fp32) are on the host.  All TP
 * ranks call it with identical tokens.  `a` may be NULL (no adapter). */
tidal_status tidal_invoke_prefill(tidal_template* tpl, const tidal_adapter* a,
                                  const int32_t* host_tokens, int n_tokens,
                                  float* host_logits_out, int32_t* host_token_out,
                                  tidal_stats* stats);

/* Batched prefill (§7.2 "TTFT with varied input lengths and batch
 * sizes", Fig. ttft-bs: batch of prompts of one input length): n_seqs prompts of
 * seq_len tokens each, host_tokens row-major [n_seqs][seq_len]; every prompt
 * attends only to itself and its positions restart at 0.  The weights are
 * streamed once for the whole batch.  1 <= n_seqs <= 64 and n_seqs * seq_len
 * <= max_tokens.  Outputs: host_tokens_out[n_seqs] (first token of each
 * prompt) and, if non-NULL, host_logits_out[n_seqs][vocab].  Same
 * synchronisation, TP and error rules as tidal_invoke_prefill, which is the
 * n_seqs = 1 case. */
tidal_status tidal_invoke_prefill_batch(tidal_template* tpl, const tidal_adapter* a,
                                        const int32_t* host_tokens, int n_seqs, int seq_len,
                                        float* host_logits_out, int32_t* host_tokens_out,
                                        tidal_stats* stats);

/* ---- decode continuation (§7 l.831, 849-851) ----
 * Greedy decoding after the first token.  tidal_template_enable_decode
 * allocates a KV cache of (max_tokens + max_new_tokens) rows per layer on the
 * template's device (K after RoPE and V, bf16, [L][rows][n_kv_heads*head_dim])
 * and extends the RoPE table; from then on every single-prompt
 * tidal_invoke_prefill also stores its K and V into the cache (from the QKV
 * GEMM epilogue).  tidal_invoke_decode continues the most recent such prefill:
 * it feeds the prefill's first token at position n_tokens and generates
 * n_steps further tokens, each step a captured CUDA graph (embed, per layer
 * LoRA shrinks + HBM-bound GEMVs with fused RMSNorm / RoPE / SiLU*mul /
 * residual + attention over the cache, head + argmax) replayed without a host
 * round trip.  All weights are read from the device (the prefill left the
 * streamed ones in the arena), so a step is bound by model bytes / HBM
 * bandwidth.  Outputs: tokens_out[n_steps] (token i generated by step i);
 * logits_out (nullable) [n_steps][vocab] fp32.  Synchronous.
 * Errors: TIDAL_ERR_INVALID when decode is not enabled, no single-prompt
 * prefill preceded, the adapter differs from the prefill's, n_steps is out of
 * [1, max_new_tokens], or the template is tensor-parallel (not implemented). */
typedef struct {
  double device_ms;                  /* all steps, CUDA events */
  double per_token_ms;
  uint64_t weight_bytes_per_token;   /* weights read per step (embedding: one row) */
  uint64_t kv_bytes_last_token;      /* K and V read by the last step */
  int n_kernels;                     /* kernels launched (graph nodes x steps + 1) */
} tidal_decode_stats;
tidal_status tidal_template_enable_decode(tidal_template* tpl, int max_new_tokens);
tidal_status tidal_invoke_decode(tidal_template* tpl, const tidal_adapter* a, int n_steps,
                                 int32_t* tokens_out, float* logits_out,
                                 tidal_decode_stats* stats);

/* ---- cross-process templates (§3, §5.1: a
 * template server keeps function templates on the GPU and function processes
 * fork from them over CUDA IPC) ----
 * Device templates live on CUDA virtual memory: one address range per
 * template backed by equal physical chunks (~1/64 of the layout, a multiple of
 * the allocation granularity, <= 512 MB) with POSIX-fd shareable handles.
 *
 * tidal_template_export: fds[0..n) of the chunks lying wholly inside the
 * resident prefix (address order) and shared_bytes = n * chunk.  With
 * fds == NULL only *n_fds / *shared_bytes are returned (size query).  The
 * caller owns the fds (close them after passing them on, e.g. SCM_RIGHTS).
 * From then on the template refuses a resize below shared_bytes (importers
 * read those bytes as their template); it must outlive its importers.
 * *fingerprint identifies the shared prefix: FNV-1a over every tensor below
 * shared_bytes (name, offset, bytes, provenance = checkpoint:name:shape).
 * Errors: INVALID (dry / no VMM / re-export of an import), BUFSZ (cap < n).
 *
 * tidal_template_import: the importer builds the same plan from the same
 * (model, trace, opts) and maps the n_fds chunks READ-ONLY at offset 0 of its
 * own layout range; the rest of its resident prefix (less than one chunk)
 * is copied from its pinned pool and its streaming arena is private, so an
 * invocation writes only private memory (copy-on-write by construction).
 * Errors: STRUCTURE if the chunks do not cover exactly shared_bytes of this
 * layout, shared_bytes exceeds the plan's resident prefix, or `fingerprint`
 * (the exporter's) differs from this plan's prefix fingerprint (another
 * trace, layout, checkpoint or weights of the same size); INVALID for dry
 * / tensor-parallel opts.  Everything else is as tidal_template_create. */
tidal_status tidal_template_export(tidal_template* tpl, int* fds, int cap, int* n_fds,
                                   uint64_t* shared_bytes, uint64_t* fingerprint /*nullable*/);
tidal_status tidal_template_import(tidal_model* model, const tidal_trace_rec* trace,
                                   const tidal_template_opts* opts, const int* fds, int n_fds,
                                   uint64_t shared_bytes, uint64_t fingerprint,
                                   tidal_template** out);

/* ---- device memory ---- */
/* Route the library's device allocations through the caller (e.g. PyTorch's
 * caching allocator), process-wide, from the next allocation on (SURVEY.md
 * §8(b); north_star "PyTorch is used only for device memory, streams and
 * process groups"): a template's layout buffer (read-only template prefix +
 * streaming arena), its activations and scratch, and the adapter arena.
 * alloc(bytes, device, ctx) returns a device pointer (>= 256-B aligned) or
 * NULL (-> TIDAL_ERR_OOM); free_(ptr, device, ctx) releases it.  Every block
 * is returned to the allocator that produced it, even if the hook changes
 * later.  Pass (NULL, NULL, NULL) to return to cudaMalloc.  A template whose
 * layout buffer comes from a hook is not on CUDA VMM and cannot be exported
 * (tidal_template_export -> INVALID).  Errors: INVALID (one of the two NULL). */
tidal_status tidal_set_device_allocator(void* (*alloc)(size_t bytes, int device, void* ctx),
                                       void (*free_)(void* ptr, int device, void* ctx),
                                       void* ctx);

/* ---- pinned host memory for adapters / pools (cudaHostAlloc) ---- */
tidal_status tidal_host_alloc(uint64_t bytes, void** out);
void tidal_host_free(void* p);

/* ---- tensor parallelism (NCCL over NVLink) ---- */
tidal_status tidal_comm_unique_id(void* out128);
tidal_status tidal_comm_create(int world, int rank, const void* unique_id128, int device,
                               tidal_comm** out);
/* In-process ranks (one host thread per rank, SURVEY.md §8(e) collectives C1-C4
 * over device pointers): every rank of one process calls this with the same
 * `group` string and world; ranks may share a device (TP=N on one GPU, used by
 * the tests) or sit on peer-accessible devices.  Collectives rendezvous on the
 * host (each rank's invoke must run concurrently on its own thread; a peer
 * missing for 120 s gives TIDAL_ERR_NCCL) and sum in rank order, so all ranks
 * hold bit-identical results.  world must be <= 8. */
tidal_status tidal_comm_create_local(int world, int rank, const char* group, int device,
                                     tidal_comm** out);
void tidal_comm_destroy(tidal_comm* c);
/* Precision of the row-parallel allreduces C1/C2 (after o_proj and down_proj,
 * "fp32 for parity, bf16 measured as an option").
 * TIDAL_DTYPE_F32 (default): the fp32 residual stream itself is allreduced
 * (rank 0 carries the residual, the other ranks their partial sums only).
 * TIDAL_DTYPE_BF16: every rank's partial sum is rounded once to bf16, reduced
 * in bf16 (half the NVLink bytes) and added to the fp32 residual.  The embed
 * allreduce (C3) stays fp32.  No effect when world == 1.  Takes effect at the
 * next invoke; all ranks must set the same value.  Errors: INVALID. */
enum { TIDAL_DTYPE_F32 = 0, TIDAL_DTYPE_BF16 = 1 };
/* Self-test of a communicator's collectives (allreduce f32 / bf16, u64 max,
 * logits allgather) on n-element device buffers holding small integers, so
 * every expected value is exact.  All ranks call it at once (NCCL ranks in
 * their processes, local ranks on their threads).  tidal_comm_create also
 * builds a one-rank NCCL communicator at world 1, so the NCCL binding can be
 * exercised on a single GPU.  Errors: NCCL (mismatch or NCCL failure),
 * INVALID (a world-1 local communicator has no implementation). */
tidal_status tidal_comm_selftest(tidal_comm* c, uint64_t n);
tidal_status tidal_set_allreduce_dtype(tidal_template* tpl, int dtype);

/* ---- invariants and fault injection (test support) ---- */
enum {
  TIDAL_DEBUG_POISON = 1,      /* NaN-poison the streaming arena before each invoke */
  TIDAL_DEBUG_SKIP_BARRIER = 2,/* drop the wait on group `arg` and delay its copy */
  TIDAL_DEBUG_SCRUB_L2 = 4,    /* write 512 MB before each invoke (timing hygiene) */
  TIDAL_DEBUG_SERIAL = 8,      /* load-then-infer: compute waits for every copy first
                                  (the paper's "PyTorch-pin" baseline) */
  TIDAL_DEBUG_PROFILE = 16,    /* CUDA events around every kernel on the compute stream */
  TIDAL_DEBUG_PROFILE_GEMM = 32,/* events around the tensor-core GEMMs only (low overhead) */
  TIDAL_DEBUG_NO_GRAPH = 64,   /* enqueue the invocation eagerly instead of replaying its
                                  captured CUDA graph (single-GPU invocations are captured
                                  once per plan / shape / adapter buffer / scale and
                                  replayed; profiling and fault injection are always eager) */
  TIDAL_DEBUG_TIMELINE = 128   /* timing events at every copy-group end (copy stream) and
                                  every op start (compute stream, after its barrier wait);
                                  read with tidal_timeline_read (always eager) */
};
/* Timeline of the last invocation run with TIDAL_DEBUG_TIMELINE, in ms from
 * the invocation's first event: group_end_ms[g] when transfer group g landed
 * (plan group index), op_start_ms[k] when op k of the canonical sequence could
 * start (previous op done and its barrier satisfied), and *end_ms when the
 * token was ready.  Either array may be NULL (size query: *n_groups, *n_ops).
 * Errors: INVALID if no timeline was recorded, BUFSZ if a cap is too small. */
tidal_status tidal_timeline_read(tidal_template* tpl, double* group_end_ms, int cap_groups,
                                 double* op_start_ms, int cap_ops, int* n_groups, int* n_ops,
                                 double* end_ms);
/* Per-kernel-class totals accumulated by invokes run with TIDAL_DEBUG_PROFILE:
 * device time (events on the launching stream), launches, and the ALGORITHMIC
 * flops and HBM bytes of those launches.  Fills up to
 * `cap` entries (*n = number of classes); reset != 0 clears the totals. */
typedef struct {
  const char* name;
  double total_ms;
  long launches;
  double flops;
  double bytes;
} tidal_kernel_time;
tidal_status tidal_profile_read(tidal_template* tpl, tidal_kernel_time* out, int cap, int* n,
                                int reset);
tidal_status tidal_set_debug(tidal_template* tpl, int flags, int arg);
/* 64-bit checksum of the resident template region computed on the device
 * (the copy-on-write invariant: unchanged across invocations). */
tidal_status tidal_template_checksum(tidal_template* tpl, uint64_t* out);
/* Device pointer of weight `name` in the fork pointer table (tests only). */
tidal_status tidal_weight_ptr(const tidal_template* tpl, const char* name, void** dev_out);

#ifdef __cplusplus
}
#endif
#endif /* TIDAL_H */
