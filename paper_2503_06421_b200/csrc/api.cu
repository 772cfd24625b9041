// api.cu — the C-ABI (include/tidal.h): handles, template server (pinned
// pool + device template/arena), adaptive fork and the overlapped invoke.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "../../include/tidal.h"
#include "../../include/tidal_kernels.h"
#include "plan.h"
#include "runtime.h"

using namespace tidal;

namespace tidal {
bool nccl_unique_id(void* out128);
Comm* nccl_comm_create(int world, int rank, const void* id128, int device);
Comm* local_comm_create(int world, int rank, const std::string& key, int device);
void comm_selftest(Comm* c, size_t n);
}  // namespace tidal

namespace {
thread_local std::string g_err;

tidal_status set_err(int code, const std::string& msg) {
  g_err = msg;
  return (tidal_status)code;
}

#define TIDAL_TRY try {
#define TIDAL_CATCH                                         \
  }                                                         \
  catch (const Error& e) {                                  \
    return set_err(e.code, e.msg);                          \
  }                                                         \
  catch (const std::bad_alloc&) {                           \
    return set_err(TIDAL_ERR_OOM, "host allocation failed"); \
  }                                                         \
  catch (const std::exception& e) {                         \
    return set_err(TIDAL_ERR_INVALID, e.what());            \
  }                                                         \
  return TIDAL_OK;

void require(bool c, const std::string& msg, int code = TIDAL_ERR_INVALID) {
  if (!c) fail(code, msg);
}

__global__ void sleep_kernel(int us) {
  for (int i = 0; i < us; ++i) __nanosleep(1000);
}
}  // namespace

struct tidal_model {
  ModelShape shape;
  float theta = 1e4f, eps = 1e-5f;
  std::string checkpoint;
  int world = 1, rank = 0;
  TensorTable tt;
  std::vector<const void*> host;  // per base tensor id
  std::vector<int> user_index;
  tidal_fill_fn fill = nullptr;
  void* ctx = nullptr;

  void produce(int id, void* dst) const {
    const uint64_t b = tt.t[id].bytes;
    if (host[id]) {
      memcpy(dst, host[id], b);
    } else {
      require(fill != nullptr, "tensor " + tt.t[id].name + " has neither data nor fill callback");
      fill(dst, b, user_index[id], ctx);
    }
  }
};

struct tidal_trace_rec {
  TensorTable tt;
  Trace tr;
};

struct tidal_comm {
  Comm* impl = nullptr;  // NCCL (one process per GPU) or in-process ranks
  int world = 1, rank = 0, device = 0;
};

// Plan of the template with an adapter of (rank, mask) attached.  Depends only
// on the template (layout, resident prefix, generation) and (rank, mask), not on
// the adapter's bytes, so attaching a new adapter of a known shape is O(1).
struct AdapterPlan {
  TensorTable tt;
  Plan plan;
  uint64_t gen = 0;
};

struct tidal_template {
  std::map<std::pair<int, uint32_t>, std::shared_ptr<AdapterPlan>> aplans;
  ModelShape shape;
  float theta = 1e4f, eps = 1e-5f;
  int world = 1, rank = 0;
  TensorTable tt;
  Trace tr;
  TemplateChoice choice;
  Plan plan;
  uint64_t gen = 1;
  bool dry = true;
  int device = -1;
  int max_tokens = 0;
  uint8_t* pool = nullptr;
  uint8_t* dev = nullptr;
  VmmBuf vmm;                  // dev's backing when CUDA VMM is available
  uint64_t exported_bytes = 0; // prefix bytes handed to other processes (never rewritten)
  uint64_t shared_bytes = 0;   // importer: prefix bytes mapped read-only from the exporter
  Exec ex;
  std::vector<cudaEvent_t> ev;
  cudaEvent_t e_start = nullptr, e_h2d0 = nullptr, e_h2d1 = nullptr, e_c0 = nullptr, e_end = nullptr,
              e_tok = nullptr;
  cudaEvent_t e_fork = nullptr, e_join = nullptr;  // copy stream fork / join (graph edges)
  // The whole invocation (copy stream + compute stream, event waits as edges)
  // captured once per key and replayed (world == 1, no profiling / fault
  // injection); TIDAL_GRAPH=0 disables it.
  struct PrefillGraph {
    cudaGraphExec_t exec = nullptr;
    std::vector<uint64_t> key;
    int launches = 0;
  } graph;
  bool use_graphs = true;
  // TIDAL_DEBUG_TIMELINE: timing events per group end / op start, and the last result
  std::vector<cudaEvent_t> tl_group, tl_op;
  std::vector<double> tl_group_ms, tl_op_ms;
  double tl_end_ms = 0;
  uint8_t* arena = nullptr;  // adapter arena
  uint64_t arena_cap = 0;
  int debug = 0, debug_arg = -1;
  int load_order = 0;         // TIDAL_ORDER_*
  bool suffix_valid = false;  // the streaming arena holds the streamed weights
  void* scrub = nullptr;
  unsigned long long* d_sum = nullptr;
  tidal_comm* comm = nullptr;
  std::deque<std::string> names;

  void ensure_events(size_t n) {
    while (ev.size() < n) {
      cudaEvent_t e;
      cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
      ev.push_back(e);
    }
  }
};

struct tidal_adapter {
  tidal_template* tpl = nullptr;
  std::shared_ptr<AdapterPlan> ap;
  int rank = 0;
  float scale = 1.f;
  uint32_t mask = 0;
  const uint8_t* host = nullptr;
  uint64_t bytes = 0;
  uint64_t serial = 0;  // process-unique identity (decode must continue with the same adapter)
};
static std::atomic<uint64_t> g_adapter_serial{0};

static ModelShape shape_of(const tidal_model_config* c) {
  ModelShape m;
  m.n_layers = c->n_layers;
  m.d_model = c->d_model;
  m.n_heads = c->n_heads;
  m.n_kv_heads = c->n_kv_heads;
  m.d_ff = c->d_ff;
  m.vocab = c->vocab;
  m.tie = c->tie_embeddings != 0;
  return m;
}

static std::string dump_copy(const std::string& s, char* buf, size_t cap, size_t* needed) {
  if (needed) *needed = s.size() + 1;
  if (buf && cap >= s.size() + 1) memcpy(buf, s.c_str(), s.size() + 1);
  else if (buf && cap) fail(TIDAL_ERR_BUFSZ, "buffer too small");
  return s;
}

extern "C" {

const char* tidal_last_error(void) { return g_err.c_str(); }
const char* tidal_version(void) { return "tidal-b200 0.1 (sm_100a)"; }

tidal_status tidal_model_create(const tidal_model_config* cfg, const tidal_host_tensor* w, int n,
                                const char* checkpoint, tidal_fill_fn fill, void* fill_ctx,
                                int world, int rank, tidal_model** out) {
  TIDAL_TRY
  require(cfg && w && out && n > 0, "null argument");
  require(world >= 1 && rank >= 0 && rank < world, "bad world/rank");
  ModelShape m = shape_of(cfg);
  require(m.n_layers >= 0 && m.d_model > 0 && m.n_heads > 0 && m.n_kv_heads > 0 && m.d_ff > 0 &&
              m.vocab > 0,
          "bad model config");
  require(m.d_model % m.n_heads == 0 && m.n_heads % m.n_kv_heads == 0, "bad head config");
  const int hd = m.head_dim();
  require(hd == 64 || hd == 128, "head_dim must be 64 or 128");
  require(m.d_model % 64 == 0 && m.d_ff % 8 == 0, "d_model % 64, d_ff % 8 required");
  require(m.d_model <= 8192, "d_model <= 8192 (RMSNorm keeps a row in registers)");
  require(m.n_kv_heads % world == 0 && m.d_ff % world == 0 && m.vocab % world == 0,
          "model does not shard evenly over world");
  require((m.d_ff / world) % 8 == 0, "d_ff/world must be a multiple of 8");
  auto* mo = new tidal_model();
  mo->shape = m;
  mo->theta = cfg->rope_theta;
  mo->eps = cfg->rms_eps;
  mo->checkpoint = checkpoint ? checkpoint : "base";
  mo->world = world;
  mo->rank = rank;
  mo->fill = fill;
  mo->ctx = fill_ctx;
  build_base(mo->tt, m, world, rank, mo->checkpoint);
  mo->host.assign(mo->tt.n_base, nullptr);
  mo->user_index.assign(mo->tt.n_base, -1);
  for (int i = 0; i < n; ++i) {
    require(w[i].name != nullptr, "tensor without a name");
    const int id = mo->tt.find(w[i].name);
    if (id < 0 || id >= mo->tt.n_base) {
      delete mo;
      fail(TIDAL_ERR_STRUCTURE, std::string("unexpected tensor ") + w[i].name);
    }
    if (mo->user_index[id] >= 0 || w[i].bytes != mo->tt.t[id].bytes) {
      const std::string nm = w[i].name;
      delete mo;
      fail(TIDAL_ERR_STRUCTURE, "duplicate or mis-sized tensor " + nm);
    }
    mo->user_index[id] = i;
    mo->host[id] = w[i].host_bf16;
    if (!w[i].host_bf16 && !fill) {
      delete mo;
      fail(TIDAL_ERR_INVALID, "tensor without data and no fill callback");
    }
  }
  for (int id = 0; id < mo->tt.n_base; ++id)
    if (mo->user_index[id] < 0) {
      const std::string nm = mo->tt.t[id].name;
      delete mo;
      fail(TIDAL_ERR_STRUCTURE, "missing tensor " + nm);
    }
  *out = mo;
  TIDAL_CATCH
}

void tidal_model_destroy(tidal_model* m) { delete m; }

tidal_status tidal_trace(tidal_model* m, const int32_t* host_tokens, int n_tokens, int device,
                         float* host_logits_out, int32_t* host_token_out, double* cold_ttft_ms_out,
                         tidal_trace_rec** out) {
  TIDAL_TRY
  require(m && out, "null argument");
  auto* tr = new tidal_trace_rec();
  tr->tt = m->tt;
  tr->tr = make_trace(m->tt);
  if (device < 0) {
    *out = tr;
    return TIDAL_OK;
  }
  require(host_tokens && n_tokens >= 1, "tokens required for a traced first run");
  for (int i = 0; i < n_tokens; ++i)
    require(host_tokens[i] >= 0 && host_tokens[i] < m->shape.vocab, "token out of range");
  // First run: every weight copied in registration order, then the forward
  // with a Recorder capturing which weights each launched op reads.
  const auto t0 = std::chrono::steady_clock::now();
  Exec ex;
  uint8_t* dbuf = nullptr;
  uint8_t* stage = nullptr;
  try {
    ex.init(device, m->shape, m->eps, m->theta, m->world, m->rank, n_tokens);
    std::vector<uint64_t> off(m->tt.n_base);
    uint64_t cur = 0, maxb = 0;
    for (int id = 0; id < m->tt.n_base; ++id) {
      cur = (cur + kAlign - 1) / kAlign * kAlign;
      off[id] = cur;
      cur += m->tt.t[id].bytes;
      maxb = std::max(maxb, m->tt.t[id].bytes);
    }
    cuda_check(cudaMalloc(&dbuf, cur), "cudaMalloc(trace weights)");
    cuda_check(cudaHostAlloc(&stage, maxb, cudaHostAllocDefault), "cudaHostAlloc(stage)");
    ex.wptr.assign(m->tt.t.size(), nullptr);
    for (int id = 0; id < m->tt.n_base; ++id) {
      m->produce(id, stage);
      cuda_check(cudaMemcpy(dbuf + off[id], stage, m->tt.t[id].bytes, cudaMemcpyHostToDevice),
                 "H2D (first run)");
      ex.wptr[id] = dbuf + off[id];
    }
    memcpy(ex.h_tok, host_tokens, sizeof(int32_t) * n_tokens);
    cuda_check(cudaMemcpyAsync(ex.tok, ex.h_tok, 4 * n_tokens, cudaMemcpyHostToDevice, ex.compute),
               "H2D tokens");
    Recorder rec;
    rec.seen.assign(m->tt.t.size(), 0);
    RunArgs a;
    a.tt = &m->tt;
    a.ops = &tr->tr.ops;
    a.S = n_tokens;
    a.rec = &rec;
    a.akey = nullptr;
    run_forward(ex, a);
    cuda_check(cudaMemcpyAsync(ex.h_key, ex.key, 8, cudaMemcpyDeviceToHost, ex.compute), "D2H");
    if (host_logits_out)
      cuda_check(cudaMemcpyAsync(ex.h_logits, ex.logits, 4ull * m->shape.vocab,
                                 cudaMemcpyDeviceToHost, ex.compute),
                 "D2H");
    cuda_check(cudaStreamSynchronize(ex.compute), "first run");
    const auto t1 = std::chrono::steady_clock::now();
    if (cold_ttft_ms_out) *cold_ttft_ms_out = std::chrono::duration<double, std::milli>(t1 - t0).count();
    if (host_logits_out) memcpy(host_logits_out, ex.h_logits, 4ull * m->shape.vocab);
    if (host_token_out) *host_token_out = (int32_t)(0xFFFFFFFFu - (uint32_t)(*ex.h_key & 0xFFFFFFFFu));
    // The ids the launcher handed to its kernels must reproduce the planner's
    // trace (never-read weights at the tail): the same first-use order, and no
    // weight used at an op before the one whose barrier covers it (a fused
    // kernel may use a weight later — final_norm's gain in the head kernel).
    std::vector<char> seen(m->tt.n_base, 0);
    for (auto& p : rec.access) seen[p.first] = 1;
    for (int id = 0; id < m->tt.n_base; ++id)
      if (!seen[id]) rec.access.emplace_back(id, -1);
    bool same = rec.access.size() == tr->tr.access.size();
    for (size_t i = 0; same && i < rec.access.size(); ++i)
      same = rec.access[i].first == tr->tr.access[i].first &&
             rec.access[i].second >= tr->tr.access[i].second;
    if (!same) fail(TIDAL_ERR_INVALID, "kernel weight use order != planner trace order");
  } catch (...) {
    if (dbuf) cudaFree(dbuf);
    if (stage) cudaFreeHost(stage);
    ex.destroy();
    delete tr;
    throw;
  }
  cudaFree(dbuf);
  cudaFreeHost(stage);
  ex.destroy();
  *out = tr;
  TIDAL_CATCH
}

void tidal_trace_destroy(tidal_trace_rec* t) { delete t; }

tidal_status tidal_trace_dump(const tidal_trace_rec* t, char* buf, size_t cap, size_t* needed) {
  TIDAL_TRY
  require(t != nullptr, "null trace");
  dump_copy(trace_dump(t->tt, t->tr), buf, cap, needed);
  TIDAL_CATCH
}

static TemplateChoice choice_of(const tidal_template_opts* o) {
  TemplateChoice c;
  c.resident_bytes = o->resident_bytes;
  c.eq1 = o->eq1 != 0;
  c.t_ttft_s = o->t_ttft_s;
  c.b_pcie_Bps = o->b_pcie_Bps;
  c.group_policy = o->group_policy;
  c.max_transfers = o->max_transfers > 0 ? o->max_transfers : 300;
  return c;
}

static void warm_kernels(tidal_template* tp) {
  // A8 proactive code loading: one warm run of every kernel on dummy inputs
  // (reduced dimensions), so no invocation pays a lazy module load.
  Exec& ex = tp->ex;
  const int S = std::min(tp->max_tokens, 16);
  std::vector<int32_t> tok(S, 0);
  memcpy(ex.h_tok, tok.data(), 4 * S);
  cuda_check(cudaMemcpyAsync(ex.tok, ex.h_tok, 4 * S, cudaMemcpyHostToDevice, ex.compute), "H2D");
  ex.wptr.assign(tp->tt.t.size(), nullptr);
  for (int id = 0; id < tp->tt.n_base; ++id) ex.wptr[id] = tp->dev + tp->plan.offset[id];
  RunArgs a;
  a.tt = &tp->tt;
  a.ops = &tp->plan.ops;
  a.S = S;
  a.akey = nullptr;
  a.gen = tp->gen;
  a.comm = tp->comm ? tp->comm->impl : nullptr;
  run_forward(ex, a);
  shrink_preload();
  cuda_check(cudaStreamSynchronize(ex.compute), "warm run");
  ex.cache.clear();
}

// Identity of the bytes below `shared` in a template's layout: every tensor
// overlapping that prefix with its offset, size and provenance (checkpoint +
// name + shape), so an importer with another trace / layout / checkpoint /
// weights of the same byte size is refused.
static uint64_t prefix_fingerprint(const TensorTable& tt, const Plan& p, uint64_t shared) {
  std::string s;
  for (int id : p.layout) {
    const uint64_t o = p.offset[id];
    if (o >= shared) continue;
    s += tt.t[id].name + "@" + std::to_string(o) + ":" + std::to_string(tt.t[id].bytes) + ":" +
         tt.t[id].provenance + ";";
  }
  s += std::to_string(shared);
  return fnv1a64(s);
}

static tidal_status template_create(tidal_model* m, const tidal_trace_rec* t,
                                    const tidal_template_opts* opts, const int* fds, int n_fds,
                                    uint64_t shared_bytes, uint64_t fingerprint,
                                    tidal_template** out) {
  TIDAL_TRY
  require(m && t && opts && out, "null argument");
  require(t->tt.n_base == m->tt.n_base, "trace is from a different model", TIDAL_ERR_STRUCTURE);
  auto* tp = new tidal_template();
  tp->shape = m->shape;
  tp->theta = m->theta;
  tp->eps = m->eps;
  tp->world = m->world;
  tp->rank = m->rank;
  tp->tt = m->tt;
  tp->tr = t->tr;
  tp->choice = choice_of(opts);
  tp->plan = make_plan(tp->tt, tp->tr, tp->choice);
  tp->device = opts->device;
  tp->dry = opts->device < 0;
  tp->max_tokens = opts->max_tokens > 0 ? opts->max_tokens : 2048;
  tp->comm = opts->comm;
  if (tp->dry) {
    *out = tp;
    return TIDAL_OK;
  }
  try {
    require(m->world == 1 || (opts->comm && opts->comm->world == m->world && opts->comm->rank == m->rank),
            "tensor-parallel model needs a matching communicator");
    if (n_fds)
      require(prefix_fingerprint(tp->tt, tp->plan, shared_bytes) == fingerprint,
              "imported template chunks hold another layout / checkpoint (fingerprint mismatch)",
              TIDAL_ERR_STRUCTURE);
    tp->ex.init(tp->device, tp->shape, tp->eps, tp->theta, tp->world, tp->rank, tp->max_tokens);
    tp->ex.colocated = tp->comm && tp->comm->impl && tp->comm->impl->colocated;
    const uint64_t L = tp->plan.layout_bytes;
    {
      // pinned pool, NUMA-local to the device, whole image in layout order
      NumaGuard numa(tp->device);
      cuda_check(cudaHostAlloc((void**)&tp->pool, L, cudaHostAllocDefault), "cudaHostAlloc(pool)");
      uint64_t prev_end = 0;
      for (int id : tp->plan.layout) {
        const uint64_t o = tp->plan.offset[id];
        if (o > prev_end) memset(tp->pool + prev_end, 0, o - prev_end);
        m->produce(id, tp->pool + o);
        prev_end = o + tp->tt.t[id].bytes;
      }
    }
    if (vmm_available() && !device_allocator_set()) {
      vmm_alloc(tp->vmm, L, tp->device, fds, n_fds);
      tp->dev = reinterpret_cast<uint8_t*>(tp->vmm.va);
      if (n_fds)
        require((uint64_t)n_fds * tp->vmm.chunk == shared_bytes &&
                    shared_bytes <= tp->plan.resident_end,
                "imported chunks do not match this template's layout / resident prefix",
                TIDAL_ERR_STRUCTURE);
    } else {
      require(n_fds == 0, "template memory not on CUDA VMM (unavailable, or a caller allocator "
                          "is set): cannot import");
      tp->dev = reinterpret_cast<uint8_t*>(dev_alloc(L, tp->device, "template + streaming arena"));
    }
    tp->shared_bytes = shared_bytes;
    // the shared prefix is already on the device (the exporter's bytes)
    if (tp->plan.resident_end > shared_bytes)
      cuda_check(cudaMemcpy(tp->dev + shared_bytes, tp->pool + shared_bytes,
                            tp->plan.resident_end - shared_bytes, cudaMemcpyHostToDevice),
                 "H2D resident prefix");
    for (cudaEvent_t* e : {&tp->e_start, &tp->e_h2d0, &tp->e_h2d1, &tp->e_c0, &tp->e_end, &tp->e_tok})
      cuda_check(cudaEventCreate(e), "cudaEventCreate");
    for (cudaEvent_t* e : {&tp->e_fork, &tp->e_join})
      cuda_check(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "cudaEventCreate");
    {
      const char* g = getenv("TIDAL_GRAPH");
      tp->use_graphs = !(g && g[0] == '0');
    }
    tp->ensure_events(tp->plan.groups.size() + 2 * tp->shape.n_layers + 4);
    tp->d_sum = reinterpret_cast<unsigned long long*>(dev_alloc(64, tp->device, "checksum"));
    // warm run streams nothing: make every weight valid once (prefix resident,
    // suffix copied) so the warm launches read real bytes
    if (tp->plan.resident_end < L)
      cuda_check(cudaMemcpy(tp->dev + tp->plan.resident_end, tp->pool + tp->plan.resident_end,
                            L - tp->plan.resident_end, cudaMemcpyHostToDevice),
                 "H2D warm");
    warm_kernels(tp);
    tp->suffix_valid = true;  // the warm-up copied the whole layout
  } catch (...) {
    tidal_template_destroy(tp);
    throw;
  }
  *out = tp;
  TIDAL_CATCH
}

tidal_status tidal_template_create(tidal_model* m, const tidal_trace_rec* t,
                                   const tidal_template_opts* opts, tidal_template** out) {
  return template_create(m, t, opts, nullptr, 0, 0, 0, out);
}

tidal_status tidal_template_import(tidal_model* m, const tidal_trace_rec* t,
                                   const tidal_template_opts* opts, const int* fds, int n_fds,
                                   uint64_t shared_bytes, uint64_t fingerprint,
                                   tidal_template** out) {
  if (!opts || opts->device < 0) return set_err(TIDAL_ERR_INVALID, "import needs a device template");
  if (n_fds < 1 || !fds) return set_err(TIDAL_ERR_INVALID, "no chunks to import");
  if (opts->comm) return set_err(TIDAL_ERR_INVALID, "tensor-parallel import is not implemented");
  return template_create(m, t, opts, fds, n_fds, shared_bytes, fingerprint, out);
}

tidal_status tidal_template_export(tidal_template* tp, int* fds, int cap, int* n_fds,
                                   uint64_t* shared_bytes, uint64_t* fingerprint) {
  TIDAL_TRY
  require(tp && n_fds && shared_bytes, "null argument");
  require(!tp->dry && tp->vmm.va, "export needs a device template on CUDA VMM");
  require(tp->shared_bytes == 0, "an imported template cannot be re-exported");
  const size_t n = tp->plan.resident_end / tp->vmm.chunk;  // chunks wholly inside the prefix
  *n_fds = (int)n;
  *shared_bytes = (uint64_t)n * tp->vmm.chunk;
  if (fingerprint) *fingerprint = prefix_fingerprint(tp->tt, tp->plan, *shared_bytes);
  if (!fds) return TIDAL_OK;  // size query
  require(cap >= (int)n, "fd buffer too small", TIDAL_ERR_BUFSZ);
  for (size_t i = 0; i < n; ++i) fds[i] = vmm_export_fd(tp->vmm, i);
  tp->exported_bytes = std::max<uint64_t>(tp->exported_bytes, *shared_bytes);
  TIDAL_CATCH
}

tidal_status tidal_template_resize(tidal_template* tp, const tidal_template_opts* opts) {
  TIDAL_TRY
  require(tp && opts, "null argument");
  TemplateChoice c = tp->choice;
  c.resident_bytes = opts->resident_bytes;
  c.eq1 = opts->eq1 != 0;
  c.t_ttft_s = opts->t_ttft_s;
  c.b_pcie_Bps = opts->b_pcie_Bps;
  const uint64_t old_end = tp->plan.resident_end;
  Plan p = make_plan(tp->tt, tp->tr, c);
  // exported / imported prefix bytes are a shared template: they must stay resident
  require(p.resident_end >= std::max(tp->exported_bytes, tp->shared_bytes),
          "resize would stream into a prefix shared with other processes");
  if (!tp->dry) {
    cuda_check(cudaSetDevice(tp->device), "cudaSetDevice");
    cuda_check(cudaDeviceSynchronize(), "sync");
    if (p.resident_end > old_end)
      cuda_check(cudaMemcpy(tp->dev + old_end, tp->pool + old_end, p.resident_end - old_end,
                            cudaMemcpyHostToDevice),
                 "H2D grow template");
    tp->ensure_events(p.groups.size() + 2 * tp->shape.n_layers + 4);
  }
  tp->choice = c;
  tp->plan = std::move(p);
  ++tp->gen;
  TIDAL_CATCH
}

tidal_status tidal_template_keep_alive(tidal_template* tp) {
  TIDAL_TRY
  require(tp != nullptr && !tp->dry, "keep-alive needs a device template");
  require(tp->suffix_valid, "streaming arena does not hold valid weights");
  TemplateChoice c = tp->choice;
  c.eq1 = false;
  c.resident_bytes = UINT64_MAX;
  tp->plan = make_plan(tp->tt, tp->tr, c);  // every base weight resident; no copy needed
  tp->choice = c;
  ++tp->gen;
  TIDAL_CATCH
}

tidal_status tidal_set_load_order(tidal_template* tp, int order) {
  TIDAL_TRY
  require(tp != nullptr && order >= 0 && order <= 2, "bad load order");
  tp->load_order = order;
  TIDAL_CATCH
}

void tidal_template_destroy(tidal_template* tp) {
  if (!tp) return;
  if (!tp->dry && tp->device >= 0) {
    cudaSetDevice(tp->device);
    cudaDeviceSynchronize();
    for (cudaEvent_t e : tp->ev) cudaEventDestroy(e);
    for (cudaEvent_t e : {tp->e_start, tp->e_h2d0, tp->e_h2d1, tp->e_c0, tp->e_end, tp->e_tok,
                          tp->e_fork, tp->e_join})
      if (e) cudaEventDestroy(e);
    if (tp->graph.exec) cudaGraphExecDestroy(tp->graph.exec);
    for (cudaEvent_t e : tp->tl_group) cudaEventDestroy(e);
    for (cudaEvent_t e : tp->tl_op) cudaEventDestroy(e);
    if (tp->vmm.va)
      vmm_free(tp->vmm);
    else
      dev_free(tp->dev);
    dev_free(tp->arena);
    dev_free(tp->scrub);
    dev_free(tp->d_sum);
    if (tp->pool) cudaFreeHost(tp->pool);
    tp->ex.destroy();
  }
  delete tp;
}

static void adapter_table(const tidal_template* tp, int rank, uint32_t mask, TensorTable& tt,
                          const std::string& ckpt) {
  require(rank == 8 || rank == 16 || rank == 32 || rank == 64, "LoRA rank must be 8, 16, 32 or 64");
  require(mask != 0 && (mask & ~0x7Fu) == 0, "target_mask must be a non-empty subset of 0x7F");
  tt = tp->tt;
  add_adapter(tt, rank, mask, ckpt);
}

tidal_status tidal_adapter_layout(const tidal_template* tp, int rank, uint32_t mask,
                                  tidal_slot* slots, int cap, int* n, uint64_t* total) {
  TIDAL_TRY
  require(tp != nullptr, "null template");
  TensorTable tt;
  adapter_table(tp, rank, mask, tt, "adapter");
  std::vector<int> ids;
  std::vector<uint64_t> offs;
  uint64_t tot = 0;
  adapter_layout(tt, ids, offs, tot);
  if (n) *n = (int)ids.size();
  if (total) *total = tot;
  auto* mtp = const_cast<tidal_template*>(tp);
  for (int i = 0; i < (int)ids.size() && i < cap && slots; ++i) {
    mtp->names.push_back(tt.t[ids[i]].name);
    slots[i].name = mtp->names.back().c_str();
    slots[i].offset = offs[i];
    slots[i].bytes = tt.t[ids[i]].bytes;
    slots[i].rows = tt.t[ids[i]].rows;
    slots[i].cols = tt.t[ids[i]].cols;
  }
  TIDAL_CATCH
}

static std::shared_ptr<AdapterPlan> get_adapter_plan(tidal_template* tp, int rank, uint32_t mask) {
  auto& slot = tp->aplans[{rank, mask}];
  if (!slot || slot->gen != tp->gen) {
    auto ap = std::make_shared<AdapterPlan>();
    adapter_table(tp, rank, mask, ap->tt, "adapter");
    ap->plan = make_plan(ap->tt, tp->tr, tp->choice);
    ap->gen = tp->gen;
    slot = ap;
  }
  return slot;
}

tidal_status tidal_attach_lora(tidal_template* tp, const tidal_lora_desc* d, tidal_adapter** out) {
  TIDAL_TRY
  require(tp && d && out, "null argument");
  auto* a = new tidal_adapter();
  try {
    a->ap = get_adapter_plan(tp, d->rank, d->target_mask);
    require(d->bytes == a->ap->plan.adapter_bytes,
            "adapter buffer is " + std::to_string(d->bytes) + " B, layout needs " +
                std::to_string(a->ap->plan.adapter_bytes),
            TIDAL_ERR_STRUCTURE);
    require(d->host_pinned != nullptr || tp->dry, "adapter needs a pinned host buffer");
  } catch (...) {
    delete a;
    throw;
  }
  a->tpl = tp;
  a->rank = d->rank;
  a->scale = d->scale;
  a->mask = d->target_mask;
  a->host = reinterpret_cast<const uint8_t*>(d->host_pinned);
  a->bytes = d->bytes;
  a->serial = ++g_adapter_serial;
  *out = a;
  TIDAL_CATCH
}

void tidal_adapter_destroy(tidal_adapter* a) { delete a; }

tidal_status tidal_plan_dump(const tidal_template* tp, const tidal_adapter* a, char* buf, size_t cap,
                             size_t* needed) {
  TIDAL_TRY
  require(tp != nullptr, "null template");
  if (a) {
    require(a->tpl == tp, "adapter attached to another template");
    auto* ma = const_cast<tidal_adapter*>(a);
    if (ma->ap->gen != tp->gen)
      ma->ap = get_adapter_plan(const_cast<tidal_template*>(tp), ma->rank, ma->mask);
    dump_copy(plan_dump(ma->ap->tt, ma->ap->plan), buf, cap, needed);
  } else {
    dump_copy(plan_dump(tp->tt, tp->plan), buf, cap, needed);
  }
  TIDAL_CATCH
}

tidal_status tidal_invoke_prefill(tidal_template* tp, const tidal_adapter* ca,
                                  const int32_t* host_tokens, int n_tokens, float* host_logits_out,
                                  int32_t* host_token_out, tidal_stats* stats) {
  return tidal_invoke_prefill_batch(tp, ca, host_tokens, 1, n_tokens, host_logits_out,
                                    host_token_out, stats);
}

tidal_status tidal_invoke_prefill_batch(tidal_template* tp, const tidal_adapter* ca,
                                        const int32_t* host_tokens, int n_seqs, int seq_len,
                                        float* host_logits_out, int32_t* host_tokens_out,
                                        tidal_stats* stats) {
  TIDAL_TRY
  const auto t_entry = std::chrono::steady_clock::now();
  require(tp && host_tokens && host_tokens_out, "null argument");
  require(!tp->dry, "dry template cannot be invoked");
  require(n_seqs >= 1 && n_seqs <= kMaxBatch, "n_seqs out of range (1..64)");
  require(seq_len >= 1 && (int64_t)n_seqs * seq_len <= tp->max_tokens,
          "n_seqs * seq_len exceeds the template's max_tokens");
  const int n_tokens = n_seqs * seq_len;
  const int V = tp->shape.vocab;
  for (int i = 0; i < n_tokens; ++i)
    require(host_tokens[i] >= 0 && host_tokens[i] < V, "token out of range");
  auto* a = const_cast<tidal_adapter*>(ca);
  if (a) {
    require(a->tpl == tp, "adapter attached to another template");
    if (a->ap->gen != tp->gen) a->ap = get_adapter_plan(tp, a->rank, a->mask);
  }
  const std::shared_ptr<AdapterPlan> hold = a ? a->ap : nullptr;
  const Plan& P = a ? hold->plan : tp->plan;
  const TensorTable& tt = a ? hold->tt : tp->tt;
  Exec& ex = tp->ex;
  cuda_check(cudaSetDevice(tp->device), "cudaSetDevice");
  if (a && P.adapter_bytes > tp->arena_cap) {
    if (tp->arena) {
      cuda_check(cudaStreamSynchronize(ex.compute), "sync");
      dev_free(tp->arena);
    }
    tp->arena = nullptr;
    tp->arena = reinterpret_cast<uint8_t*>(dev_alloc(P.adapter_bytes, tp->device, "adapter arena"));
    tp->arena_cap = P.adapter_bytes;
  }
  tp->ensure_events(P.groups.size());
  // adaptive fork: pointer table (resident -> template, streamed -> arena
  // suffix of the same layout buffer, adapter -> adapter arena)
  ex.wptr.assign(tt.t.size(), nullptr);
  for (int id = 0; id < tt.n_base; ++id) ex.wptr[id] = tp->dev + P.offset[id];
  for (int id : P.adapter_layout) ex.wptr[id] = tp->arena + P.offset[id];
  // debug preparation (outside the measured window)
  if (tp->debug & TIDAL_DEBUG_POISON) {
    cuda_check(poison_launch(tp->dev + P.resident_end, P.layout_bytes - P.resident_end, ex.compute),
               "poison");
    if (a) cuda_check(poison_launch(tp->arena, P.adapter_bytes, ex.compute), "poison");
  }
  if (tp->debug & TIDAL_DEBUG_SCRUB_L2) {
    if (!tp->scrub) tp->scrub = dev_alloc(512ull << 20, tp->device, "L2 scrub buffer");
    cuda_check(scrub_launch(tp->scrub, 512ull << 20, ex.compute), "scrub");
  }
  if (tp->debug & (TIDAL_DEBUG_POISON | TIDAL_DEBUG_SCRUB_L2))
    cuda_check(cudaStreamSynchronize(ex.compute), "debug prep");
  const auto t0 = (tp->debug & (TIDAL_DEBUG_POISON | TIDAL_DEBUG_SCRUB_L2))
                      ? std::chrono::steady_clock::now()
                      : t_entry;
  tp->suffix_valid = false;  // set again once every streamed group has landed
  ex.launches = 0;
  ex.profile = (tp->debug & (TIDAL_DEBUG_PROFILE | TIDAL_DEBUG_PROFILE_GEMM)) != 0;
  ex.profile_all = (tp->debug & TIDAL_DEBUG_PROFILE) != 0;
  ex.prof_pending.clear();
  memcpy(ex.h_tok, host_tokens, 4ull * n_tokens);
  const int skip = (tp->debug & TIDAL_DEBUG_SKIP_BARRIER) ? tp->debug_arg : -1;
  const bool graph_ok = tp->use_graphs && tp->world == 1 &&
                        !(tp->debug & (TIDAL_DEBUG_PROFILE | TIDAL_DEBUG_PROFILE_GEMM |
                                       TIDAL_DEBUG_SKIP_BARRIER | TIDAL_DEBUG_SERIAL |
                                       TIDAL_DEBUG_NO_GRAPH | TIDAL_DEBUG_TIMELINE));
  const bool timeline = (tp->debug & TIDAL_DEBUG_TIMELINE) != 0;
  if (timeline) {
    auto grow = [](std::vector<cudaEvent_t>& v, size_t n) {
      while (v.size() < n) {
        cudaEvent_t e;
        cuda_check(cudaEventCreate(&e), "cudaEventCreate(timeline)");
        v.push_back(e);
      }
    };
    grow(tp->tl_group, P.groups.size());
    grow(tp->tl_op, P.ops.size());
  }
  // everything a captured invocation bakes in: plan, shapes, buffers, scale
  float scale_v = a ? a->scale : 1.f;
  uint32_t scale_bits = 0;
  memcpy(&scale_bits, &scale_v, 4);
  const std::vector<uint64_t> gkey = {
      (uint64_t)(uintptr_t)&P, tp->gen, (uint64_t)n_tokens, (uint64_t)n_seqs,
      (uint64_t)(uintptr_t)(a ? a->host : nullptr), (uint64_t)(uintptr_t)tp->arena, scale_bits,
      (uint64_t)tp->load_order, (uint64_t)(host_logits_out != nullptr),
      (uint64_t)(uintptr_t)ex.dec.kc, (uint64_t)ex.fuse_shrink, (uint64_t)ex.ar_bf16};
  const unsigned rec_flags = graph_ok ? cudaEventRecordExternal : cudaEventRecordDefault;
  auto rec = [&](cudaEvent_t e, cudaStream_t st) {  // timing events: real records in a graph
    cuda_check(cudaEventRecordWithFlags(e, st, rec_flags), "event");
  };
  auto enqueue = [&]() {
    rec(tp->e_start, ex.compute);
    cuda_check(cudaEventRecord(tp->e_fork, ex.compute), "event");
    cuda_check(cudaStreamWaitEvent(ex.copy, tp->e_fork, 0), "wait");
    // the prompt goes first on the (high-priority) copy stream: a token copy on
    // the compute stream larger than ~24 KB was starved behind every weight
    // group (measured: at S >= 7168 the prefill started after the last group)
    cuda_check(cudaMemcpyAsync(ex.tok, ex.h_tok, 4ull * n_tokens, cudaMemcpyHostToDevice, ex.copy),
               "H2D tokens");
    cuda_check(cudaEventRecord(tp->e_tok, ex.copy), "event");
    // ---- copy stream: groups in traced access order, one event each ----
    rec(tp->e_h2d0, ex.copy);
    // copy order (traced by default; ablations reverse / registration order)
    std::vector<int> order(P.groups.size());
    for (size_t g = 0; g < order.size(); ++g) order[g] = (int)g;
    if (tp->load_order == TIDAL_ORDER_REVERSE) {
      std::reverse(order.begin(), order.end());
    } else if (tp->load_order == TIDAL_ORDER_REGISTRATION) {
      auto first_id = [&](int g) {
        int m = INT32_MAX;
        for (int id : P.groups[g].members) m = std::min(m, id);
        return m;
      };
      std::stable_sort(order.begin(), order.end(),
                       [&](int x, int y) { return first_id(x) < first_id(y); });
    }
    std::vector<int> copy_pos(P.groups.size());
    for (size_t i = 0; i < order.size(); ++i) copy_pos[order[i]] = (int)i;
    for (int g : order) {
      const Group& G = P.groups[g];
      const uint8_t* src = G.adapter ? a->host + G.offset : tp->pool + G.offset;
      uint8_t* dst = G.adapter ? tp->arena + G.offset : tp->dev + G.offset;
      if (g == skip) {
        sleep_kernel<<<1, 1, 0, ex.copy>>>(20000);  // fault injection: late group
        cuda_check(cudaGetLastError(), "sleep");
      }
      cuda_check(cudaMemcpyAsync(dst, src, G.bytes, cudaMemcpyHostToDevice, ex.copy), "H2D group");
      cuda_check(cudaEventRecord(tp->ev[g], ex.copy), "event");
      if (timeline) cuda_check(cudaEventRecord(tp->tl_group[g], ex.copy), "event");
    }
    rec(tp->e_h2d1, ex.copy);
    cuda_check(cudaEventRecord(tp->e_join, ex.copy), "event");
    // ---- compute stream ----
    cuda_check(cudaStreamWaitEvent(ex.compute, tp->e_tok, 0), "wait tokens");
    if (tp->debug & 8) cuda_check(cudaStreamWaitEvent(ex.compute, tp->e_join, 0), "serial");
    rec(tp->e_c0, ex.compute);
    RunArgs ra;
    ra.tt = &tt;
    ra.ops = &P.ops;
    ra.barriers = &P.barriers;
    ra.events = &tp->ev;
    ra.copy_pos = &copy_pos;
    ra.group_of = &P.group_of;
    ra.tl_op = timeline ? &tp->tl_op : nullptr;
    ra.skip_group = skip;
    ra.S = n_tokens;
    ra.nseq = n_seqs;
    ra.lora_scale = a ? a->scale : 1.f;
    ra.akey = a ? (const void*)tp->arena : nullptr;
    ra.gen = tp->gen;
    ra.comm = tp->comm ? tp->comm->impl : nullptr;
    run_forward(ex, ra);
    cuda_check(cudaStreamWaitEvent(ex.compute, tp->e_join, 0), "wait copies");
    cuda_check(cudaMemcpyAsync(ex.h_key, ex.key, 8ull * n_seqs, cudaMemcpyDeviceToHost, ex.compute),
               "D2H key");
    if (host_logits_out)
      cuda_check(cudaMemcpyAsync(ex.h_logits, ex.logits, 4ull * V * n_seqs, cudaMemcpyDeviceToHost,
                                 ex.compute),
                 "D2H logits");
    rec(tp->e_end, ex.compute);
  };
  if (graph_ok && tp->graph.exec && tp->graph.key == gkey) {
    cuda_check(cudaGraphLaunch(tp->graph.exec, ex.compute), "graph launch");
    ex.launches = tp->graph.launches;
  } else if (graph_ok) {
    if (tp->graph.exec) cudaGraphExecDestroy(tp->graph.exec);
    for (cudaEvent_t e : tp->tl_group) cudaEventDestroy(e);
    for (cudaEvent_t e : tp->tl_op) cudaEventDestroy(e);
    tp->graph.exec = nullptr;
    cudaGraph_t graph = nullptr;
    cuda_check(cudaStreamBeginCapture(ex.compute, cudaStreamCaptureModeThreadLocal), "begin capture");
    try {
      enqueue();
    } catch (...) {
      cudaStreamEndCapture(ex.compute, &graph);
      if (graph) cudaGraphDestroy(graph);
      throw;
    }
    cuda_check(cudaStreamEndCapture(ex.compute, &graph), "end capture");
    const cudaError_t ie = cudaGraphInstantiate(&tp->graph.exec, graph, 0);
    cudaGraphDestroy(graph);
    cuda_check(ie, "graph instantiate");
    tp->graph.key = gkey;
    tp->graph.launches = ex.launches;
    cuda_check(cudaGraphLaunch(tp->graph.exec, ex.compute), "graph launch");
  } else {
    enqueue();
  }
  ex.dec.prompt_akey = a ? (const void*)tp->arena : nullptr;
  cuda_check(cudaEventSynchronize(tp->e_end), "invoke");
  ex.dbg_dump();
  if (timeline) {
    float ms = 0;
    tp->tl_group_ms.assign(P.groups.size(), 0.0);
    tp->tl_op_ms.assign(P.ops.size(), 0.0);
    for (size_t g = 0; g < P.groups.size(); ++g) {
      cuda_check(cudaEventElapsedTime(&ms, tp->e_start, tp->tl_group[g]), "elapsed");
      tp->tl_group_ms[g] = ms;
    }
    for (size_t k = 0; k < P.ops.size(); ++k) {
      cuda_check(cudaEventElapsedTime(&ms, tp->e_start, tp->tl_op[k]), "elapsed");
      tp->tl_op_ms[k] = ms;
    }
    cuda_check(cudaEventElapsedTime(&ms, tp->e_start, tp->e_end), "elapsed");
    tp->tl_end_ms = ms;
  }
  tp->suffix_valid = skip < 0;
  // decode continuation: the cache now holds this prompt's K/V (single prompt)
  ex.dec.prompt_len = (ex.dec.kc && n_seqs == 1) ? n_tokens : 0;
  ex.dec.prompt_adapter = a ? a->serial : 0;
  ex.dec.prompt_gen = tp->gen;
  if (ex.profile) ex.prof_collect();
  for (int b = 0; b < n_seqs; ++b)  // packed key: low word = ~token
    host_tokens_out[b] = (int32_t)(0xFFFFFFFFu - (uint32_t)(ex.h_key[b] & 0xFFFFFFFFu));
  if (host_logits_out) {
    // device layout [world][n_seqs][V / world] -> [n_seqs][V]
    const int W = tp->world, Vl = V / W;
    for (int k = 0; k < W; ++k)
      for (int b = 0; b < n_seqs; ++b)
        memcpy(host_logits_out + (size_t)b * V + (size_t)k * Vl,
               ex.h_logits + ((size_t)k * n_seqs + b) * Vl, 4ull * Vl);
  }
  const auto t1 = std::chrono::steady_clock::now();
  if (stats) {
    memset(stats, 0, sizeof *stats);
    stats->ttft_host_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
    float ms = 0;
    cudaEventElapsedTime(&ms, tp->e_start, tp->e_end);
    stats->device_ms = ms;
    cudaEventElapsedTime(&ms, tp->e_start, tp->e_h2d0);
    stats->h2d_first_ms = ms;
    cudaEventElapsedTime(&ms, tp->e_start, tp->e_h2d1);
    stats->h2d_last_ms = ms;
    cudaEventElapsedTime(&ms, tp->e_start, tp->e_c0);
    stats->compute_first_ms = ms;
    stats->compute_last_ms = stats->device_ms;
    stats->bytes_streamed = P.stream_bytes;
    stats->bytes_resident = P.resident_bytes;
    stats->bytes_adapter = P.adapter_payload;
    stats->n_copies = (int)P.groups.size();
    stats->n_kernels = ex.launches;
  }
  for (int i = 0; i < n_seqs; ++i) {
    const unsigned long long key = ex.h_key[i];
    const uint32_t hi = (uint32_t)(key >> 32);
    const uint32_t bits = (hi & 0x80000000u) ? (hi & 0x7FFFFFFFu) : ~hi;
    float best;
    memcpy(&best, &bits, 4);
    if (key == 0 || std::isnan(best)) fail(TIDAL_ERR_NUMERIC, "NaN in logits (argmax undefined)");
  }
  TIDAL_CATCH
}

tidal_status tidal_template_enable_decode(tidal_template* tp, int max_new_tokens) {
  TIDAL_TRY
  require(tp, "null template");
  require(!tp->dry, "dry template cannot decode");
  require(tp->world == 1, "decode with tensor parallelism is not implemented");
  require(max_new_tokens >= 1 && max_new_tokens <= (1 << 20), "max_new_tokens out of range");
  tp->ex.enable_decode(max_new_tokens);
  TIDAL_CATCH
}

tidal_status tidal_invoke_decode(tidal_template* tp, const tidal_adapter* ca, int n_steps,
                                 int32_t* tokens_out, float* logits_out,
                                 tidal_decode_stats* stats) {
  TIDAL_TRY
  require(tp && tokens_out, "null argument");
  require(!tp->dry, "dry template cannot decode");
  Exec& ex = tp->ex;
  require(ex.dec.kc != nullptr, "decode not enabled (tidal_template_enable_decode)");
  require(ex.dec.prompt_len > 0, "decode must follow a single-prompt prefill");
  require(tp->suffix_valid, "streamed weights are not all on the device");
  auto* a = const_cast<tidal_adapter*>(ca);
  if (a) require(a->tpl == tp, "adapter attached to another template");
  const std::shared_ptr<AdapterPlan> hold = a ? a->ap : nullptr;
  const TensorTable& tt = a ? hold->tt : tp->tt;
  const void* akey = a ? (const void*)tp->arena : nullptr;
  require(ex.dec.prompt_akey == akey && ex.dec.prompt_gen == tp->gen &&
              ex.dec.prompt_adapter == (a ? a->serial : 0) && (!a || a->ap->gen == tp->gen),
          "decode must use the adapter of the preceding prefill");
  require(n_steps >= 1 && n_steps <= ex.dec.max_new, "n_steps out of range (1..max_new_tokens)");
  cuda_check(cudaSetDevice(tp->device), "cudaSetDevice");
  ex.launches = 0;
  cuda_check(cudaEventRecord(tp->e_start, ex.compute), "event");
  run_decode(ex, tt, n_steps, a ? a->scale : 1.f, akey, tp->gen, logits_out != nullptr);
  cuda_check(cudaEventRecord(tp->e_end, ex.compute), "event");
  cuda_check(cudaMemcpyAsync(tokens_out, ex.dec.toks, 4ull * n_steps, cudaMemcpyDeviceToHost,
                             ex.compute),
             "D2H tokens");
  if (logits_out)
    cuda_check(cudaMemcpyAsync(logits_out, ex.dec.logits_all, 4ull * n_steps * tp->shape.vocab,
                               cudaMemcpyDeviceToHost, ex.compute),
               "D2H logits");
  cuda_check(cudaStreamSynchronize(ex.compute), "decode");
  if (stats) {
    memset(stats, 0, sizeof *stats);
    float ms = 0;
    cudaEventElapsedTime(&ms, tp->e_start, tp->e_end);
    stats->device_ms = ms;
    stats->per_token_ms = ms / n_steps;
    uint64_t wb = 0;
    for (int id = 0; id < (int)tt.t.size(); ++id) {
      const TensorInfo& ti = tt.t[id];
      if (ti.role == R_EMBED && id != tt.head) {
        wb += ti.bytes / std::max(1, ti.rows);  // one row gathered
      } else if (!ti.adapter || tt.lora_rank) {
        wb += ti.bytes;
      }
    }
    stats->weight_bytes_per_token = wb;
    const ModelShape& m = tp->shape;
    stats->kv_bytes_last_token = 2ull * m.n_layers * (uint64_t)(ex.dec.prompt_len + n_steps) *
                                 m.n_kv_heads * m.head_dim() * 2;
    stats->n_kernels = ex.launches;
  }
  for (int i = 0; i < n_steps; ++i)
    require(tokens_out[i] >= 0 && tokens_out[i] < tp->shape.vocab, "NaN in decode logits",
            TIDAL_ERR_NUMERIC);
  TIDAL_CATCH
}

tidal_status tidal_host_alloc(uint64_t bytes, void** out) {
  TIDAL_TRY
  require(out != nullptr, "null argument");
  cuda_check(cudaHostAlloc(out, bytes ? bytes : 16, cudaHostAllocPortable), "cudaHostAlloc");
  TIDAL_CATCH
}

void tidal_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

tidal_status tidal_comm_unique_id(void* out128) {
  TIDAL_TRY
  require(out128 != nullptr, "null argument");
  nccl_unique_id(out128);
  TIDAL_CATCH
}

tidal_status tidal_comm_create(int world, int rank, const void* id, int device, tidal_comm** out) {
  TIDAL_TRY
  require(out && id && world >= 1 && rank >= 0 && rank < world, "bad argument");
  auto* c = new tidal_comm();
  c->world = world;
  c->rank = rank;
  c->device = device;
  {  // also at world 1 (a valid one-rank NCCL communicator; tidal_comm_selftest uses it)
    try {
      c->impl = nccl_comm_create(world, rank, id, device);
    } catch (...) {
      delete c;
      throw;
    }
  }
  *out = c;
  TIDAL_CATCH
}

tidal_status tidal_comm_create_local(int world, int rank, const char* group, int device,
                                     tidal_comm** out) {
  TIDAL_TRY
  require(out && group && world >= 1 && rank >= 0 && rank < world, "bad argument");
  auto* c = new tidal_comm();
  c->world = world;
  c->rank = rank;
  c->device = device;
  if (world > 1) {
    try {
      c->impl = local_comm_create(world, rank, group, device);
    } catch (...) {
      delete c;
      throw;
    }
  }
  *out = c;
  TIDAL_CATCH
}

tidal_status tidal_comm_selftest(tidal_comm* c, uint64_t n) {
  TIDAL_TRY
  require(c != nullptr && c->impl != nullptr, "communicator has no implementation (world 1 local)");
  require(n >= 1 && n <= (1ull << 26), "n out of range");
  comm_selftest(c->impl, (size_t)n);
  TIDAL_CATCH
}

void tidal_comm_destroy(tidal_comm* c) {
  if (!c) return;
  delete c->impl;
  delete c;
}

tidal_status tidal_set_debug(tidal_template* tp, int flags, int arg) {
  TIDAL_TRY
  require(tp != nullptr, "null template");
  tp->debug = flags;
  tp->debug_arg = arg;
  TIDAL_CATCH
}

tidal_status tidal_set_device_allocator(void* (*alloc)(size_t, int, void*),
                                       void (*free_)(void*, int, void*), void* ctx) {
  TIDAL_TRY
  require((alloc == nullptr) == (free_ == nullptr), "alloc and free must both be set or both NULL");
  set_device_allocator(alloc, free_, ctx);
  TIDAL_CATCH
}

tidal_status tidal_timeline_read(tidal_template* tp, double* group_end_ms, int cap_groups,
                                 double* op_start_ms, int cap_ops, int* n_groups, int* n_ops,
                                 double* end_ms) {
  TIDAL_TRY
  require(tp != nullptr, "null template");
  require(!tp->tl_op_ms.empty(), "no timeline recorded (invoke with TIDAL_DEBUG_TIMELINE)");
  if (n_groups) *n_groups = (int)tp->tl_group_ms.size();
  if (n_ops) *n_ops = (int)tp->tl_op_ms.size();
  if (end_ms) *end_ms = tp->tl_end_ms;
  if (group_end_ms) {
    require(cap_groups >= (int)tp->tl_group_ms.size(), "group buffer too small", TIDAL_ERR_BUFSZ);
    std::copy(tp->tl_group_ms.begin(), tp->tl_group_ms.end(), group_end_ms);
  }
  if (op_start_ms) {
    require(cap_ops >= (int)tp->tl_op_ms.size(), "op buffer too small", TIDAL_ERR_BUFSZ);
    std::copy(tp->tl_op_ms.begin(), tp->tl_op_ms.end(), op_start_ms);
  }
  TIDAL_CATCH
}

tidal_status tidal_set_allreduce_dtype(tidal_template* tp, int dtype) {
  TIDAL_TRY
  require(tp != nullptr, "null template");
  require(dtype == TIDAL_DTYPE_F32 || dtype == TIDAL_DTYPE_BF16, "dtype must be F32 or BF16");
  tp->ex.ar_bf16 = dtype == TIDAL_DTYPE_BF16;
  TIDAL_CATCH
}

tidal_status tidal_profile_read(tidal_template* tp, tidal_kernel_time* out, int cap, int* n,
                                int reset) {
  TIDAL_TRY
  require(tp != nullptr, "null template");
  Exec& ex = tp->ex;
  if (ex.prof_tot.size() < KC_COUNT) ex.prof_tot.resize(KC_COUNT);
  if (n) *n = KC_COUNT;
  for (int i = 0; i < KC_COUNT && i < cap && out; ++i) {
    out[i].name = kKernelClassNames[i];
    out[i].total_ms = ex.prof_tot[i].ms;
    out[i].launches = ex.prof_tot[i].launches;
    out[i].flops = ex.prof_tot[i].flops;
    out[i].bytes = ex.prof_tot[i].bytes;
  }
  if (reset) ex.prof_tot.assign(KC_COUNT, Exec::ProfTot());
  TIDAL_CATCH
}

tidal_status tidal_template_checksum(tidal_template* tp, uint64_t* out) {
  TIDAL_TRY
  require(tp && out && !tp->dry, "bad argument");
  cuda_check(cudaSetDevice(tp->device), "cudaSetDevice");
  cuda_check(checksum_launch(tp->dev, tp->plan.resident_end, tp->d_sum, tp->ex.compute), "checksum");
  unsigned long long h = 0;
  cuda_check(cudaMemcpyAsync(&h, tp->d_sum, 8, cudaMemcpyDeviceToHost, tp->ex.compute), "D2H");
  cuda_check(cudaStreamSynchronize(tp->ex.compute), "checksum");
  *out = h;
  TIDAL_CATCH
}

tidal_status tidal_weight_ptr(const tidal_template* tp, const char* name, void** dev_out) {
  TIDAL_TRY
  require(tp && name && dev_out && !tp->dry, "bad argument");
  const int id = tp->tt.find(name);
  require(id >= 0 && id < tp->tt.n_base, std::string("unknown weight ") + name);
  *dev_out = tp->dev + tp->plan.offset[id];
  TIDAL_CATCH
}

// ---------------- kernel-level entry points (include/tidal_kernels.h) ----------------
static int g_sms = 0;
static int sms() {
  if (!g_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return g_sms;
}

static tidal_status sync_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return set_err(TIDAL_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return TIDAL_OK;
}

tidal_status tidal_k_rmsnorm(const float* X, const void* g, void* Y, int S, int d, float eps) {
  return sync_status(rmsnorm_launch(X, (const bf16*)g, (bf16*)Y, S, d, eps, 0), "rmsnorm");
}

tidal_status tidal_k_embed(const int32_t* tok, const void* E, float* X, int S, int d, int row0,
                           int rows) {
  return sync_status(embed_launch(tok, (const bf16*)E, X, S, d, row0, rows, 0), "embed");
}

tidal_status tidal_k_lora_shrink(const void* X, int M, int K, const void* A, void* T, int r,
                                 float scale) {
  const bf16* As[1] = {(const bf16*)A};
  bf16* Ts[1] = {(bf16*)T};
  TIDAL_TRY
  float* ws = nullptr;
  cuda_check(cudaMalloc(&ws, (size_t)SHRINK_MAX_SPLIT * M * r * 4 + 16), "cudaMalloc(ws)");
  ShrinkPlan sp;
  const bool ok = shrink_plan(&sp, (const bf16*)X, M, K, As, Ts, 1, r, ws, sms());
  tidal_status st = ok ? sync_status(shrink_run(sp, scale, sms(), 0), "shrink")
                       : set_err(TIDAL_ERR_INVALID, "shrink tensor maps");
  cudaFree(ws);
  return st;
  TIDAL_CATCH
}

tidal_status tidal_k_attention(const void* qkv, void* O, int S, int H, int KV, int hd) {
  return sync_status(attention_launch((const bf16*)qkv, (bf16*)O, S, H, KV, hd, 0), "attention");
}

tidal_status tidal_k_attention_tc(const void* qkv, const void* vt, int vt_ld, void* O, int S, int H,
                                  int KV) {
  TIDAL_TRY
  AttnParams p;
  memset(&p, 0, sizeof p);
  require(attn_tc_params(&p, (const bf16*)qkv, (const bf16*)vt, vt_ld, (bf16*)O, S, H, KV),
          "attention tensor maps");
  // per-call variant (tests exercise both kernels): TIDAL_ATTN=1 single, 2 pairs
  if (const char* v = getenv("TIDAL_ATTN")) p.variant = atoi(v);
  const char* rep = getenv("TIDAL_K_REPEAT");  // timing harness: n launches back to back
  const int reps = rep && atoi(rep) > 0 ? atoi(rep) : 1;
  // diagnostic: TIDAL_ATTN_TRACE=<file> dumps a per-tile timeline of the last launch
  const char* trace = getenv("TIDAL_ATTN_TRACE");
  const size_t tn = (size_t)sms() * 64 * 8;
  if (trace) {
    cuda_check(cudaMalloc(&p.dbg, tn * 8), "cudaMalloc(trace)");
    cuda_check(cudaMemset(p.dbg, 0, tn * 8), "memset(trace)");
  }
  cudaError_t e = cudaSuccess;
  for (int i = 0; i < reps && e == cudaSuccess; ++i) e = attn_tc_launch(p, 0);
  tidal_status s = sync_status(e, "attention_tc");
  if (trace && p.dbg) {
    std::vector<unsigned long long> h(tn);
    cudaMemcpy(h.data(), p.dbg, tn * 8, cudaMemcpyDeviceToHost);
    cudaFree(p.dbg);
    if (FILE* f = fopen(trace, "wb")) {
      fwrite(h.data(), 8, h.size(), f);
      fclose(f);
    }
  }
  if (s != TIDAL_OK) return s;
  TIDAL_CATCH
}

tidal_status tidal_k_head(const float* xlast, const void* g, const void* W, int V, int d, float eps,
                          float* logits, unsigned long long* key) {
  cudaError_t e = cudaMemset(key, 0, 8);
  if (e == cudaSuccess)
    e = head_launch(xlast, 0, 1, (const bf16*)g, (const bf16*)W, V, d, eps, logits, V, key, 0, sms(), 0);
  return sync_status(e, "head");
}

tidal_status tidal_k_gemm(int epi, const void* A, const void* const* W, const int* seg_n, int nseg,
                          void* out, int ldo, int M, int K, const void* const* T,
                          const void* const* B, int r, const void* rope, int head_dim) {
  TIDAL_TRY
  const int epi_code = epi;
  const int cg_req = (epi >> 20) & 0x3;  // bits 20-21: CTA group (0 = auto)
  const int mc_req = (epi >> 22) & 0x3;  // bits 22-23: CTA pairs per cluster (0 = auto)
  const int ks_req = (epi >> 24) & 0xF;  // bits 24-27: EPI_RESID split-K parts (0 = auto)
  const int bn_req = (epi >> 8) & 0x1FF;  // bits 8-16: N tile (0 = auto)
  epi &= 0xFF;
  require(epi >= 0 && epi <= 3 && nseg >= 1 && nseg <= 3, "bad gemm arguments");
  for (int i = 0; i < nseg; ++i) require(seg_n[i] > 0 && seg_n[i] % 8 == 0, "seg_n must be a positive multiple of 8");
  require(K > 0 && K % 8 == 0 && M > 0, "K must be a positive multiple of 8, M positive");
  require(ldo % (epi == 3 ? 4 : 8) == 0, "ldo must keep output rows 16-byte aligned");
  GemmParams p;
  memset(&p, 0, sizeof p);
  p.bn = bn_req ? bn_req : gemm_pick_bn(epi, M, seg_n, epi == EPI_SILU ? 1 : nseg, sms());
  require(p.bn == 256 || p.bn == 192 || p.bn == 128, "bn must be 256, 192 or 128");
  if (epi == EPI_SILU) p.bn = 128;
  if (epi == EPI_ROPE && p.bn == 192) p.bn = 256;
  p.cg = cg_req ? cg_req : gemm_pick_cg(M);
  require(p.cg == 1 || p.cg == 2, "cg must be 1 or 2");
  p.mc = mc_req ? mc_req : (p.cg == 2 ? gemm_pick_mc(M, sms()) : 1);
  require(p.mc == 1 || (p.mc == 2 && p.cg == 2), "mc must be 1, or 2 with cg 2");
  if (epi == EPI_RESID) {
    int bn_auto = 256, ks = 1, nfull = 0;
    const bool tail_req = (epi_code >> 28) & 1;  // bit 28: tail split (whole tiles for full waves)
    gemm_plan_resid(M, seg_n[0], K, sms(), &bn_auto, &ks, nullptr, true, &nfull);
    if (ks_req) ks = ks_req;
    const int nk = (K + GEMM_BK - 1) / GEMM_BK;
    require(ks >= 1 && ks <= nk, "bad split-K");
    p.kblocks_per_split = (nk + ks - 1) / ks;
    p.ksplit = (nk + p.kblocks_per_split - 1) / p.kblocks_per_split;  // parts non-empty
    if (!bn_req) p.bn = bn_auto;
    if (ks_req) {  // explicit request: tail mode only with bit 28
      nfull = 0;
      if (tail_req && p.ksplit > 1) {
        const int units = gemm_units(p.cg, p.mc, sms());
        const int tiles = gemm_m_tiles(M, p.cg, p.mc) * ((seg_n[0] + p.bn - 1) / p.bn);
        nfull = tiles / units * units;
        if (nfull >= tiles) nfull = 0;
      }
    } else if (bn_req && bn_req != bn_auto) {
      nfull = 0;
    }
    p.n_full = p.ksplit > 1 ? nfull : 0;
    static int* flags = nullptr;  // per process; this entry is synchronous
    if (!flags) {
      cudaError_t e = cudaMalloc(&flags, GEMM_MAX_FLAGS * sizeof(int));
      if (e == cudaSuccess) e = cudaMemset(flags, 0, GEMM_MAX_FLAGS * sizeof(int));
      if (e != cudaSuccess) return sync_status(e, "gemm flags");
    }
    p.flags = flags;
  }
  const int bbox = gemm_b_box(epi, p.bn, p.cg, p.mc), tbbox = gemm_tb_box(epi, p.bn, p.cg, p.mc);
  auto mk = [&](CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box) {
    require(make_tmap(m, base, rows, cols, cols * 2, box, 64), "tensor map encode failed");
  };
  mk(&p.a, A, M, K, 128);
  const int mt = gemm_m_tiles(M, p.cg, p.mc);
  p.M = M;
  p.K = K;
  p.m_tiles = mt;
  p.out = out;
  p.ldo = ldo;
  p.rope = (const float2*)rope;
  p.head_dim = head_dim;
  p.lora_r = (T && B) ? r : 0;
  if (epi == EPI_SILU) {
    mk(&p.b[0], W[0], seg_n[0], K, bbox);
    mk(&p.b[1], W[1], seg_n[0], K, bbox);
    if (p.lora_r) {
      mk(&p.ta[0], T[0], M, r, 128);
      mk(&p.ta[1], T[1], M, r, 128);
      mk(&p.tb[0], B[0], seg_n[0], r, tbbox);
      mk(&p.tb[1], B[1], seg_n[0], r, tbbox);
    }
    p.nseg = 1;
    p.seg[0].n = seg_n[0];
    p.seg[0].lora = p.lora_r > 0;
    p.n_tiles[0] = (seg_n[0] + 127) / 128;
    p.total_tiles = p.n_tiles[0] * mt;
  } else {
    int col = 0;
    p.nseg = nseg;
    for (int s = 0; s < nseg; ++s) {
      mk(&p.b[s], W[s], seg_n[s], K, bbox);
      p.seg[s].n = seg_n[s];
      p.seg[s].out_col = col;
      p.seg[s].rope = (epi == EPI_ROPE) && s < 2;
      p.seg[s].lora = p.lora_r > 0 && T[s] && B[s];
      if (p.seg[s].lora) {
        mk(&p.ta[s], T[s], M, r, 128);
        mk(&p.tb[s], B[s], seg_n[s], r, tbbox);
      }
      col += seg_n[s];
      p.n_tiles[s] = (seg_n[s] + p.bn - 1) / p.bn;
      p.total_tiles += p.n_tiles[s] * mt;
    }
  }
  // TIDAL_K_REPEAT=n launches the same GEMM n times back to back (timing
  // harness tools/gemm_bench.py; epilogues that accumulate keep accumulating)
  const char* rep = getenv("TIDAL_K_REPEAT");
  const int reps = rep ? atoi(rep) : 1;
  cudaError_t e = cudaSuccess;
  for (int i = 0; i < (reps > 0 ? reps : 1) && e == cudaSuccess; ++i) e = gemm_launch(p, epi, sms(), 0);
  tidal_status s = sync_status(e, "gemm");
  if (s != TIDAL_OK) return s;
  TIDAL_CATCH
}

}  // extern "C"
