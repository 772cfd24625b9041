// comm.cu — tensor-parallel exchange steps: allreduce of the
// row-parallel partial sums (C1/C2) and of the vocab-parallel embedding (C3),
// max-reduce of the packed argmax key and allgather of logit slices (C4).
//
// Two implementations of the same three collectives behind `Comm`:
//   NcclComm   one process per GPU (the deployment path; bench.py under
//              torchrun).  NCCL is resolved at run time with dlopen (the
//              torch-bundled libnccl.so.2 is already mapped in a torch
//              process), so the library loads on boxes without it.
//   LocalComm  the ranks of one process (one thread per rank), over device
//              pointers: each rank publishes its buffer, every rank reduces
//              all ranks' buffers in rank order into private scratch, and a
//              second rendezvous keeps a buffer alive until every peer read
//              it.  Ranks may share a GPU, so TP=N runs (and is tested) on a
//              single device; across GPUs it needs peer access, enabled at
//              create.  Rendezvous are host-side (the collective's enqueue
//              blocks until all ranks enqueued theirs); ordering on the
//              device is by cross-stream events.  Sums are left folds in rank
//              order, so every rank holds bit-identical results (like NCCL).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "runtime.h"

namespace tidal {

namespace {
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
enum { ncclSuccess = 0 };
enum { ncclUint64 = 5, ncclFloat32 = 7, ncclBfloat16 = 9 };
enum { ncclSum = 0, ncclMax = 2 };

struct NcclApi {
  int (*GetUniqueId)(ncclUniqueId*) = nullptr;
  int (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
  bool ok = false;
};
NcclApi g_nccl;
std::once_flag g_nccl_once;

const NcclApi& nccl() {
  std::call_once(g_nccl_once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    void* h = nullptr;
    for (const char* n : names)
      if ((h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!h) return;
    g_nccl.GetUniqueId = (int (*)(ncclUniqueId*))dlsym(h, "ncclGetUniqueId");
    g_nccl.CommInitRank = (int (*)(ncclComm_t*, int, ncclUniqueId, int))dlsym(h, "ncclCommInitRank");
    g_nccl.AllReduce = (int (*)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t))dlsym(
        h, "ncclAllReduce");
    g_nccl.AllGather =
        (int (*)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t))dlsym(h, "ncclAllGather");
    g_nccl.CommDestroy = (int (*)(ncclComm_t))dlsym(h, "ncclCommDestroy");
    g_nccl.GetErrorString = (const char* (*)(int))dlsym(h, "ncclGetErrorString");
    g_nccl.ok = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.AllReduce && g_nccl.AllGather &&
                g_nccl.CommDestroy;
  });
  return g_nccl;
}

void nccl_check(int r, const char* what) {
  if (r != ncclSuccess) {
    const char* s = g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?";
    fail(4, std::string(what) + ": " + s);
  }
}

struct NcclComm final : Comm {
  ncclComm_t c = nullptr;
  ~NcclComm() override {
    if (c && g_nccl.ok) g_nccl.CommDestroy(c);
  }
  void allreduce_f32(float* buf, size_t n, cudaStream_t s) override {
    nccl_check(g_nccl.AllReduce(buf, buf, n, ncclFloat32, ncclSum, c, s), "ncclAllReduce");
  }
  void allreduce_bf16(bf16* buf, size_t n, cudaStream_t s) override {
    nccl_check(g_nccl.AllReduce(buf, buf, n, ncclBfloat16, ncclSum, c, s), "ncclAllReduce(bf16)");
  }
  void max_u64(unsigned long long* key, size_t n, cudaStream_t s) override {
    nccl_check(g_nccl.AllReduce(key, key, n, ncclUint64, ncclMax, c, s), "ncclAllReduce(max)");
  }
  void allgather_f32(float* buf, size_t n, cudaStream_t s) override {
    nccl_check(g_nccl.AllGather(buf + (size_t)rank * n, buf, n, ncclFloat32, c, s), "ncclAllGather");
  }
};

// ---------------- in-process ranks ----------------
constexpr int kMaxLocal = 8;
struct SrcPtrs {
  const float* p[kMaxLocal];
  int n;
};

__global__ void sum_ranks_kernel(SrcPtrs src, float* __restrict__ out, size_t n4) {
  // out = ((src0 + src1) + src2) + ...   (rank order: identical on every rank)
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4;
       i += (size_t)gridDim.x * blockDim.x) {
    float4 acc = reinterpret_cast<const float4*>(src.p[0])[i];
    for (int k = 1; k < src.n; ++k) {
      const float4 v = reinterpret_cast<const float4*>(src.p[k])[i];
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    reinterpret_cast<float4*>(out)[i] = acc;
  }
}

// bf16 sum in rank order, accumulated in fp32, rounded once (8 elements per thread)
__global__ void sum_ranks_bf16_kernel(SrcPtrs src, bf16* __restrict__ out, size_t n8) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n8;
       i += (size_t)gridDim.x * blockDim.x) {
    float acc[8];
    for (int k = 0; k < src.n; ++k) {
      const uint4 v = reinterpret_cast<const uint4*>(src.p[k])[i];
      const bf16* h = reinterpret_cast<const bf16*>(&v);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = k ? acc[j] + __bfloat162float(h[j]) : __bfloat162float(h[j]);
    }
    uint4 o;
    bf16* ho = reinterpret_cast<bf16*>(&o);
#pragma unroll
    for (int j = 0; j < 8; ++j) ho[j] = __float2bfloat16_rn(acc[j]);
    reinterpret_cast<uint4*>(out)[i] = o;
  }
}

__global__ void max_ranks_kernel(SrcPtrs src, unsigned long long* out, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    unsigned long long m = 0;
    for (int k = 0; k < src.n; ++k) {
      const unsigned long long v = reinterpret_cast<const unsigned long long*>(src.p[k])[i];
      m = v > m ? v : m;
    }
    out[i] = m;
  }
}

struct LocalGroup {
  int world;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t phase = 0;
  void* ptr[kMaxLocal] = {};
  cudaEvent_t ev_a[kMaxLocal] = {}, ev_b[kMaxLocal] = {};
  int joined = 0;

  void rendezvous() {
    std::unique_lock<std::mutex> lk(m);
    const uint64_t ph = phase;
    if (++arrived == world) {
      arrived = 0;
      ++phase;
      cv.notify_all();
    } else if (!cv.wait_for(lk, std::chrono::seconds(120), [&] { return phase != ph; })) {
      fail(4, "local communicator: a peer rank never reached the collective (120 s)");
    }
  }
};

std::mutex g_groups_mu;
std::map<std::string, std::weak_ptr<LocalGroup>> g_groups;

struct LocalComm final : Comm {
  std::shared_ptr<LocalGroup> g;
  float* scratch = nullptr;
  size_t scratch_n = 0;
  unsigned long long* kscratch = nullptr;

  ~LocalComm() override {
    if (scratch) cudaFree(scratch);
    if (kscratch) cudaFree(kscratch);
    if (g) {
      cudaEventDestroy(g->ev_a[rank]);
      cudaEventDestroy(g->ev_b[rank]);
    }
  }
  // Phase 1: publish `p`, order this stream after every peer's producer.
  void publish(void* p, cudaStream_t s) {
    g->ptr[rank] = p;
    cuda_check(cudaEventRecord(g->ev_a[rank], s), "cudaEventRecord");
    g->rendezvous();
    for (int k = 0; k < world; ++k)
      if (k != rank) cuda_check(cudaStreamWaitEvent(s, g->ev_a[k], 0), "cudaStreamWaitEvent");
  }
  // Phase 2: after this rank's reads of peer buffers, wait until every peer's
  // reads of ours are done before anything later on `s` may overwrite it.
  void retire(cudaStream_t s) {
    cuda_check(cudaEventRecord(g->ev_b[rank], s), "cudaEventRecord");
    g->rendezvous();
    for (int k = 0; k < world; ++k)
      if (k != rank) cuda_check(cudaStreamWaitEvent(s, g->ev_b[k], 0), "cudaStreamWaitEvent");
  }
  SrcPtrs srcs() const {
    SrcPtrs sp;
    sp.n = world;
    for (int k = 0; k < world; ++k) sp.p[k] = static_cast<const float*>(g->ptr[k]);
    return sp;
  }
  void allreduce_f32(float* buf, size_t n, cudaStream_t s) override {
    if (n % 4) fail(1, "local allreduce: length must be a multiple of 4");
    if (n > scratch_n) {
      if (scratch) cudaFree(scratch);
      scratch = nullptr;
      cuda_check(cudaMalloc(&scratch, n * 4), "cudaMalloc(comm scratch)");
      scratch_n = n;
    }
    publish(buf, s);
    const SrcPtrs sp = srcs();
    sum_ranks_kernel<<<4 * 148, 256, 0, s>>>(sp, scratch, n / 4);  // plain launch: no PDL overlap
    cuda_check(cudaGetLastError(), "sum_ranks");
    retire(s);
    cuda_check(cudaMemcpyAsync(buf, scratch, n * 4, cudaMemcpyDeviceToDevice, s), "D2D");
  }
  void allreduce_bf16(bf16* buf, size_t n, cudaStream_t s) override {
    if (n % 8) fail(1, "local allreduce: bf16 length must be a multiple of 8");
    if (n * 2 > scratch_n * 4) {
      if (scratch) cudaFree(scratch);
      scratch = nullptr;
      cuda_check(cudaMalloc(&scratch, n * 2), "cudaMalloc(comm scratch)");
      scratch_n = (n * 2 + 3) / 4;
    }
    publish(buf, s);
    sum_ranks_bf16_kernel<<<4 * 148, 256, 0, s>>>(srcs(), reinterpret_cast<bf16*>(scratch), n / 8);
    cuda_check(cudaGetLastError(), "sum_ranks_bf16");
    retire(s);
    cuda_check(cudaMemcpyAsync(buf, scratch, n * 2, cudaMemcpyDeviceToDevice, s), "D2D");
  }
  void max_u64(unsigned long long* key, size_t n, cudaStream_t s) override {
    if (n > kMaxBatch) fail(1, "local max-reduce: too many keys");
    publish(key, s);
    max_ranks_kernel<<<1, 64, 0, s>>>(srcs(), kscratch, (int)n);
    cuda_check(cudaGetLastError(), "max_ranks");
    retire(s);
    cuda_check(cudaMemcpyAsync(key, kscratch, 8 * n, cudaMemcpyDeviceToDevice, s), "D2D");
  }
  void allgather_f32(float* buf, size_t n, cudaStream_t s) override {
    publish(buf, s);
    for (int k = 0; k < world; ++k)
      if (k != rank)
        cuda_check(cudaMemcpyAsync(buf + (size_t)k * n, static_cast<const float*>(g->ptr[k]) + (size_t)k * n,
                                   n * 4, cudaMemcpyDeviceToDevice, s),
                   "allgather D2D");
    retire(s);
  }
};
}  // namespace

bool nccl_unique_id(void* out128) {
  const NcclApi& n = nccl();
  if (!n.ok) fail(4, "libnccl.so.2 not found (tensor parallelism needs NCCL)");
  ncclUniqueId id;
  nccl_check(n.GetUniqueId(&id), "ncclGetUniqueId");
  memcpy(out128, &id, sizeof id);
  return true;
}

Comm* nccl_comm_create(int world, int rank, const void* id128, int device) {
  const NcclApi& n = nccl();
  if (!n.ok) fail(4, "libnccl.so.2 not found (tensor parallelism needs NCCL)");
  cuda_check(cudaSetDevice(device), "cudaSetDevice");
  ncclUniqueId id;
  memcpy(&id, id128, sizeof id);
  auto* c = new NcclComm();
  c->world = world;
  c->rank = rank;
  c->device = device;
  const int r = n.CommInitRank(&c->c, world, id, rank);
  if (r != ncclSuccess) {
    delete c;
    nccl_check(r, "ncclCommInitRank");
  }
  return c;
}

Comm* local_comm_create(int world, int rank, const std::string& key, int device) {
  if (world > kMaxLocal) fail(1, "local communicator: at most 8 ranks");
  cuda_check(cudaSetDevice(device), "cudaSetDevice");
  std::shared_ptr<LocalGroup> g;
  {
    std::lock_guard<std::mutex> lk(g_groups_mu);
    g = g_groups[key].lock();
    if (!g) {
      g = std::make_shared<LocalGroup>();
      g->world = world;
      g_groups[key] = g;
    }
  }
  if (g->world != world) fail(1, "local communicator: world size differs from the group's");
  {
    std::lock_guard<std::mutex> lk(g->m);
    if (g->ev_a[rank]) fail(1, "local communicator: rank joined twice");
    cuda_check(cudaEventCreateWithFlags(&g->ev_a[rank], cudaEventDisableTiming), "cudaEventCreate");
    cuda_check(cudaEventCreateWithFlags(&g->ev_b[rank], cudaEventDisableTiming), "cudaEventCreate");
    ++g->joined;
  }
  auto* c = new LocalComm();
  c->colocated = true;  // in-process ranks: assume they may share a device
  c->world = world;
  c->rank = rank;
  c->device = device;
  c->g = g;
  cuda_check(cudaMalloc(&c->kscratch, 8 * kMaxBatch), "cudaMalloc");
  // peers on other devices are read directly: enable access to all of them
  int ndev = 0;
  cudaGetDeviceCount(&ndev);
  for (int d = 0; d < ndev; ++d) {
    int can = 0;
    if (d != device && cudaDeviceCanAccessPeer(&can, device, d) == cudaSuccess && can) {
      const cudaError_t e = cudaDeviceEnablePeerAccess(d, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) cuda_check(e, "peer access");
      cudaGetLastError();
    }
  }
  return c;
}

// Exercise every collective of `c` on small buffers with exact expected values
// (integers representable in fp32 / bf16): allreduce f32 and bf16, the u64 max
// and the logits allgather.  Every rank of the communicator calls it at once.
void comm_selftest(Comm* c, size_t n) {
  n = (n + 7) / 8 * 8;
  const int W = c->world, R = c->rank;
  cuda_check(cudaSetDevice(c->device), "cudaSetDevice");
  cudaStream_t s = nullptr;
  cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
  std::vector<float> hf(n), hg((size_t)W * n, -1.f);
  std::vector<bf16> hb(n);
  std::vector<unsigned long long> hk(4);
  for (size_t i = 0; i < n; ++i) {
    hf[i] = (float)(R * 1000 + (int)(i % 997));
    hb[i] = __float2bfloat16_rn((float)((int)(i % 13) + R));
    hg[(size_t)R * n + i] = (float)(R + (int)(i % 100));
  }
  for (int j = 0; j < 4; ++j) hk[j] = (unsigned long long)j * 10 + R;
  float *f = nullptr, *g = nullptr;
  bf16* b = nullptr;
  unsigned long long* k = nullptr;
  cuda_check(cudaMalloc(&f, n * 4), "cudaMalloc");
  cuda_check(cudaMalloc(&g, (size_t)W * n * 4), "cudaMalloc");
  cuda_check(cudaMalloc(&b, n * 2), "cudaMalloc");
  cuda_check(cudaMalloc(&k, 32), "cudaMalloc");
  cuda_check(cudaMemcpy(f, hf.data(), n * 4, cudaMemcpyHostToDevice), "H2D");
  cuda_check(cudaMemcpy(g, hg.data(), (size_t)W * n * 4, cudaMemcpyHostToDevice), "H2D");
  cuda_check(cudaMemcpy(b, hb.data(), n * 2, cudaMemcpyHostToDevice), "H2D");
  cuda_check(cudaMemcpy(k, hk.data(), 32, cudaMemcpyHostToDevice), "H2D");
  c->allreduce_f32(f, n, s);
  c->allreduce_bf16(b, n, s);
  c->max_u64(k, 4, s);
  c->allgather_f32(g, n, s);
  cuda_check(cudaStreamSynchronize(s), "selftest");
  cuda_check(cudaMemcpy(hf.data(), f, n * 4, cudaMemcpyDeviceToHost), "D2H");
  cuda_check(cudaMemcpy(hg.data(), g, (size_t)W * n * 4, cudaMemcpyDeviceToHost), "D2H");
  cuda_check(cudaMemcpy(hb.data(), b, n * 2, cudaMemcpyDeviceToHost), "D2H");
  cuda_check(cudaMemcpy(hk.data(), k, 32, cudaMemcpyDeviceToHost), "D2H");
  cudaFree(f);
  cudaFree(g);
  cudaFree(b);
  cudaFree(k);
  cudaStreamDestroy(s);
  const int tri = W * (W - 1) / 2;
  for (size_t i = 0; i < n; ++i) {
    if (hf[i] != (float)(1000 * tri + W * (int)(i % 997))) fail(4, "selftest: allreduce f32 mismatch");
    if (__bfloat162float(hb[i]) != (float)(W * (int)(i % 13) + tri))
      fail(4, "selftest: allreduce bf16 mismatch");
    for (int q = 0; q < W; ++q)
      if (hg[(size_t)q * n + i] != (float)(q + (int)(i % 100))) fail(4, "selftest: allgather mismatch");
  }
  for (int j = 0; j < 4; ++j)
    if (hk[j] != (unsigned long long)j * 10 + (W - 1)) fail(4, "selftest: max_u64 mismatch");
}

void tp_allreduce_f32(Exec& ex, Comm* comm, float* buf, size_t n) {
  if (ex.world <= 1) return;
  if (!comm) fail(1, "tensor-parallel template without a communicator");
  comm->allreduce_f32(buf, n, ex.compute);
}

void tp_allreduce_bf16(Exec& ex, Comm* comm, bf16* buf, size_t n) {
  if (ex.world <= 1) return;
  if (!comm) fail(1, "tensor-parallel template without a communicator");
  comm->allreduce_bf16(buf, n, ex.compute);
}

void tp_argmax_reduce(Exec& ex, Comm* comm, unsigned long long* key, int nseq) {
  if (ex.world <= 1) return;
  if (!comm) fail(1, "tensor-parallel template without a communicator");
  comm->max_u64(key, (size_t)nseq, ex.compute);
}

// logits are [world][nseq][V / world]: rank r's slices are contiguous
void tp_allgather_logits(Exec& ex, Comm* comm, int nseq) {
  if (ex.world <= 1) return;
  if (!comm) fail(1, "tensor-parallel template without a communicator");
  comm->allgather_f32(ex.logits, (size_t)nseq * (ex.m.vocab / ex.world), ex.compute);
}

}  // namespace tidal
