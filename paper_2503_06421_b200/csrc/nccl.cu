// nccl.cu — tensor-parallel exchange steps: allreduce of the
// row-parallel partial sums (C1/C2) and of the vocab-parallel embedding (C3),
// max-reduce of the packed argmax key and allgather of logit slices (C4).
// NCCL is resolved at run time with dlopen (the torch-bundled libnccl.so.2 is
// already mapped in a torch process), so the library loads on boxes without it.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstring>
#include <mutex>

#include "runtime.h"

namespace tidal {

namespace {
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
enum { ncclSuccess = 0 };
enum { ncclUint64 = 5, ncclFloat32 = 7 };
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
}  // namespace

bool nccl_unique_id(void* out128) {
  const NcclApi& n = nccl();
  if (!n.ok) fail(4, "libnccl.so.2 not found (tensor parallelism needs NCCL)");
  ncclUniqueId id;
  nccl_check(n.GetUniqueId(&id), "ncclGetUniqueId");
  memcpy(out128, &id, sizeof id);
  return true;
}

void* nccl_comm_create(int world, int rank, const void* id128, int device) {
  const NcclApi& n = nccl();
  if (!n.ok) fail(4, "libnccl.so.2 not found (tensor parallelism needs NCCL)");
  cuda_check(cudaSetDevice(device), "cudaSetDevice");
  ncclUniqueId id;
  memcpy(&id, id128, sizeof id);
  ncclComm_t c = nullptr;
  nccl_check(n.CommInitRank(&c, world, id, rank), "ncclCommInitRank");
  return c;
}

void nccl_comm_destroy(void* c) {
  if (c && g_nccl.ok) g_nccl.CommDestroy((ncclComm_t)c);
}

void tp_allreduce_f32(Exec& ex, void* comm, float* buf, size_t n) {
  if (ex.world <= 1) return;
  if (!comm) fail(1, "tensor-parallel template without a communicator");
  nccl_check(g_nccl.AllReduce(buf, buf, n, ncclFloat32, ncclSum, (ncclComm_t)comm, ex.compute),
             "ncclAllReduce");
}

void tp_argmax_reduce(Exec& ex, void* comm, unsigned long long* key) {
  if (ex.world <= 1) return;
  nccl_check(g_nccl.AllReduce(key, key, 1, ncclUint64, ncclMax, (ncclComm_t)comm, ex.compute),
             "ncclAllReduce(max)");
}

void tp_allgather_logits(Exec& ex, void* comm) {
  if (ex.world <= 1) return;
  const size_t Vl = (size_t)ex.m.vocab / ex.world;
  nccl_check(g_nccl.AllGather(ex.logits + (size_t)ex.rank * Vl, ex.logits, Vl, ncclFloat32,
                              (ncclComm_t)comm, ex.compute),
             "ncclAllGather");
}

}  // namespace tidal
