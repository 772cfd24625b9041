// vmm.cu — template device memory on CUDA virtual memory management, so the
// read-only template can be shared with other processes (
// PAPER.md §3/§5: the template server keeps function templates on the GPU and
// function processes fork from them over CUDA IPC).
//
// One virtual range per template, backed by equal physical chunks (each a
// separate allocation with a POSIX-fd shareable handle).  The exporter hands
// out the fds of the chunks that lie entirely inside the resident prefix; an
// importer reserves its own range of the same size, maps those chunks
// read-only at the same offsets and backs the rest (the prefix tail and the
// streaming arena) with private chunks — so the template keeps one contiguous
// access-ordered address space in every process and no process can write
// another's template bytes.  Driver entry points are resolved through the
// runtime (no link-time libcuda dependency).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <mutex>
#include <string>

#include "runtime.h"

namespace tidal {

namespace {

struct Drv {
  CUresult (*granularity)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags);
  CUresult (*reserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
  CUresult (*addr_free)(CUdeviceptr, size_t);
  CUresult (*create)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*,
                     unsigned long long);
  CUresult (*release)(CUmemGenericAllocationHandle);
  CUresult (*map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
  CUresult (*unmap)(CUdeviceptr, size_t);
  CUresult (*set_access)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
  CUresult (*export_h)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType,
                       unsigned long long);
  CUresult (*import_h)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType);
  bool ok = false;
};

Drv g_drv;
std::once_flag g_drv_once;

template <typename F>
bool resolve(const char* name, F& fn) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !p)
    return false;
  fn = reinterpret_cast<F>(p);
  return true;
}

const Drv& drv() {
  std::call_once(g_drv_once, [] {
    Drv& d = g_drv;
    d.ok = resolve("cuMemGetAllocationGranularity", d.granularity) &&
           resolve("cuMemAddressReserve", d.reserve) && resolve("cuMemAddressFree", d.addr_free) &&
           resolve("cuMemCreate", d.create) && resolve("cuMemRelease", d.release) &&
           resolve("cuMemMap", d.map) && resolve("cuMemUnmap", d.unmap) &&
           resolve("cuMemSetAccess", d.set_access) &&
           resolve("cuMemExportToShareableHandle", d.export_h) &&
           resolve("cuMemImportFromShareableHandle", d.import_h);
  });
  return g_drv;
}

void cu_check(CUresult r, const char* what) {
  if (r != CUDA_SUCCESS) {
    if (r == CUDA_ERROR_OUT_OF_MEMORY) fail(2, std::string(what) + ": out of device memory");
    fail(3, std::string(what) + ": CUresult " + std::to_string((int)r));
  }
}

CUmemAllocationProp prop_of(int device) {
  CUmemAllocationProp p = {};
  p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  p.location.id = device;
  p.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  return p;
}

void set_access(CUdeviceptr va, size_t bytes, int device, bool read_only) {
  CUmemAccessDesc a = {};
  a.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  a.location.id = device;
  a.flags = read_only ? CU_MEM_ACCESS_FLAGS_PROT_READ : CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  cu_check(drv().set_access(va, bytes, &a, 1), "cuMemSetAccess");
}

}  // namespace

// TIDAL_VMM=0 falls back to cudaMalloc'd templates (no export / import)
bool vmm_available() {
  static const bool off = [] {
    const char* e = getenv("TIDAL_VMM");
    return e && e[0] == '0';
  }();
  return !off && drv().ok;
}

// chunk size: about 1/64 of the buffer, a multiple of the allocation
// granularity, at most 512 MB (so an exported template is <= ~64 fds)
static size_t chunk_size(size_t bytes, int device) {
  size_t g = 0;
  const CUmemAllocationProp p = prop_of(device);
  cu_check(drv().granularity(&g, &p, CU_MEM_ALLOC_GRANULARITY_MINIMUM), "cuMemGetAllocationGranularity");
  size_t c = (bytes / 64 + g - 1) / g * g;
  if (c < g) c = g;
  const size_t cap = (size_t)512 << 20;
  if (c > cap) c = cap / g * g;
  return c;
}

void vmm_alloc(VmmBuf& b, size_t bytes, int device, const int* fds, int n_shared) {
  if (!vmm_available()) fail(3, "CUDA virtual memory management unavailable");
  b = VmmBuf();
  b.device = device;
  b.chunk = chunk_size(bytes, device);
  const size_t n = (bytes + b.chunk - 1) / b.chunk;
  b.size = n * b.chunk;
  if (n_shared < 0 || (size_t)n_shared > n) fail(1, "more shared chunks than the template holds");
  cu_check(drv().reserve(&b.va, b.size, 0, 0, 0), "cuMemAddressReserve");
  b.h.assign(n, 0);
  b.n_shared = n_shared;
  const CUmemAllocationProp p = prop_of(device);
  try {
    for (size_t i = 0; i < n; ++i) {
      if ((int)i < n_shared) {
        cu_check(drv().import_h(&b.h[i], (void*)(uintptr_t)fds[i],
                                CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
                 "cuMemImportFromShareableHandle");
      } else {
        cu_check(drv().create(&b.h[i], b.chunk, &p, 0), "cuMemCreate");
      }
      cu_check(drv().map(b.va + i * b.chunk, b.chunk, 0, b.h[i], 0), "cuMemMap");
      set_access(b.va + i * b.chunk, b.chunk, device, (int)i < n_shared);
    }
  } catch (...) {
    vmm_free(b);
    throw;
  }
}

void vmm_free(VmmBuf& b) {
  if (!b.va) return;
  for (size_t i = 0; i < b.h.size(); ++i) {
    if (b.h[i]) {
      drv().unmap(b.va + i * b.chunk, b.chunk);
      drv().release(b.h[i]);
    }
  }
  drv().addr_free(b.va, b.size);
  b = VmmBuf();
}

int vmm_export_fd(const VmmBuf& b, size_t i) {
  if (i >= b.h.size() || (int)i < b.n_shared) fail(1, "chunk not exportable");
  int fd = -1;
  cu_check(drv().export_h(&fd, b.h[i], CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0),
           "cuMemExportToShareableHandle");
  return fd;
}

}  // namespace tidal
