// launch.cuh — kernel launch with programmatic dependent launch (PDL): the
// next kernel's CTAs may be scheduled (and run their prologue up to
// griddepcontrol.wait) while this one drains, hiding the per-kernel launch gap
// of the ~450-kernel forward.  Optional 2-CTA cluster dimension.
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <utility>

namespace tidal {

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("TIDAL_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

// No PDL attribute for the LoRA-shrink reduce, nor for launches whose tag is
// in TIDAL_PDL_OFF: with early launch on the LoRA-shrink reduce, the 13B-width
// S = 4096 / r = 64 parity sweep hung intermittently (watchdog trap, 4 of 5
// runs); bisected per kernel class, the reduce alone in plain stream order
// passes 10 of 10 with the same-box TTFT unchanged.
template <typename... KArgs, typename... Args>
cudaError_t launch_kt(const char* tag, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                      cudaStream_t s, int cluster_x, Args&&... args);

inline bool pdl_off_for(const char* tag) {
  // the reduce is always excluded (a user list only adds tags)
  static const char* off = getenv("TIDAL_PDL_OFF");
  if (!tag) return false;
  if (strcmp(tag, "reduce") == 0) return true;
  return off && strstr(off, tag) != nullptr;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     int cluster_x, Args&&... args) {
  return launch_kt(nullptr, kernel, grid, block, smem, s, cluster_x, std::forward<Args>(args)...);
}

template <typename... KArgs, typename... Args>
cudaError_t launch_kt(const char* tag, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                      cudaStream_t s, int cluster_x, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int n = 0;
  if (cluster_x > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = cluster_x;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  if (pdl_enabled() && !pdl_off_for(tag)) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace tidal
