// launch.hpp — kernel launches with programmatic dependent launch (PDL).
//
// Every kernel of the decode chain is launched with
// cudaLaunchAttributeProgrammaticStreamSerialization: it may become resident
// while its predecessor is still running, executes `griddepcontrol.wait`
// (pdl_wait) before it touches anything a predecessor writes or reads, and
// signals `griddepcontrol.launch_dependents` (pdl_trigger) at its start so its
// own successor is scheduled as early as possible.  Inside the captured decode
// graph these become programmatic edges: a kernel's launch latency, prologue
// (barrier init, TMEM allocation, descriptor prefetch) and -- for the GEMMs --
// the first weight tiles of its stream overlap the predecessor's tail.
// srl_tuning.pdl = 0 launches everything with plain stream order.
#pragma once
#include <cuda_runtime.h>

#include <utility>

#include "tuning.hpp"

namespace srl {

inline bool pdl_enabled() { return tuning().pdl != 0; }

template <typename... Exp, typename... Act>
inline cudaError_t launch_k(void (*kern)(Exp...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, int cluster,
                            Act&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  unsigned n = 0;
  if (cluster > 1) {
    at[n].id = cudaLaunchAttributeClusterDimension;
    at[n].val.clusterDim.x = cluster;
    at[n].val.clusterDim.y = 1;
    at[n].val.clusterDim.z = 1;
    ++n;
  }
  if (pdl_enabled()) {
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.attrs = at;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Act>(args)...);
}

}  // namespace srl
