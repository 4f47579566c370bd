// launch.cuh — kernel launch with programmatic dependent launch (PDL).
//
// The BAPG iteration is a chain of dependent kernels on one stream (13 per
// iteration at c1).  Launched with the programmatic-serialization attribute,
// a kernel's CTAs are scheduled while its predecessor drains; each such
// kernel calls ptx::griddep_wait() before it reads anything the predecessor
// wrote, so results are unchanged and only the launch / prologue latency
// overlaps.  Captured into CUDA graphs as programmatic edges.
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>

namespace gwb {

// GWB_NO_PDL=1 launches everything fully serialised (A/B knob).
inline bool pdl_enabled() {
  static const bool on = std::getenv("GWB_NO_PDL") == nullptr;
  return on;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t stream, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

}  // namespace gwb
