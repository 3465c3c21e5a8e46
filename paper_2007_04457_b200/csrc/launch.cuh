// launch.cuh -- kernel launches with programmatic dependent launch (PDL).
//
// The hot kernels are launched with cudaLaunchAttributeProgrammaticStreamSerialization:
// each calls ptx::pdl_trigger() on entry and ptx::pdl_wait() before its first
// access to data of earlier launches, so the next kernel's CTAs are scheduled
// into the SMs the current one is draining and run their prologue (tables,
// barriers, descriptor fetches) under its tail; inside a CUDA graph the
// dependency becomes a programmatic edge (on small levels only, see pdl_for).
#pragma once

#include <cstdlib>
#include <utility>

#include "common.cuh"

namespace hgrb {

// PDL only pays on small levels, whose kernels are a few microseconds of
// launch-bound work; on the big ones the early-scheduled CTAs of the next kernel
// cost more than the gap they hide (A/B at 1025^3: +7 %). `level_nodes` is the
// node count of the level the launch works on (fine level for its coarse
// arrays); knob HGR_PDL_NODES (0 disables PDL).
inline bool pdl_for(int64_t level_nodes) {
  static const int64_t lim = [] {
    const char* v = std::getenv("HGR_PDL_NODES");
    return v ? int64_t(std::atoll(v)) : int64_t(1) << 20;
  }();
  return level_nodes < lim;
}

// Raise a kernel's dynamic shared-memory limit to at least `bytes` on the
// current device. Process-wide and only ever raised (under a mutex): a
// per-thread record could let one thread lower the limit below what another
// thread's later launch needs. (kernels_basic.cu)
void set_smem_attr(const void* fn, size_t bytes);

// throws with the kernel name and launch geometry in the message (kernels_basic.cu)
[[noreturn]] void launch_failed(cudaError_t e, const void* kern, dim3 grid, dim3 block, size_t smem);

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                int64_t level_nodes, Args&&... args) {
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_for(level_nodes) ? 1 : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
  if (e != cudaSuccess) launch_failed(e, reinterpret_cast<const void*>(kern), grid, block, smem);
}

}  // namespace hgrb
