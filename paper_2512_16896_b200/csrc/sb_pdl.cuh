// Programmatic dependent launch (PDL, sm_90+) for the engine's kernel chains.
//
// A kernel launched by launch_pdl() may have its CTAs scheduled while its predecessor on the
// stream is still draining its last wave. Every such kernel starts with pdl_enter(): it
// waits for the predecessor's completion and memory flush (griddepcontrol.wait; a no-op for
// a plain launch), which keeps stream order transitive along the chain, and then allows its
// own successor to launch. SB_PDL=0 launches plainly.
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>
#include <stdexcept>
#include <string>

namespace sbk {

__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

inline bool pdl_on() {
  static const bool on = [] {
    const char* e = std::getenv("SB_PDL");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*k)(KArgs...), unsigned grid, unsigned block, size_t smem,
                       cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_on() ? 1 : 0;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
  if (e != cudaSuccess) throw std::runtime_error(std::string("cudaLaunchKernelEx: ") + cudaGetErrorString(e));
}

}  // namespace sbk
