// Programmatic dependent launch (PDL) helpers shared by the kernel files.
//
// A kernel launched with programmatic stream serialization may be scheduled
// while its predecessor on the stream drains. It must call pdl_wait() before
// it reads anything a predecessor wrote or writes anything global; pdl_wait()
// returns once the predecessor grid has completed and its writes are visible,
// so completion stays ordered along the stream. pdl_trigger() lets the next
// PDL kernel be scheduled. Launched without the attribute (GKB_NO_PDL=1, or a
// plain <<<>>> launch) both instructions are no-ops.
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>

namespace gkb {
namespace dev {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

inline bool pdl_enabled() {
  static const bool on = std::getenv("GKB_NO_PDL") == nullptr;
  return on;
}

template <class... KArgs, class... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t s, bool pdl, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = (pdl && pdl_enabled()) ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

}  // namespace dev
}  // namespace gkb
