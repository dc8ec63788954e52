// Programmatic dependent launch (PDL) for the factor path's kernels.
//
// Most launches of the upper levels are small, dependent and short: the gap
// between one kernel's end and the next one's first instruction (grid launch,
// CTA dispatch) is a visible share of the chain.  Kernels launched through
// launch_pdl() carry cudaLaunchAttributeProgrammaticStreamSerialization, so
// the next kernel in the stream is dispatched while its predecessor still
// runs; every such kernel starts with ACR_PDL_ENTRY(): griddepcontrol.wait
// (block until the predecessor grid has completed and its writes are
// visible) before touching any data, then griddepcontrol.launch_dependents
// (let the successor be dispatched).  Ordering is therefore exactly the
// stream order; only the launch latency overlaps.  ACR_NO_PDL=1 disables it.
#pragma once
#include <cuda_runtime.h>
#include <cstdlib>
#include <utility>

#define ACR_PDL_ENTRY()                                           \
  do {                                                            \
    asm volatile("griddepcontrol.wait;\n" ::: "memory");          \
    asm volatile("griddepcontrol.launch_dependents;\n" :::);      \
  } while (0)

// in launchers returning cudaError_t
#define CK_PDL(x)                       \
  do {                                  \
    cudaError_t e_pdl_ = (x);           \
    if (e_pdl_ != cudaSuccess) return e_pdl_; \
  } while (0)

namespace acr {

inline bool pdl_enabled() {
  static const bool on = getenv("ACR_NO_PDL") == nullptr;
  return on;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace acr
