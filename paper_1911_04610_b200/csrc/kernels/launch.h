// launch.h -- programmatic dependent launch (PDL) for every kernel of the hot path.
// Each kernel is launched with programmatic stream serialisation and calls pdl_wait() before
// it touches memory written by the previous kernel of its stream; its prologue (smem carve-up,
// mbarrier init, TMEM allocation) therefore overlaps the predecessor's tail.  pdl_trigger()
// lets the successor launch early.  Captured into CUDA graphs as programmatic edges.
#pragma once
#include <cuda_runtime.h>

#include <utility>

namespace xp {

__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
// griddepcontrol.wait blocks until the predecessor grid has COMPLETED and its memory is
// visible, so where the successor is allowed to launch (trigger) only decides how early its
// CTAs are scheduled, never what they read.  The elementwise/reduction kernels trigger right
// after their wait (measured: 1-stage pipeline +3 %, 4-stage equal); the GEMM keeps its late
// trigger (an early one parks 97 KB-smem CTAs on SMs other stages' GEMMs need: 4-stage -3 %).
#ifndef XP_NO_EARLY_TRIGGER
#define XP_EARLY_TRIGGER
#endif
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
#ifdef XP_EARLY_TRIGGER
  pdl_trigger();
#endif
}
__device__ __forceinline__ void pdl_wait_only() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace xp
