// Programmatic dependent launch (PDL) for every libgmi kernel.
//
// An iteration is ~10^2-10^3 short kernels in stream order, so the launch latency and the
// prologue (barrier init, TMEM allocation, tensor-map prefetch) of kernel i+1 would
// otherwise sit on the critical path after the tail of kernel i. Every kernel is launched
// with cudaLaunchAttributeProgrammaticStreamSerialization; each kernel calls
// pdl_trigger() early (lets the next grid be scheduled once all of this grid's CTAs have
// started) and pdl_wait() before it touches memory produced by earlier work in the stream
// (griddepcontrol.wait returns only after the preceding grid has completed and flushed).
// Every CTA of every kernel executes pdl_wait(), so completion of a grid still implies
// completion of everything before it in the stream.
#pragma once

#include <cuda_runtime.h>

#include <utility>

#include "../host/errors.hpp"

namespace gmi {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... Params, typename... Args>
void launch_pdl(void (*kernel)(Params...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  GMI_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

}  // namespace gmi
