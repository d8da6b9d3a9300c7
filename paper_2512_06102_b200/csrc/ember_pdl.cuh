// Programmatic dependent launch (PDL) for chains of dependent launches on one stream (the C4
// forward t -> t+1 and backward t -> t-1, the halo-tiled work-list launches): each CTA lets the next
// launch start as soon as every CTA of this one is running, and waits for the previous launch
// (completion and memory visibility) before its first global access, so the next grid's CTAs fill
// the SMs the last wave frees instead of waiting for a launch after the grid drains.  A kernel
// launched without the attribute returns from the wait at once.
#pragma once
#include <cuda_runtime.h>

#ifndef EBL_PDL
#define EBL_PDL 1
#endif

namespace ebl {

__device__ __forceinline__ void pdl_enter() {
#if EBL_PDL
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
#if EBL_PDL
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
  return cudaLaunchKernelEx(&cfg, kern, args...);
#else
  kern<<<grid, block, smem, s>>>(args...);
  return cudaGetLastError();
#endif
}

}  // namespace ebl
