// launch.cuh -- kernel launches with Programmatic Dependent Launch (PDL).
//
// Forward-path kernels are launched with programmatic stream serialisation: kernel N+1 is
// scheduled as soon as every CTA of kernel N has started (they all call pdl_trigger() first),
// runs its data-independent prologue (barrier init, TMEM allocation, descriptor prefetch) and
// blocks in pdl_wait() until kernel N has completed and flushed. Every kernel launched here
// must call pdl_wait() before its first global-memory access that depends on earlier work.
#pragma once
#include <cuda_runtime.h>

#include <utility>

#include "common.cuh"

namespace rs {

#ifdef __CUDACC__
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
#endif

template <class... KArgs, class... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = tuning().pdl >= 0 ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    RS_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

}  // namespace rs
