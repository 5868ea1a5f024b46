// Kernel launch with programmatic dependent launch (PDL): consecutive kernels of a forward overlap
// the next kernel's prologue (and the GEMMs' weight prefetch) with the previous kernel's tail.  Every
// kernel launched this way calls griddep_wait() before touching data produced on the stream.
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"

namespace dbl {

bool pdl_enabled();  // DBL_PDL=0 disables (A/B measurements)

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    CUDA_CHECK(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
    ++launch_counter();
}

}  // namespace dbl
