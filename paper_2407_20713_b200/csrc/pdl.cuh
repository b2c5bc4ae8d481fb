// pdl.cuh — programmatic dependent launch for the per-step kernel chains
// (internal).  A kernel launched with launch_pdl may be scheduled while its
// stream predecessor still runs: everything before pdl_wait() (stream-
// independent set-up: table staging, the MC streams' jump-ahead) overlaps the
// predecessor, and pdl_wait() returns once the predecessor grid has completed
// and its memory is visible.  A predecessor that calls pdl_trigger() lets its
// dependent launch before it finishes (the small kernels do so at entry; the
// MC tile kernels never, so a waiting dependent cannot take their SM slots).
// In a grid launched without the attribute both instructions are no-ops.
#pragma once

#include <cstdlib>
#include <cuda_runtime.h>
#include <utility>

namespace sabr_gpu {

__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// SABR_T2_PDL=0 launches the T_II step chain without the attribute (A/B
// checks; read at every launch so one process can time both)
inline bool t2_pdl_enabled() {
    const char* e = std::getenv("SABR_T2_PDL");
    return !(e && std::atoi(e) == 0);
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = t2_pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
    return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace sabr_gpu
