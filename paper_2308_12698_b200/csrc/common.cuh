// common.cuh -- error reporting shared by the C-ABI translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdio.h>

#include "swarmstep_b200.h"

namespace ssb {

// tiled SoA addressing (include/swarmstep_b200.h): element (c, r) lives at
// tile_base(r) + c * SWARMSTEP_TILE
__host__ __device__ __forceinline__ int64_t tile_base(int64_t r)
{
    return (r >> 7) * (int64_t)(SWARMSTEP_NCOL * SWARMSTEP_TILE) + (r & (SWARMSTEP_TILE - 1));
}

__host__ __device__ __forceinline__ int64_t at(int c, int64_t r)
{
    return tile_base(r) + (int64_t)c * SWARMSTEP_TILE;
}

// one thread-local message buffer for the whole library (C++17 inline)
inline char *err_buf()
{
    static thread_local char buf[512] = "";
    return buf;
}

inline int set_err(int code, const char *msg)
{
    snprintf(err_buf(), 512, "%s", msg);
    return code;
}

inline int cuda_status(const char *where)
{
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        snprintf(err_buf(), 512, "%s: %s", where, cudaGetErrorString(e));
        return SWARMSTEP_ECUDA;
    }
    return SWARMSTEP_OK;
}

}  // namespace ssb
