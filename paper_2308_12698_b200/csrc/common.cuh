// common.cuh -- error reporting shared by the C-ABI translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
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

// Compensated position: the low parts of x, y, z packed into the one 32-bit
// word of column SWARMSTEP_COL_POS_LO (include/swarmstep_b200.h), 10 signed
// bits each in units of ulp(hi) / 512.  The unit is a power of two, so
// decoding is exact and encode(decode(w)) == w; encoding rounds lo to the
// nearest unit (error <= ulp(hi) / 1024, once per launch).
__device__ __forceinline__ float pos_lo_unit(float hi)        // ulp(hi) / 512 = 2^(e - 159)
{
    const uint32_t e = max((__float_as_uint(hi) >> 23) & 0xFFu, 33u);
    return __uint_as_float((e - 32u) << 23);
}
__device__ __forceinline__ float pos_lo_inv_unit(float hi)    // 512 / ulp(hi) = 2^(159 - e)
{
    const uint32_t e = max((__float_as_uint(hi) >> 23) & 0xFFu, 33u);
    return __uint_as_float((286u - e) << 23);
}
__device__ __forceinline__ float pos_lo_decode(uint32_t w, int i, float hi)
{
    const int q = (int)(w << (22 - 10 * i)) >> 22;            // sign-extended field i
    return (float)q * pos_lo_unit(hi);
}
__device__ __forceinline__ uint32_t pos_lo_field(float lo, int i, float hi)
{
    int q = __float2int_rn(lo * pos_lo_inv_unit(hi));
    q = min(max(q, -511), 511);
    return ((uint32_t)q & 0x3FFu) << (10 * i);
}
__device__ __forceinline__ uint32_t pos_lo_encode(const float lo[3], const float hi[3])
{
    return pos_lo_field(lo[0], 0, hi[0]) | pos_lo_field(lo[1], 1, hi[1]) | pos_lo_field(lo[2], 2, hi[2]);
}
// low part of row r, axis i, from the tiled columns
__device__ __forceinline__ float pos_lo(const float *cols, int64_t r, int i)
{
    return pos_lo_decode(__float_as_uint(cols[at(SWARMSTEP_COL_POS_LO, r)]), i, cols[at(SWARMSTEP_COL_POS + i, r)]);
}
// double-precision position of row r, axis i (hi + lo) from the tiled columns
__device__ __forceinline__ double pos_f64(const float *cols, int64_t r, int i, bool compensated)
{
    const float hi = cols[at(SWARMSTEP_COL_POS + i, r)];
    if (!compensated) return (double)hi;
    return (double)hi + (double)pos_lo(cols, r, i);
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
