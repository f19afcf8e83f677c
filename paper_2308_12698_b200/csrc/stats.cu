// stats.cu -- swarm-wide reductions over one group's device state.
//
// The reference reduces over the whole swarm on the host every time a caller
// asks for alive counts (World.alive_counts, core.py:370; cli.py:161) or sizes
// the collision grid from the occupied extent (collision.py:124-128).  Here one
// launch reduces the tiled columns in place: alive count, position sum
// (centroid), sum and max of |v|^2, and the alive bounding box.
//
// Deterministic: every thread folds a fixed grid-stride set of rows in order,
// warps combine with a fixed shuffle butterfly, warps with a fixed shared-
// memory order, and the LAST block to finish (atomic ticket) folds the block
// partials in block-index order -- same bits on every run, one launch.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "common.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxBlocks = 148 * 4;

struct Acc {
    double alive, px, py, pz, v2;
    float v2max, lo[3], hi[3];
};

__device__ __forceinline__ void acc_init(Acc &a)
{
    a.alive = a.px = a.py = a.pz = a.v2 = 0.0;
    a.v2max = 0.0f;
    for (int i = 0; i < 3; i++) {
        a.lo[i] = INFINITY;
        a.hi[i] = -INFINITY;
    }
}

__device__ __forceinline__ void acc_merge(Acc &a, const Acc &b)
{
    a.alive += b.alive; a.px += b.px; a.py += b.py; a.pz += b.pz; a.v2 += b.v2;
    a.v2max = fmaxf(a.v2max, b.v2max);
    for (int i = 0; i < 3; i++) {
        a.lo[i] = fminf(a.lo[i], b.lo[i]);
        a.hi[i] = fmaxf(a.hi[i], b.hi[i]);
    }
}

__device__ __forceinline__ void acc_shfl(Acc &a, int o)
{
    Acc b;
    b.alive = __shfl_xor_sync(0xffffffffu, a.alive, o);
    b.px = __shfl_xor_sync(0xffffffffu, a.px, o);
    b.py = __shfl_xor_sync(0xffffffffu, a.py, o);
    b.pz = __shfl_xor_sync(0xffffffffu, a.pz, o);
    b.v2 = __shfl_xor_sync(0xffffffffu, a.v2, o);
    b.v2max = __shfl_xor_sync(0xffffffffu, a.v2max, o);
    for (int i = 0; i < 3; i++) {
        b.lo[i] = __shfl_xor_sync(0xffffffffu, a.lo[i], o);
        b.hi[i] = __shfl_xor_sync(0xffffffffu, a.hi[i], o);
    }
    acc_merge(a, b);
}

// another block's partial, read from L2 (written before its ticket increment)
__device__ __forceinline__ Acc load_cg(const Acc *p)
{
    Acc a;
    a.alive = __ldcg(&p->alive); a.px = __ldcg(&p->px); a.py = __ldcg(&p->py); a.pz = __ldcg(&p->pz);
    a.v2 = __ldcg(&p->v2); a.v2max = __ldcg(&p->v2max);
    for (int i = 0; i < 3; i++) {
        a.lo[i] = __ldcg(&p->lo[i]);
        a.hi[i] = __ldcg(&p->hi[i]);
    }
    return a;
}

// block-wide fixed-order reduction; the result is valid in thread 0
__device__ __forceinline__ void block_reduce(Acc &a, Acc *sh)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc_shfl(a, o);
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) sh[w] = a;
    __syncthreads();
    if (threadIdx.x == 0)
        for (int i = 1; i < kWarps; i++) acc_merge(a, sh[i]);
}

__global__ void __launch_bounds__(kThreads) swarm_stats_kernel(const float *cols, const uint8_t *flags, int64_t n,
                                                               int compensated, Acc *partials,
                                                               unsigned int *ticket, double *out)
{
    __shared__ Acc sh[kWarps];
    __shared__ bool last;
    Acc a;
    acc_init(a);
    for (int64_t r = (int64_t)blockIdx.x * kThreads + threadIdx.x; r < n; r += (int64_t)gridDim.x * kThreads) {
        if (!(flags[r] & SWARMSTEP_FLAG_ALIVE)) continue;
        double q[3];
        for (int i = 0; i < 3; i++) {
            q[i] = (double)cols[ssb::at(SWARMSTEP_COL_POS + i, r)];
            if (compensated) q[i] += (double)ssb::pos_lo(cols, r, i);
            a.lo[i] = fminf(a.lo[i], (float)q[i]);
            a.hi[i] = fmaxf(a.hi[i], (float)q[i]);
        }
        const float vx = cols[ssb::at(SWARMSTEP_COL_VEL + 0, r)], vy = cols[ssb::at(SWARMSTEP_COL_VEL + 1, r)];
        const float vz = cols[ssb::at(SWARMSTEP_COL_VEL + 2, r)];
        const float v2 = fmaf(vx, vx, fmaf(vy, vy, vz * vz));
        a.alive += 1.0;
        a.px += q[0]; a.py += q[1]; a.pz += q[2];
        a.v2 += (double)v2;
        a.v2max = fmaxf(a.v2max, v2);
    }
    block_reduce(a, sh);
    if (threadIdx.x == 0) {
        partials[blockIdx.x] = a;
        __threadfence();
        last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    // the last block folds the partials in block order (fixed shape)
    __threadfence();
    acc_init(a);
    for (int b = threadIdx.x; b < (int)gridDim.x; b += kThreads) acc_merge(a, load_cg(partials + b));
    __syncthreads();
    block_reduce(a, sh);
    if (threadIdx.x == 0) {
        out[0] = a.alive;
        out[1] = a.px; out[2] = a.py; out[3] = a.pz;
        out[4] = a.v2;
        out[5] = (double)a.v2max;
        for (int i = 0; i < 3; i++) {
            out[6 + i] = (double)a.lo[i];
            out[9 + i] = (double)a.hi[i];
        }
        *ticket = 0u;      // ready for the next launch (stream order)
    }
}

int blocks_for(int64_t n)
{
    const int64_t b = (n + kThreads - 1) / kThreads;
    return (int)(b < 1 ? 1 : (b > kMaxBlocks ? kMaxBlocks : b));
}

size_t ws_bytes() { return (size_t)kMaxBlocks * sizeof(Acc) + 256; }

}  // namespace

extern "C" {

int swarmstep_swarm_stats_workspace_bytes(uint64_t *bytes)
{
    if (!bytes) return ssb::set_err(SWARMSTEP_EINVAL, "null argument");
    *bytes = (uint64_t)ws_bytes();
    return SWARMSTEP_OK;
}

int swarmstep_quad_swarm_stats(const swarmstep_group_view *g, double *out12, void *workspace, uint64_t ws,
                               void *stream)
{
    if (!g || !g->cols || !g->flags || !out12 || !workspace) return ssb::set_err(SWARMSTEP_EINVAL, "null argument");
    if (ws < ws_bytes()) return ssb::set_err(SWARMSTEP_EINVAL, "workspace too small");
    if ((reinterpret_cast<uintptr_t>(workspace) & 15u) != 0)
        return ssb::set_err(SWARMSTEP_EINVAL, "workspace must be 16-byte aligned");
    // the ticket lives after the partials and must start (and is left) at 0:
    // callers zero the workspace once when they allocate it
    Acc *partials = (Acc *)workspace;
    unsigned int *ticket = (unsigned int *)((char *)workspace + (size_t)kMaxBlocks * sizeof(Acc));
    swarm_stats_kernel<<<blocks_for(g->n), kThreads, 0, (cudaStream_t)stream>>>(
        g->cols, g->flags, g->n, g->compensated, partials, ticket, out12);
    return ssb::cuda_status("swarm_stats_kernel");
}

}  // extern "C"
