// exchange.cu -- the config-5 position exchange fused into the pack kernel.
//
// NCCL all-gather baseline (parallel.py): pack the shard's positions into a
// local buffer, then ncclAllGather.  Here the pack kernel itself is the
// all-gather: every thread stores its agent's float4 straight into the
// gathered buffer of EVERY rank over NVLink (peer pointers of a symmetric
// allocation, torch.distributed._symmetric_memory), so the transfer overlaps
// the packing row by row and no separate collective launch or staging copy
// exists.  Completion is signalled per (writer, reader) pair:
//
//   pack_push (every rank)         wait (every rank)
//   stores -> fence.sys ->         spin until signal[w] >= E for every
//   arrive counter; the last       writer w (ld.acquire.sys), then
//   block st.release.sys E into    epoch := E
//   signal[rank] of every peer
//
// Buffers are double-buffered by epoch parity: a rank can be at most one
// epoch ahead of any peer (its wait needs the peer's signal of the same
// epoch), so slot E & 1 is never written while a peer still reads it.
// Readers pick the slot on the device from the epoch counter, so the whole
// chain is CUDA-graph capturable.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace {

__device__ __forceinline__ void st_release_sys(uint32_t *p, uint32_t v)
{
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t *p)
{
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__global__ void pack_push_kernel(const float *cols, const uint8_t *flags, int64_t n, int compensated,
                                 int64_t n_pad, int world, int rank, float4 *const *bufs,
                                 uint32_t *const *signals, const uint32_t *epoch, uint32_t *arrive)
{
    const uint32_t E = *epoch + 1u;
    const int64_t n_all = n_pad * world;
    const int64_t slot = (int64_t)(E & 1u) * n_all;
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n_pad) {
        const float nan = __int_as_float(0x7fc00000);
        float4 p = make_float4(nan, nan, nan, 0.0f);
        if (r < n && (flags[r] & SWARMSTEP_FLAG_ALIVE)) {
            float x = cols[ssb::at(SWARMSTEP_COL_POS + 0, r)];
            float y = cols[ssb::at(SWARMSTEP_COL_POS + 1, r)];
            float z = cols[ssb::at(SWARMSTEP_COL_POS + 2, r)];
            if (compensated) {
                x += ssb::pos_lo(cols, r, 0);
                y += ssb::pos_lo(cols, r, 1);
                z += ssb::pos_lo(cols, r, 2);
            }
            p = make_float4(x, y, z, 0.0f);
        }
        const int64_t dst = slot + (int64_t)rank * n_pad + r;
        for (int q = 0; q < world; q++) bufs[q][dst] = p;   // NVLink stores for q != rank
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        // gpu-scope fence + counter orders every block's stores before the
        // last block's; its system-scope fence + release stores extend that
        // order to the peers (causality order is transitive across scopes)
        __threadfence();
        if (atomicAdd(arrive, 1u) == gridDim.x - 1) {
            __threadfence_system();
            for (int q = 0; q < world; q++) st_release_sys(signals[q] + rank, E);
            *arrive = 0u;
        }
    }
}

__global__ void wait_kernel(const uint32_t *signals, int world, uint32_t *epoch)
{
    const uint32_t E = *epoch + 1u;
    for (int w = threadIdx.x; w < world; w += blockDim.x) {
        uint64_t t0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        while ((int32_t)(ld_acquire_sys(signals + w) - E) < 0) {
            uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > 10000000000ull) __trap();   // a peer never arrived (10 s): fail loudly, never hang
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) *epoch = E;
}

// Single-process variant (several devices, or several shards on one device):
// the pack is the all-gather -- every thread stores its row's float4 into
// every shard's gathered buffer (NVLink peer stores between devices with
// peer access enabled) -- and completion is ordered by CUDA events on the
// host side (each reader's stream waits for every writer's pack), so there
// are no device-side signals or spins.
__global__ void pack_scatter_kernel(const float *cols, const uint8_t *flags, int64_t n, int compensated,
                                    int64_t n_pad, int world, int rank, float4 *const *bufs, int64_t offset)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_pad) return;
    const float nan = __int_as_float(0x7fc00000);
    float4 p = make_float4(nan, nan, nan, 0.0f);
    if (r < n && (flags[r] & SWARMSTEP_FLAG_ALIVE)) {
        float x = cols[ssb::at(SWARMSTEP_COL_POS + 0, r)];
        float y = cols[ssb::at(SWARMSTEP_COL_POS + 1, r)];
        float z = cols[ssb::at(SWARMSTEP_COL_POS + 2, r)];
        if (compensated) {
            x += ssb::pos_lo(cols, r, 0);
            y += ssb::pos_lo(cols, r, 1);
            z += ssb::pos_lo(cols, r, 2);
        }
        p = make_float4(x, y, z, 0.0f);
    }
    const int64_t dst = offset + (int64_t)rank * n_pad + r;
    for (int q = 0; q < world; q++) bufs[q][dst] = p;
}

}  // namespace

extern "C" {

int swarmstep_pack_scatter(const swarmstep_group_view *g, void *const *bufs, int world, int rank, int64_t n_pad,
                           int64_t offset, void *stream)
{
    if (!g || !g->cols || !g->flags || !bufs) return ssb::set_err(SWARMSTEP_EINVAL, "null argument");
    if (world < 1 || rank < 0 || rank >= world) return ssb::set_err(SWARMSTEP_EINVAL, "bad world / rank");
    if (n_pad < g->n || offset < 0) return ssb::set_err(SWARMSTEP_EINVAL, "n_pad < n or negative offset");
    if (n_pad == 0) return SWARMSTEP_OK;
    pack_scatter_kernel<<<(unsigned)((n_pad + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        g->cols, g->flags, g->n, g->compensated, n_pad, world, rank, (float4 *const *)bufs, offset);
    return ssb::cuda_status("pack_scatter_kernel");
}

int swarmstep_enable_peer_access(int device, int peer)
{
    if (device == peer) return SWARMSTEP_OK;
    int can = 0;
    if (cudaDeviceCanAccessPeer(&can, device, peer) != cudaSuccess) return ssb::cuda_status("cudaDeviceCanAccessPeer");
    if (!can) return ssb::set_err(SWARMSTEP_ENODEV, "no peer access between these devices");
    int cur = 0;
    if (cudaGetDevice(&cur) != cudaSuccess) return ssb::cuda_status("cudaGetDevice");
    if (cudaSetDevice(device) != cudaSuccess) return ssb::cuda_status("cudaSetDevice");
    const cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
    cudaSetDevice(cur);
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();   // clear the (non-sticky) "already enabled" error
        return SWARMSTEP_OK;
    }
    if (e != cudaSuccess) return ssb::cuda_status("cudaDeviceEnablePeerAccess");
    return SWARMSTEP_OK;
}

int swarmstep_p2p_pack_push(const swarmstep_group_view *g, void *const *peer_bufs, int world, int rank,
                            int64_t n_pad, uint32_t *const *peer_signals, const uint32_t *epoch, uint32_t *arrive,
                            void *stream)
{
    if (!g || !g->cols || !g->flags || !peer_bufs || !peer_signals || !epoch || !arrive)
        return ssb::set_err(SWARMSTEP_EINVAL, "null argument");
    if (world < 1 || rank < 0 || rank >= world) return ssb::set_err(SWARMSTEP_EINVAL, "bad world / rank");
    if (n_pad < g->n) return ssb::set_err(SWARMSTEP_EINVAL, "n_pad < n");
    const int64_t blocks = n_pad > 0 ? (n_pad + 255) / 256 : 1;
    pack_push_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
        g->cols, g->flags, g->n, g->compensated, n_pad, world, rank, (float4 *const *)peer_bufs, peer_signals,
        epoch, arrive);
    return ssb::cuda_status("pack_push_kernel");
}

int swarmstep_p2p_wait(const uint32_t *local_signals, int world, uint32_t *epoch, void *stream)
{
    if (!local_signals || !epoch) return ssb::set_err(SWARMSTEP_EINVAL, "null argument");
    if (world < 1) return ssb::set_err(SWARMSTEP_EINVAL, "bad world");
    wait_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(local_signals, world, epoch);
    return ssb::cuda_status("wait_kernel");
}

}  // extern "C"
