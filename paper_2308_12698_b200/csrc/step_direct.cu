// step_direct.cu -- the one-row-per-thread step kernels (K = 1, the rotor-lag
// and circle-feed variants, the TMA-staged variant): instantiation and launch
// (step_core.cuh has the kernels, step_launch.h the interface the C ABI calls).
#include <mutex>

#include "step_core.cuh"
#include "step_launch.h"

namespace {
inline unsigned grid_for(int64_t n, int block) { return (unsigned)((n + block - 1) / block); }

// TMA kernel launch configuration, per device and per variant
constexpr int kMaxDevices = 64;
struct TmaLaunchCfg {
    int blocks_per_sm, sm_count;
};
TmaLaunchCfg g_tma_cfg[kMaxDevices][2];
std::mutex g_tma_mu;

}  // namespace

namespace ssbl {

int launch_direct(const StepArgs &a, bool axi, const swarmstep_quad_params &P, const ssb::Derived &D, cudaStream_t s,
                  const Pdl &pdl)
{
    auto kern = axi ? (a.compensated ? quad_step_kernel<true, true> : quad_step_kernel<false, true>)
                    : (a.compensated ? quad_step_kernel<true, false> : quad_step_kernel<false, false>);
    return launch_step(kern, grid_for(a.n, kBlock), kBlock, s, pdl.tile_epoch != nullptr, "quad_step_kernel", a.cols,
                       a.flags, a.n, a.counters, a.fault_log, a.fault_cap, a.overlay, a.tick_base, a.tick_dev, P, D,
                       a.dt, a.k, pdl);
}

int launch_lag(const StepArgs &a, float *motor, float phi, float e_full, const swarmstep_quad_params &P,
               const ssb::Derived &D, cudaStream_t s)
{
    auto kern = a.compensated ? quad_step_lag_kernel<true> : quad_step_lag_kernel<false>;
    kern<<<grid_for(a.n, kBlock), kBlock, 0, s>>>(a.cols, a.flags, motor, a.n, a.counters, a.fault_log, a.fault_cap,
                                                  a.overlay, a.tick_base, a.tick_dev, P, D, phi, e_full, a.dt, a.k);
    return ssb::cuda_status("quad_step_lag_kernel");
}

int launch_circle(const StepArgs &a, const swarmstep_circle_feed &feed, const swarmstep_quad_params &P,
                  const ssb::Derived &D, cudaStream_t s, const Pdl &pdl)
{
    const bool axi = D.axisym != 0;
    auto kern = axi ? (a.compensated ? quad_step_circle_kernel<true, true> : quad_step_circle_kernel<false, true>)
                    : (a.compensated ? quad_step_circle_kernel<true, false> : quad_step_circle_kernel<false, false>);
    return launch_step(kern, grid_for(a.n, kBlock), kBlock, s, pdl.tile_epoch != nullptr, "quad_step_circle_kernel",
                       a.cols, a.flags, a.n, a.counters, a.fault_log, a.fault_cap, a.tick_base, a.tick_dev, P, D, feed,
                       circle_rot(feed.dt, feed.radius, feed.omega), a.dt, a.k, pdl);
}

int launch_tma(const StepArgs &a, int motor_possible, const swarmstep_quad_params &P, const ssb::Derived &D,
               cudaStream_t s)
{
    // the > 48 KB dynamic shared memory opt-in is per device and per
    // kernel: configure once per (device, variant), under a lock
    const size_t smem = sizeof(TmaSmem);
    auto kern = a.compensated ? quad_step_tma_kernel<true> : quad_step_tma_kernel<false>;
    const int ci = a.compensated ? 1 : 0;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return ssb::cuda_status("cudaGetDevice");
    if (dev < 0 || dev >= kMaxDevices) return ssb::set_err(SWARMSTEP_EINVAL, "device ordinal out of range");
    int blocks_per_sm = 0, sm_count = 0;
    {
        std::lock_guard<std::mutex> lock(g_tma_mu);
        TmaLaunchCfg &cfg = g_tma_cfg[dev][ci];
        if (!cfg.blocks_per_sm) {
            cudaDeviceGetAttribute(&cfg.sm_count, cudaDevAttrMultiProcessorCount, dev);
            if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
                return ssb::cuda_status("cudaFuncSetAttribute");
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cfg.blocks_per_sm, kern, SWARMSTEP_TILE, smem);
            if (cfg.blocks_per_sm < 1) cfg.blocks_per_sm = 1;
        }
        blocks_per_sm = cfg.blocks_per_sm;
        sm_count = cfg.sm_count;
    }
    const int64_t ntiles = (a.n + SWARMSTEP_TILE - 1) / SWARMSTEP_TILE;
    int64_t grid = (int64_t)sm_count * blocks_per_sm;
    if (grid > ntiles) grid = ntiles;
    kern<<<(unsigned)grid, SWARMSTEP_TILE, smem, s>>>(a.cols, a.flags, ntiles, a.counters, a.fault_log, a.fault_cap,
                                                      a.overlay, motor_possible, a.tick_base, a.tick_dev, P, D, a.dt,
                                                      a.k);
    return ssb::cuda_status("quad_step_tma_kernel");
}

int preload_direct()
{
    cudaFuncAttributes attr;
    const void *fns[] = {(const void *)quad_step_kernel<true, false>, (const void *)quad_step_kernel<false, false>,
                         (const void *)quad_step_kernel<true, true>, (const void *)quad_step_kernel<false, true>,
                         (const void *)quad_step_tma_kernel<true>, (const void *)quad_step_tma_kernel<false>,
                         (const void *)quad_step_lag_kernel<true>, (const void *)quad_step_lag_kernel<false>,
                         (const void *)quad_step_circle_kernel<true, false>,
                         (const void *)quad_step_circle_kernel<false, false>,
                         (const void *)quad_step_circle_kernel<true, true>,
                         (const void *)quad_step_circle_kernel<false, true>};
    for (const void *f : fns)
        if (cudaFuncGetAttributes(&attr, f) != cudaSuccess) return ssb::cuda_status("cudaFuncGetAttributes");
    return SWARMSTEP_OK;
}

}  // namespace ssbl
