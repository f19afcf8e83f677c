// step_pair.cu -- the paired FFMA2 step kernels (K >= 2 ticks per launch):
// instantiation and launch (step_core.cuh has the kernels, step_launch.h the
// interface the C ABI calls).
#include "step_core.cuh"
#include "step_launch.h"

namespace ssbl {

int launch_pair(const StepArgs &a, bool axi, const swarmstep_quad_params &P, const ssb::Derived &D, cudaStream_t s,
                const Pdl &pdl)
{
    auto kern = axi ? (a.compensated ? quad_step_pair_kernel<true, true> : quad_step_pair_kernel<false, true>)
                    : (a.compensated ? quad_step_pair_kernel<true, false> : quad_step_pair_kernel<false, false>);
    return launch_step(kern, (unsigned)((a.n + SWARMSTEP_TILE - 1) / SWARMSTEP_TILE), 64, s, pdl.tile_epoch != nullptr,
                       "quad_step_pair_kernel", a.cols, a.flags, a.n, a.counters, a.fault_log, a.fault_cap, a.overlay,
                       a.tick_base, a.tick_dev, P, D, a.dt, a.k, pdl);
}

int launch_pair_lag(const StepArgs &a, float *motor, float phi, float e_full, const swarmstep_quad_params &P,
                    const ssb::Derived &D, cudaStream_t s)
{
    auto kern = a.compensated ? quad_step_pair_lag_kernel<true> : quad_step_pair_lag_kernel<false>;
    kern<<<(unsigned)((a.n + SWARMSTEP_TILE - 1) / SWARMSTEP_TILE), 64, 0, s>>>(
        a.cols, a.flags, motor, a.n, a.counters, a.fault_log, a.fault_cap, a.overlay, a.tick_base, a.tick_dev, P, D,
        phi, e_full, a.dt, a.k);
    return ssb::cuda_status("quad_step_pair_lag_kernel");
}

int launch_pair_circle(const StepArgs &a, const swarmstep_circle_feed &feed, const swarmstep_quad_params &P,
                       const ssb::Derived &D, cudaStream_t s, const Pdl &pdl)
{
    const bool axi = D.axisym != 0;
    auto kern = axi ? (a.compensated ? quad_step_pair_circle_kernel<true, true> : quad_step_pair_circle_kernel<false, true>)
                    : (a.compensated ? quad_step_pair_circle_kernel<true, false>
                                     : quad_step_pair_circle_kernel<false, false>);
    return launch_step(kern, (unsigned)((a.n + SWARMSTEP_TILE - 1) / SWARMSTEP_TILE), 64, s, pdl.tile_epoch != nullptr,
                       "quad_step_pair_circle_kernel", a.cols, a.flags, a.n, a.counters, a.fault_log, a.fault_cap,
                       a.tick_base, a.tick_dev, P, D, feed, circle_rot(feed.dt, feed.radius, feed.omega), a.dt, a.k,
                       pdl);
}

int preload_pair()
{
    cudaFuncAttributes attr;
    const void *fns[] = {(const void *)quad_step_pair_kernel<true, false>, (const void *)quad_step_pair_kernel<false, false>,
                         (const void *)quad_step_pair_kernel<true, true>, (const void *)quad_step_pair_kernel<false, true>,
                         (const void *)quad_step_pair_lag_kernel<true>, (const void *)quad_step_pair_lag_kernel<false>,
                         (const void *)quad_step_pair_circle_kernel<true, false>,
                         (const void *)quad_step_pair_circle_kernel<false, false>,
                         (const void *)quad_step_pair_circle_kernel<true, true>,
                         (const void *)quad_step_pair_circle_kernel<false, true>};
    for (const void *f : fns)
        if (cudaFuncGetAttributes(&attr, f) != cudaSuccess) return ssb::cuda_status("cudaFuncGetAttributes");
    return SWARMSTEP_OK;
}

}  // namespace ssbl
