// step_launch.h -- internal: the step kernels' launchers, one translation unit
// per kernel family (step_pair.cu: the paired FFMA2 kernels; step_direct.cu:
// one row per thread, TMA-staged), called by the C ABI in swarmstep_b200.cu.
// Each returns an int status like the ABI.
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "swarmstep_b200.h"
#include "quad_math.cuh"

#ifndef SSB_PAIR_MIN_K
#define SSB_PAIR_MIN_K 2   // auto picks the paired (FFMA2) kernel from this many ticks per launch
#endif
#ifndef SSB_TMA_MAX_K
#define SSB_TMA_MAX_K 0   // auto never picks the TMA-staged kernel (measured slower)
#endif

namespace ssbl {

struct StepArgs {
    float *cols;
    uint8_t *flags;
    int64_t n;
    uint32_t *counters;
    uint64_t *fault_log;
    int64_t fault_cap;
    int overlay;
    uint32_t tick_base;
    const int64_t *tick_dev;
    float dt;
    int k;
    bool compensated;
};

// Overlapping back-to-back step launches (step_core.cuh pdl_enter / pdl_exit):
// per-tile epochs in device memory, the epoch this launch waits for (0: none)
// and the one it publishes.  tile_epoch == nullptr: a plain launch.
struct Pdl {
    uint32_t *tile_epoch;
    uint32_t wait, set;
};

// Per-launch constants of the fused circle feed's rotation (step_core.cuh
// circle_advance), computed once on the host in double precision.
struct CircleRot {
    float omc, sd, omc2, sd2;   // 1 - cos d, sin d, and the same for d / 2 (d = omega dt)
    float rs, nrs, rws;         // sign(omega) R, -sign(omega) R, sign(omega) R omega
};
inline CircleRot circle_rot(double dt, double radius, double omega)
{
    const double d = omega * dt, sg = copysign(1.0, omega);
    const double sh = sin(0.5 * d), sq = sin(0.25 * d);
    CircleRot r;
    r.omc = (float)(2.0 * sh * sh);        // 1 - cos d without cancellation
    r.sd = (float)sin(d);
    r.omc2 = (float)(2.0 * sq * sq);
    r.sd2 = (float)sh;
    r.rs = (float)(sg * radius);
    r.nrs = -r.rs;
    r.rws = (float)(sg * radius) * (float)omega;
    return r;
}

int launch_pair(const StepArgs &a, bool axi, const swarmstep_quad_params &P, const ssb::Derived &D, cudaStream_t s,
                const Pdl &pdl = Pdl{nullptr, 0, 0});
int launch_pair_lag(const StepArgs &a, float *motor, float phi, float e_full, const swarmstep_quad_params &P,
                    const ssb::Derived &D, cudaStream_t s);
int launch_pair_circle(const StepArgs &a, const swarmstep_circle_feed &feed, const swarmstep_quad_params &P,
                       const ssb::Derived &D, cudaStream_t s,
                       const Pdl &pdl = Pdl{nullptr, 0, 0});
int preload_pair();

int launch_direct(const StepArgs &a, bool axi, const swarmstep_quad_params &P, const ssb::Derived &D, cudaStream_t s,
                  const Pdl &pdl = Pdl{nullptr, 0, 0});
int launch_lag(const StepArgs &a, float *motor, float phi, float e_full, const swarmstep_quad_params &P,
               const ssb::Derived &D, cudaStream_t s);
int launch_circle(const StepArgs &a, const swarmstep_circle_feed &feed, const swarmstep_quad_params &P,
                  const ssb::Derived &D, cudaStream_t s,
                       const Pdl &pdl = Pdl{nullptr, 0, 0});
int launch_tma(const StepArgs &a, int motor_possible, const swarmstep_quad_params &P, const ssb::Derived &D,
               cudaStream_t s);
int preload_direct();

}  // namespace ssbl
