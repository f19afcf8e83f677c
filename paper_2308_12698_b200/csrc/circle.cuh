// circle.cuh -- the device circle strategy's per-row setpoint, shared by the
// standalone feed kernel (feed.cu) and the fused feed of the step kernels
// (swarmstep_b200.cu), so both produce identical bits.
//
// circle_reference (control.py:297-315) for phase `phase` (make_circle_layout,
// client.py:43-52): p = (R cos th, R sin th, z), v = (-R w sin th,
// R w cos th, 0), yaw = th + copysign(pi/2, w), th = w t + phase.
#pragma once
#include <math.h>
#include <stdint.h>

namespace ssb {

// x mod 2 pi in [0, 2 pi) for |x| < 2^40: Cody-Waite with a two-word 2 pi
// (the product k * 2pi_hi is exact for k < 2^19 ulps of slack), two FMAs
// instead of fmod's iterative reduction
__device__ __forceinline__ double reduce_2pi(double x)
{
    const double two_pi_hi = 6.283185307179586, two_pi_lo = 2.4492935982947064e-16;
    const double k = floor(x * 0.15915494309189535);
    return fma(-k, two_pi_lo, fma(-k, two_pi_hi, x));
}

// tick `tick` at step dt: vals = (p_sp xyz, v_sp xyz, yaw); the angle is
// formed and reduced in double (|w t| grows without bound; only cos / sin of
// the heading are used, control.py:259-260)
__device__ __forceinline__ void circle_values(int64_t tick, double dt, double radius, double omega, double z,
                                              double phase, float vals[7])
{
    const double t = (double)tick * dt;
    const double th_full = omega * t + phase;
    const double yaw = reduce_2pi(th_full + copysign(1.5707963267948966, omega));
    const double th = reduce_2pi(th_full);
    float s, c;
    sincosf((float)th, &s, &c);
    const float R = (float)radius, W = (float)omega;
    vals[0] = R * c;
    vals[1] = R * s;
    vals[2] = (float)z;
    vals[3] = -R * W * s;
    vals[4] = R * W * c;
    vals[5] = 0.0f;
    vals[6] = (float)yaw;
}

}  // namespace ssb
