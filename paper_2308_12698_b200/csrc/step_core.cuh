// step_core.cuh -- the step kernels' shared templates and the kernels
// themselves (included by step_pair.cu and step_direct.cu, each of which
// instantiates and launches its own kernels; csrc/step_launch.h).
//
// Hot path: quad_step_pair_kernel / quad_step_kernel = K fused
// QuadGroup.step(dt) calls (core.py:166-202) per launch, state
// register-resident across the K substeps.
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>

#include "swarmstep_b200.h"
#include "circle.cuh"
#include "common.cuh"
#include "quad_math.cuh"
#include "step_launch.h"

namespace {

#ifndef SSB_STEP_BLOCK
#define SSB_STEP_BLOCK 128
#endif
#ifndef SSB_STEP_MINB
#define SSB_STEP_MINB 6
#endif
// 128-thread CTAs, >= 6 resident per SM: caps the step kernel at 85
// registers (no spills with the tiled layout) for 24 warps per SM.
constexpr int kBlock = SSB_STEP_BLOCK;

// ---------------------------------------------------------------------------
// The fused step kernel.
// ---------------------------------------------------------------------------
#ifndef SSB_TICK_UNROLL
#define SSB_TICK_UNROLL 1
#endif
constexpr int kTickUnroll = SSB_TICK_UNROLL;

// One or two agents' registers for a launch (T = float or ssb::f2).
template <class T>
struct RowT {
    T p_hi[3], p_lo[3], v[3], q[4], w[3], integ[3], prev[3];
    // u[]: per-launch setpoint registers, shared by the three levels
    //   POS:   p_sp xyz, v_sp xyz (+ overlay on tick 0), cos(yaw), sin(yaw),
    //          cos(yaw/2), sin(yaw/2)
    //   MOTOR: rotor-model wrench f_c, tau xyz (core.py:189-197)
    T u[10];
    T w_sp[3], f_sp;   // inner-loop setpoints (stale ones for MOTOR rows)
};
using Row = RowT<float>;

// one lane of a paired row
__device__ __forceinline__ Row lane_row(const RowT<ssb::f2> &R, int i)
{
    Row o;
#pragma unroll
    for (int k = 0; k < 3; k++) {
        o.p_hi[k] = ssb::lane(R.p_hi[k], i); o.p_lo[k] = ssb::lane(R.p_lo[k], i); o.v[k] = ssb::lane(R.v[k], i);
        o.w[k] = ssb::lane(R.w[k], i); o.integ[k] = ssb::lane(R.integ[k], i); o.prev[k] = ssb::lane(R.prev[k], i);
        o.w_sp[k] = ssb::lane(R.w_sp[k], i);
    }
#pragma unroll
    for (int k = 0; k < 4; k++) o.q[k] = ssb::lane(R.q[k], i);
#pragma unroll
    for (int k = 0; k < 10; k++) o.u[k] = ssb::lane(R.u[k], i);
    o.f_sp = ssb::lane(R.f_sp, i);
    return o;
}

// Row accessors: the same step code reads a row from global memory (direct
// kernels, streaming loads) or from a shared-memory tile staged by TMA.
struct GlobalRow {
    float *p;
    __device__ __forceinline__ float ld(int c) const { return __ldcs(p + c * SWARMSTEP_TILE); }
    __device__ __forceinline__ float ldc(int c) const { return __ldg(p + c * SWARMSTEP_TILE); }
    __device__ __forceinline__ void st(int c, float v) const { __stcs(p + c * SWARMSTEP_TILE, v); }
};
struct SmemRow {
    float *p;
    __device__ __forceinline__ float ld(int c) const { return p[c * SWARMSTEP_TILE]; }
    __device__ __forceinline__ float ldc(int c) const { return p[c * SWARMSTEP_TILE]; }
    __device__ __forceinline__ void st(int c, float v) const { p[c * SWARMSTEP_TILE] = v; }
};
// Two rows read / written as one f2 lane pair (the paired kernel).
template <class A>
struct PairRow {
    A a, b;
    __device__ __forceinline__ ssb::f2 ld(int c) const { return ssb::f2{make_float2(a.ld(c), b.ld(c))}; }
    __device__ __forceinline__ ssb::f2 ldc(int c) const { return ssb::f2{make_float2(a.ldc(c), b.ldc(c))}; }
    __device__ __forceinline__ void st(int c, ssb::f2 v) const { a.st(c, v.v.x); b.st(c, v.v.y); }
};

// Two adjacent rows (2t, 2t + 1) of one tile as one f2 lane pair: every
// column is one 8-byte access per thread, so a warp moves 256 contiguous
// bytes per column with one LDG.64 / STG.64 (half the memory instructions of
// two separate rows) and the lanes land directly in the FFMA2 register pair.
struct VecPairRow {
    float *p;     // row 2t, column 0 (8-byte aligned: tiles are 512 B per column)
    __device__ __forceinline__ ssb::f2 ld(int c) const
    {
        return ssb::f2{__ldcs(reinterpret_cast<const float2 *>(p + c * SWARMSTEP_TILE))};
    }
    __device__ __forceinline__ ssb::f2 ldc(int c) const
    {
        return ssb::f2{__ldg(reinterpret_cast<const float2 *>(p + c * SWARMSTEP_TILE))};
    }
    __device__ __forceinline__ void st(int c, ssb::f2 v) const
    {
        __stcs(reinterpret_cast<float2 *>(p + c * SWARMSTEP_TILE), v.v);
    }
};

template <class T> __device__ __forceinline__ T zero_t() { return ssb::bc<T>(0.0f); }

// Motor-lag policy of a launch.  NoLag: the reference's instantaneous mixer
// (every hot kernel).  MotorLag: the opt-in first-order rotor lag
// (quad_math.cuh), scalar rows only; the four rotor thrusts live in their own
// tiled array (4 columns x 128 rows per tile) next to the state.
// AXI: the inertia is axisymmetric (I_xx == I_yy, e.g. the default X quad):
// the yaw gyroscopic coefficient (I_yy - I_xx) / I_zz is exactly 0 and the
// derivative skips that term (deriv<AXI>).
template <bool AXI>
struct NoLagT {
    static constexpr bool lag_on = false, feed_on = false, axisym = AXI;
    template <class T> __device__ __forceinline__ void feed(int, RowT<T> &) const {}
    template <class A> __device__ __forceinline__ void store_cmd(const A &, int) const {}
    __device__ __forceinline__ void load() {}
    __device__ __forceinline__ void store() const {}
};
using NoLag = NoLagT<false>;

struct MotorLag {
    static constexpr bool lag_on = true, feed_on = false, axisym = false;
    template <class T> __device__ __forceinline__ void feed(int, RowT<T> &) const {}
    template <class A> __device__ __forceinline__ void store_cmd(const A &, int) const {}
    float *p;          // this row's rotor-thrust column 0 (column i at p + 128 i)
    float phi, e_full;      // (tau_m / dt)(1 - e^(-dt / tau_m)), e^(-dt / tau_m)
    float f[4];
    __device__ __forceinline__ void load()
    {
#pragma unroll
        for (int i = 0; i < 4; i++) f[i] = p[i * SWARMSTEP_TILE];
    }
    __device__ __forceinline__ void store() const
    {
#pragma unroll
        for (int i = 0; i < 4; i++) p[i * SWARMSTEP_TILE] = f[i];
    }
};

// Two rows' rotor thrusts as one f2 lane pair (the paired kernel).
struct MotorLagPair {
    static constexpr bool lag_on = true, feed_on = false, axisym = false;
    template <class T> __device__ __forceinline__ void feed(int, RowT<T> &) const {}
    template <class A> __device__ __forceinline__ void store_cmd(const A &, int) const {}
    float *p0, *p1;          // rows 2t and 2t + 1 of one tile (column i at + 128 i)
    float phi, e_full;
    ssb::f2 f[4];
    __device__ __forceinline__ void load()
    {
#pragma unroll
        for (int i = 0; i < 4; i++) f[i] = ssb::f2{make_float2(p0[i * SWARMSTEP_TILE], p1[i * SWARMSTEP_TILE])};
    }
    __device__ __forceinline__ void store() const
    {
#pragma unroll
        for (int i = 0; i < 4; i++) {
            p0[i * SWARMSTEP_TILE] = f[i].v.x;
            p1[i * SWARMSTEP_TILE] = f[i].v.y;
        }
    }
};

// In-kernel circle feed (the circle strategy of feed.cu evaluated per tick
// inside the step, so K ticks of a time-varying reference fuse into one
// launch).  Tick 0 of a launch uses circle_reference at t = tick0 dt with this
// row's phase, computed exactly as circle_kernel computes it; ticks 1..K-1
// advance the setpoint by rotation: the angle th grows by delta = omega dt per
// tick, so (cos yaw, sin yaw) turns by delta and (cos yaw/2, sin yaw/2) by
// delta / 2 (yaw = th + sign(omega) pi/2, control.py:297-315), each a
// compensated rotation c' = c - (c (1 - cos d) + s sin d) (four FP32 ops, paired
// in the FFMA2 kernel) instead of a double-precision angle reduction and two
// sincos per tick; p and v follow from (cos yaw, sin yaw) with three products.
// One launch of K ticks agrees with K x (circle_kernel + 1-tick step) to the
// rotation's rounding (~1e-7 relative over 25 ticks; a one-tick launch is
// bit-identical), and the command columns it leaves are tick K-1's exact values.
// (c, s) turned by the angle with 1 - cos = omc, sin = sd
template <class T>
__device__ __forceinline__ void rotate_cs(T &c, T &s, T omc, T sd)
{
    const T dc = ssb::fma(c, omc, ssb::mul(s, sd));
    const T ds = ssb::fnma(c, sd, ssb::mul(s, omc));
    c = ssb::sub(c, dc);
    s = ssb::sub(s, ds);
}
// tick k >= 1 of a fused circle launch: u[0..9] of tick k-1 advanced by one tick
template <class T>
__device__ __forceinline__ void circle_advance(RowT<T> &R, const ssbl::CircleRot &r)
{
    using ssb::bc;
    rotate_cs(R.u[6], R.u[7], bc<T>(r.omc), bc<T>(r.sd));
    rotate_cs(R.u[8], R.u[9], bc<T>(r.omc2), bc<T>(r.sd2));
    // th = yaw - sign pi/2: (cos th, sin th) = sign (sin yaw, -cos yaw)
    R.u[0] = ssb::mul(bc<T>(r.rs), R.u[7]);
    R.u[1] = ssb::mul(bc<T>(r.nrs), R.u[6]);
    R.u[3] = ssb::mul(bc<T>(r.rws), R.u[6]);
    R.u[4] = ssb::mul(bc<T>(r.rws), R.u[7]);
}

template <bool AXI>
struct CircleFeedRowT {
    static constexpr bool lag_on = false, feed_on = true, axisym = AXI;
    int64_t tick0;
    double dt, radius, omega, z, phase;
    ssbl::CircleRot rot;
    __device__ __forceinline__ void load() {}
    __device__ __forceinline__ void store() const {}
    __device__ __forceinline__ void values(int k, float vals[7]) const
    {
        ssb::circle_values(tick0 + k, dt, radius, omega, z, phase, vals);
    }
    __device__ __forceinline__ void feed(int k, RowT<float> &R) const
    {
        if (k > 0) {
            circle_advance(R, rot);
            return;
        }
        float v[7];
        values(0, v);
#pragma unroll
        for (int i = 0; i < 6; i++) R.u[i] = v[i];
        ssb::yaw_terms(v[6], R.u[6], R.u[7], R.u[8], R.u[9]);
    }
    // the command columns the unfused feed would have left: tick k's values
    template <class A> __device__ __forceinline__ void store_cmd(const A &C, int k) const
    {
        float v[7];
        values(k, v);
#pragma unroll
        for (int i = 0; i < 7; i++) C.st(SWARMSTEP_COL_CMD + i, v[i]);
    }
};

// Two rows' circle feeds as one f2 lane pair (the paired kernel).
template <bool AXI>
struct CircleFeedPairT {
    static constexpr bool lag_on = false, feed_on = true, axisym = AXI;
    CircleFeedRowT<AXI> a, b;
    __device__ __forceinline__ void load() {}
    __device__ __forceinline__ void store() const {}
    __device__ __forceinline__ void feed(int k, RowT<ssb::f2> &R) const
    {
        if (k > 0) {
            circle_advance(R, a.rot);     // the rotation is the same for every row
            return;
        }
        float va[7], vb[7];
        a.values(0, va);
        b.values(0, vb);
#pragma unroll
        for (int i = 0; i < 6; i++) R.u[i] = ssb::f2{make_float2(va[i], vb[i])};
        float ca, sa, cha, sha, cb, sb, chb, shb;
        ssb::yaw_terms(va[6], ca, sa, cha, sha);
        ssb::yaw_terms(vb[6], cb, sb, chb, shb);
        R.u[6] = ssb::f2{make_float2(ca, cb)};
        R.u[7] = ssb::f2{make_float2(sa, sb)};
        R.u[8] = ssb::f2{make_float2(cha, chb)};
        R.u[9] = ssb::f2{make_float2(sha, shb)};
    }
    template <class A> __device__ __forceinline__ void store_cmd(const A &C, int k) const
    {
        float va[7], vb[7];
        a.values(k, va);
        b.values(k, vb);
#pragma unroll
        for (int i = 0; i < 7; i++) C.st(SWARMSTEP_COL_CMD + i, ssb::f2{make_float2(va[i], vb[i])});
    }
};

// packed compensated-position word <-> three float low parts (common.cuh)
__device__ __forceinline__ void decode_lo(float w, const float hi[3], float lo[3])
{
#pragma unroll
    for (int i = 0; i < 3; i++) lo[i] = ssb::pos_lo_decode(__float_as_uint(w), i, hi[i]);
}
__device__ __forceinline__ void decode_lo(ssb::f2 w, const ssb::f2 hi[3], ssb::f2 lo[3])
{
#pragma unroll
    for (int i = 0; i < 3; i++)
        lo[i] = ssb::f2{make_float2(ssb::pos_lo_decode(__float_as_uint(w.v.x), i, hi[i].v.x),
                                    ssb::pos_lo_decode(__float_as_uint(w.v.y), i, hi[i].v.y))};
}
__device__ __forceinline__ float encode_lo(const float hi[3], const float lo[3])
{
    return __uint_as_float(ssb::pos_lo_encode(lo, hi));
}
__device__ __forceinline__ ssb::f2 encode_lo(const ssb::f2 hi[3], const ssb::f2 lo[3])
{
    const float ha[3] = {hi[0].v.x, hi[1].v.x, hi[2].v.x}, la[3] = {lo[0].v.x, lo[1].v.x, lo[2].v.x};
    const float hb[3] = {hi[0].v.y, hi[1].v.y, hi[2].v.y}, lb[3] = {lo[0].v.y, lo[1].v.y, lo[2].v.y};
    return ssb::f2{make_float2(__uint_as_float(ssb::pos_lo_encode(la, ha)), __uint_as_float(ssb::pos_lo_encode(lb, hb)))};
}

template <bool COMP, class T, class A>
__device__ __forceinline__ void load_state(const A &C, RowT<T> &R)
{
#pragma unroll
    for (int i = 0; i < 3; i++) {
        R.p_hi[i] = C.ld(SWARMSTEP_COL_POS + i);
        R.v[i] = C.ld(SWARMSTEP_COL_VEL + i);
        R.w[i] = C.ld(SWARMSTEP_COL_OMEGA + i);
        R.integ[i] = C.ld(SWARMSTEP_COL_INTEGRAL + i);
        R.prev[i] = C.ld(SWARMSTEP_COL_PREV + i);
    }
    if (COMP) {
        decode_lo(C.ld(SWARMSTEP_COL_POS_LO), R.p_hi, R.p_lo);
    } else {
#pragma unroll
        for (int i = 0; i < 3; i++) R.p_lo[i] = zero_t<T>();
    }
#pragma unroll
    for (int i = 0; i < 4; i++) R.q[i] = C.ld(SWARMSTEP_COL_QUAT + i);
#pragma unroll
    for (int i = 0; i < 7; i++) R.u[i] = C.ld(SWARMSTEP_COL_CMD + i);
    R.u[7] = R.u[8] = R.u[9] = zero_t<T>();
}

template <bool COMP, class T, class A>
__device__ __forceinline__ void store_state(const A &C, int level, RowT<T> &R)
{
    // the launch-local position accumulator back into (hi, lo) (rk4_inplace ACC)
    if (COMP) ssb::fold_position(R.p_hi, R.p_lo);
#pragma unroll
    for (int i = 0; i < 3; i++) {
        C.st(SWARMSTEP_COL_POS + i, R.p_hi[i]);
        C.st(SWARMSTEP_COL_VEL + i, R.v[i]);
        C.st(SWARMSTEP_COL_OMEGA + i, R.w[i]);
        C.st(SWARMSTEP_COL_INTEGRAL + i, R.integ[i]);
        C.st(SWARMSTEP_COL_PREV + i, R.prev[i]);
    }
    if (COMP) C.st(SWARMSTEP_COL_POS_LO, encode_lo(R.p_hi, R.p_lo));
#pragma unroll
    for (int i = 0; i < 4; i++) C.st(SWARMSTEP_COL_QUAT + i, R.q[i]);
    if (level != SWARMSTEP_LEVEL_MOTOR) {
        // the last tick's setpoints become the stale setpoints a later MOTOR
        // command runs the PID on (core.py:178-182)
#pragma unroll
        for (int i = 0; i < 3; i++) C.st(SWARMSTEP_COL_SP + i, R.w_sp[i]);
        C.st(SWARMSTEP_COL_SP + 3, R.f_sp);
    }
}

__device__ __forceinline__ void yaw_lane(float yaw, float &c, float &s, float &ch, float &sh)
{
    ssb::yaw_terms(yaw, c, s, ch, sh);
}
__device__ __forceinline__ void yaw_lane(ssb::f2 yaw, ssb::f2 &c, ssb::f2 &s, ssb::f2 &ch, ssb::f2 &sh)
{
    ssb::yaw_terms(yaw.v.x, c.v.x, s.v.x, ch.v.x, sh.v.x);
    ssb::yaw_terms(yaw.v.y, c.v.y, s.v.y, ch.v.y, sh.v.y);
}

// Per-launch setpoint preparation (commands are fixed across the K ticks).
// has_prev: per-row "previous rate sample exists" (control.py:104).
template <class L = NoLag, class T, class A, class M>
__device__ __forceinline__ void setup_level(const A &C, int level, int overlay_active,
                                            const swarmstep_quad_params &P, M has_prev, RowT<T> &R)
{
    // first sample: no D term (control.py:175-177) <=> prev := w
#pragma unroll
    for (int i = 0; i < 3; i++) R.prev[i] = ssb::sel(has_prev, R.prev[i], R.w[i]);
    R.w_sp[0] = R.w_sp[1] = R.w_sp[2] = R.f_sp = zero_t<T>();
    if (level == SWARMSTEP_LEVEL_POS) {
        T s, c, sh, ch;
        yaw_lane(R.u[6], c, s, ch, sh);
        R.u[6] = c;
        R.u[7] = s;
        R.u[8] = ch;
        R.u[9] = sh;
        if (overlay_active) {
#pragma unroll
            for (int i = 0; i < 3; i++) R.u[3 + i] = ssb::add(R.u[3 + i], C.ldc(SWARMSTEP_COL_OVERLAY + i));
        }
    } else if (level == SWARMSTEP_LEVEL_RATE) {
        R.w_sp[0] = R.u[0]; R.w_sp[1] = R.u[1]; R.w_sp[2] = R.u[2]; R.f_sp = R.u[3];
    } else if constexpr (sizeof(T) == sizeof(float)) {
        // MOTOR (scalar rows only): the PID still runs on the stale setpoints
        // (core.py:109-110, 184-186); the integrated wrench comes from the
        // rotor model
#pragma unroll
        for (int i = 0; i < 3; i++) R.w_sp[i] = C.ldc(SWARMSTEP_COL_SP + i);
        R.f_sp = C.ldc(SWARMSTEP_COL_SP + 3);
        if constexpr (L::lag_on) {
            // lagged: the commanded rotor thrusts k_t clip(rpm)^2 (quad.py:134-137)
#pragma unroll
            for (int i = 0; i < 4; i++) {
                const float c = ssb::clip(R.u[i], 0.0f, P.omega_max);
                R.u[i] = P.k_t * (c * c);
            }
        } else {
            float mt[3], mf;
            ssb::motor_wrench(R.u, P, mf, mt);
            R.u[0] = mf; R.u[1] = mt[0]; R.u[2] = mt[1]; R.u[3] = mt[2];
        }
    }
}

// A non-finite position / velocity / quaternion / rate is absorbing: NaN and
// inf survive every later tick's arithmetic (a zero quaternion norm turns
// into NaN at the next renormalisation), so "some tick faulted" is exactly
// "the final state is non-finite" and the fast pass tests once per launch.
template <bool COMP, class T>
__device__ __forceinline__ ssb::mask_t<T> state_finite(const RowT<T> &R)
{
    using namespace ssb;
    T s = add(add(add(R.p_hi[0], R.p_hi[1]), add(R.p_hi[2], R.v[0])), add(add(R.v[1], R.v[2]), add(R.w[0], R.w[1])));
    s = add(s, add(R.w[2], add(add(R.q[0], R.q[1]), add(R.q[2], R.q[3]))));
    if (COMP) s = add(s, add(add(R.p_lo[0], R.p_lo[1]), R.p_lo[2]));
    return eq(mul(bc<T>(0.0f), s), bc<T>(0.0f));
}

// K ticks at a fixed command level (the body of QuadGroup.step, core.py:
// 166-202, repeated), state updated in place.  Passes:
//  * fast (default): no per-tick fault test; returns K if the state is
//    non-finite after the last tick (some tick faulted), else -1;
//  * CHECK: the reference's per-tick fault predicate (quad.py:404-430);
//    returns the first tick at which a lane faulted (registers then garbage);
//  * RERUN: stops after the controller part of tick pid_only_at (rebuilds a
//    faulted row's state, see step_row).
// All three execute identical arithmetic per tick, so they agree bit for bit.
template <int LEVEL, bool COMP, bool RERUN, bool CHECK, class T, class L>
__device__ __forceinline__ int run_ticks(const swarmstep_quad_params &P, const ssb::Derived &D,
                                         float dt, int K, int pid_only_at, RowT<T> &R, L &lag)
{
#pragma unroll kTickUnroll
    for (int k = 0; k < K; k++) {
        T S[3];                 // thrust terms of the tick's quaternion (POS: from the outer loop)
        const T *S1 = LEVEL == SWARMSTEP_LEVEL_POS ? S : nullptr;
        if (LEVEL == SWARMSTEP_LEVEL_POS) {
            if constexpr (L::feed_on) lag.feed(k, R);
            const T *u = R.u;
            T p_err[3];
#pragma unroll
            for (int i = 0; i < 3; i++) p_err[i] = ssb::sub(ssb::sub(u[i], R.p_hi[i]), R.p_lo[i]);
            ssb::outer_row<L::axisym>(p_err, R.v, R.q, u + 3, u[6], u[7], u[8], u[9], P, D, R.w_sp, R.f_sp, S);
        }
        T tau[3], f_c = R.f_sp;
        ssb::pid_row<L::axisym>(R.w, R.w_sp, P, D, dt, R.integ, R.prev, tau);
        if (RERUN && k == pid_only_at) return -1;
        if constexpr (L::lag_on) {
            // commanded rotor thrusts u; the body integrates the wrench of the
            // tick-mean lagged thrust, the rotors end the tick lagged by e_full
            T u[4], fbar[4];
            if (LEVEL == SWARMSTEP_LEVEL_MOTOR) {
#pragma unroll
                for (int i = 0; i < 4; i++) u[i] = R.u[i];
            } else {
                ssb::mix_motors(f_c, tau, P, D, u);
            }
            ssb::lag_thrust(lag.f, u, ssb::bc<T>(lag.phi), fbar);
            ssb::thrust_wrench(fbar, P, f_c, tau);
            const auto ok = ssb::rk4_inplace<T, COMP, true, L::axisym>(R.p_hi, R.p_lo, R.v, R.q, R.w, f_c, tau, P, D, dt, S1);
            if (CHECK && ssb::any(ssb::mnot(ok))) return k;
            ssb::lag_thrust(lag.f, u, ssb::bc<T>(lag.e_full), lag.f);
        } else {
            if (LEVEL == SWARMSTEP_LEVEL_MOTOR) {
                f_c = R.u[0]; tau[0] = R.u[1]; tau[1] = R.u[2]; tau[2] = R.u[3];
            } else {
                ssb::mix_row(f_c, tau, P, D);
            }
            const auto ok = ssb::rk4_inplace<T, COMP, true, L::axisym>(R.p_hi, R.p_lo, R.v, R.q, R.w, f_c, tau, P, D, dt, S1);
            if (CHECK && ssb::any(ssb::mnot(ok))) return k;
        }
    }
    if (!CHECK && !RERUN && ssb::any(ssb::mnot(state_finite<COMP>(R)))) return K;
    return -1;
}

template <bool COMP, bool RERUN, bool CHECK, class T, class A, class L>
__device__ __forceinline__ int run_level(const A &C, int level, int overlay_active,
                                         const swarmstep_quad_params &P, const ssb::Derived &D,
                                         float dt, int K, int pid_only_at, RowT<T> &R, L &lag)
{
    // level-specialised tick loops: no per-tick level branches
    if (level == SWARMSTEP_LEVEL_POS) {
        if (!overlay_active)
            return run_ticks<SWARMSTEP_LEVEL_POS, COMP, RERUN, CHECK>(P, D, dt, K, pid_only_at, R, lag);
        // tick 0 sees v_sp + overlay (setup_level added it); the overlay lasts
        // one tick (core.py:172-175, 199-201), so tick 0 is peeled off
        int f = run_ticks<SWARMSTEP_LEVEL_POS, COMP, RERUN, CHECK>(P, D, dt, 1, pid_only_at, R, lag);
        if (f >= 0 || K == 1 || (RERUN && pid_only_at == 0)) return f;
#pragma unroll
        for (int i = 0; i < 3; i++) R.u[3 + i] = C.ldc(SWARMSTEP_COL_CMD + 3 + i);
        f = run_ticks<SWARMSTEP_LEVEL_POS, COMP, RERUN, CHECK>(P, D, dt, K - 1, pid_only_at - 1, R, lag);
        return f >= 0 ? f + 1 : -1;
    }
    if (level == SWARMSTEP_LEVEL_RATE)
        return run_ticks<SWARMSTEP_LEVEL_RATE, COMP, RERUN, CHECK>(P, D, dt, K, pid_only_at, R, lag);
    if constexpr (sizeof(T) == sizeof(float))
        return run_ticks<SWARMSTEP_LEVEL_MOTOR, COMP, RERUN, CHECK>(P, D, dt, K, pid_only_at, R, lag);
    return -1;
}

// The whole per-row launch: K ticks from the row's inputs behind accessor C,
// outputs back through C; returns the new flag byte.  A fault at tick f
// leaves the row at its pre-tick values, dead, and logged with its tick
// (quad.py:425-436).  State is updated in place, so a faulted row is rebuilt
// by re-running ticks [0, f) from the launch's inputs -- bit-identical by
// determinism -- plus the controller part of tick f (the reference updates
// the PID state before rk4_step faults the row).  Inputs must still be
// readable through C at that point (global memory, or the staged tile).
template <bool COMP, class A, class L = NoLag>
__device__ __forceinline__ uint8_t step_row(const A &C, uint8_t fl, int64_t r, int overlay_active,
                                            const swarmstep_quad_params &P, const ssb::Derived &D, float dt, int K,
                                            uint32_t tick_base, const int64_t *tick_dev,
                                            uint32_t *counters, uint64_t *fault_log, int64_t fault_cap,
                                            Row &R, bool preloaded = false, L lag = L())
{
    if (!preloaded) load_state<COMP>(C, R);
    lag.load();
    // the circle feed puts every alive row at POS level (feed.cu)
    const int level = L::feed_on ? SWARMSTEP_LEVEL_POS : (fl & SWARMSTEP_LEVEL_MASK) >> SWARMSTEP_LEVEL_SHIFT;
    const bool has_prev = (fl & SWARMSTEP_FLAG_HAS_PREV) != 0;
    setup_level<L>(C, level, overlay_active, P, has_prev, R);
    int fault_k = run_level<COMP, false, false>(C, level, overlay_active, P, D, dt, K, -1, R, lag);
    bool alive = true;
    if (fault_k >= 0) {
        // the row faulted somewhere in the launch: find the tick with the
        // per-tick predicate (re-executing from the launch inputs) ...
        load_state<COMP>(C, R);
        lag.load();
        setup_level<L>(C, level, overlay_active, P, has_prev, R);
        fault_k = run_level<COMP, false, true>(C, level, overlay_active, P, D, dt, K, -1, R, lag);
    }
    if (fault_k >= 0) {
        // ... then rebuild its state at that tick
        alive = false;
        load_state<COMP>(C, R);
        lag.load();
        setup_level<L>(C, level, overlay_active, P, has_prev, R);
        run_level<COMP, true, false>(C, level, overlay_active, P, D, dt, fault_k + 1, fault_k, R, lag);
        const uint32_t slot = atomicAdd(&counters[0], 1u);
        const uint32_t tick = (tick_dev ? (uint32_t)*tick_dev : 0u) + tick_base + (uint32_t)fault_k;
        if ((int64_t)slot < fault_cap)
            fault_log[slot] = ((uint64_t)(tick & 0xFFFFFFu) << 40) | (uint64_t)r;
    }
    store_state<COMP>(C, level, R);
    lag.store();
    lag.store_cmd(C, alive ? K - 1 : fault_k);
    // has_prev |= alive (control.py:181): every row reaching here was alive
    const uint8_t lv = L::feed_on ? (uint8_t)0 : (uint8_t)(fl & SWARMSTEP_LEVEL_MASK);
    return (uint8_t)(lv | (alive ? SWARMSTEP_FLAG_ALIVE : 0u) | SWARMSTEP_FLAG_HAS_PREV);
}

// Launch a step kernel, with the programmatic-stream-serialization attribute
// when `pdl` (the kernel then lets the next such launch start early).
template <class... KArgs, class... Args>
int launch_step(void (*kern)(KArgs...), unsigned grid, unsigned block, cudaStream_t s, bool pdl, const char *name,
                Args... args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    if (cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...) != cudaSuccess) return ssb::cuda_status(name);
    return ssb::cuda_status(name);
}

// ---- back-to-back step launches that overlap (programmatic dependent launch)
// A step launch only reads and writes its own tiles, and tile b of launch L+1
// depends on tile b of launch L alone.  With PDL (the launch attribute set by
// the host, step_*.cu) every CTA of a step launch lets the next step launch
// start right away (griddepcontrol.launch_dependents), and a CTA of the next
// launch waits for its own tile's epoch (acquire) instead of the whole
// previous grid, so one launch's last wave overlaps the next launch's first.
// Each CTA publishes its tile's epoch (release) after its stores.  Only step
// kernels launched this way trigger early; any other kernel in between keeps
// full stream ordering.  A null tile_epoch disables all of it.
__device__ __forceinline__ void pdl_enter(const ssbl::Pdl &pdl, int64_t tile)
{
    if (!pdl.tile_epoch) return;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (!pdl.wait) return;
    if (threadIdx.x == 0) {
        const long long t0 = clock64();
        for (;;) {
            uint32_t v;
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(pdl.tile_epoch + tile) : "memory");
            if ((int32_t)(v - pdl.wait) >= 0) break;
            if (clock64() - t0 > (1ll << 35)) __trap();   // ~18 s: a broken chain fails loudly
            __nanosleep(256);
        }
    }
    __syncthreads();
}
__device__ __forceinline__ void pdl_exit(const ssbl::Pdl &pdl, int64_t tile)
{
    if (!pdl.tile_epoch) return;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(pdl.tile_epoch + tile), "r"(pdl.set) : "memory");
    }
}

// ---- direct kernel: one row per thread, loads/stores straight to HBM -------
template <bool COMP, bool AXI>
__global__ void __launch_bounds__(kBlock, SSB_STEP_MINB)
quad_step_kernel(float *__restrict__ cols, uint8_t *__restrict__ flags, int64_t n,
                 uint32_t *__restrict__ counters, uint64_t *__restrict__ fault_log,
                 int64_t fault_cap, int overlay_active, uint32_t tick_base, const int64_t *tick_dev,
                 const swarmstep_quad_params P, const ssb::Derived D, float dt, int K, const ssbl::Pdl pdl)
{
    pdl_enter(pdl, blockIdx.x);      // kBlock == one tile
    const int64_t r = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    if (r < n) {
        // every state load is issued before the flag test: one memory round trip
        // per row (dead rows are rare; their loads are discarded)
        const uint8_t fl = flags[r];
        const GlobalRow C{cols + ssb::tile_base(r)};
        Row R;
        load_state<COMP>(C, R);
        // Keep every load of the row ahead of the first use: without this fence
        // ptxas sinks the level-specific command loads behind the level branch,
        // adding a second dependent memory round trip to the HBM-bound K = 1 case.
        __threadfence_block();
        if (fl & SWARMSTEP_FLAG_ALIVE) {   // dead rows are frozen (quad.py:395-437)
            const uint8_t nfl = step_row<COMP>(C, fl, r, overlay_active, P, D, dt, K, tick_base, tick_dev,
                                               counters, fault_log, fault_cap, R, true, NoLagT<AXI>());
            if (nfl != fl) flags[r] = nfl;
        }
    }
    pdl_exit(pdl, blockIdx.x);
}

// ---- motor-lag kernel: the direct kernel with the opt-in rotor lag -----------
// Off the reference path (tau_m = 0 launches the kernels above); one row per
// thread, rotor thrusts in registers across the K ticks next to the state.
template <bool COMP>
__global__ void __launch_bounds__(kBlock, 4)
quad_step_lag_kernel(float *__restrict__ cols, uint8_t *__restrict__ flags, float *__restrict__ motor, int64_t n,
                     uint32_t *__restrict__ counters, uint64_t *__restrict__ fault_log,
                     int64_t fault_cap, int overlay_active, uint32_t tick_base, const int64_t *tick_dev,
                     const swarmstep_quad_params P, const ssb::Derived D, float phi, float e_full, float dt,
                     int K)
{
    const int64_t r = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    if (r >= n) return;
    const uint8_t fl = flags[r];
    if (!(fl & SWARMSTEP_FLAG_ALIVE)) return;   // dead rows frozen, rotor thrusts included
    const GlobalRow C{cols + ssb::tile_base(r)};
    MotorLag lag{motor + (r >> 7) * (4 * SWARMSTEP_TILE) + (r & (SWARMSTEP_TILE - 1)), phi, e_full, {}};
    Row R;
    const uint8_t nfl = step_row<COMP>(C, fl, r, overlay_active, P, D, dt, K, tick_base, tick_dev,
                                       counters, fault_log, fault_cap, R, false, lag);
    if (nfl != fl) flags[r] = nfl;
}

// ---- circle-feed kernel: K ticks of the device circle strategy, fused -------
template <bool COMP, bool AXI>
__global__ void __launch_bounds__(kBlock, 4)
quad_step_circle_kernel(float *__restrict__ cols, uint8_t *__restrict__ flags, int64_t n,
                        uint32_t *__restrict__ counters, uint64_t *__restrict__ fault_log, int64_t fault_cap,
                        uint32_t tick_base, const int64_t *tick_dev, const swarmstep_quad_params P,
                        const ssb::Derived D, swarmstep_circle_feed feed, const ssbl::CircleRot rot, float dt,
                        int K, const ssbl::Pdl pdl)
{
    pdl_enter(pdl, blockIdx.x);
    const int64_t r = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    const uint8_t fl = r < n ? flags[r] : (uint8_t)0;
    if (fl & SWARMSTEP_FLAG_ALIVE) {              // the strategy skips dead agents (client.py:66-67)
        const GlobalRow C{cols + ssb::tile_base(r)};
        const CircleFeedRowT<AXI> cf{*tick_dev + (int64_t)tick_base, feed.dt, feed.radius, feed.omega, feed.z,
                                     feed.phase0 + feed.dphase * (double)r, rot};
        Row R;
        const uint8_t nfl = step_row<COMP>(C, fl, r, 0, P, D, dt, K, tick_base, tick_dev, counters, fault_log,
                                           fault_cap, R, false, cf);
        if (nfl != fl) flags[r] = nfl;
    }
    pdl_exit(pdl, blockIdx.x);
}

// ---- paired kernel: two rows per thread on packed FP32x2 (FFMA2) -------------
// Thread t of a 64-thread CTA owns rows 2t and 2t + 1 of one 128-agent tile.
// When both rows are alive at the same POS or RATE level (the common case)
// they run as one f2 lane pair: every FFMA / FADD / FMUL of the step becomes
// one FFMA2 / FADD2 / FMUL2 for both agents, halving the issued FP
// instructions of this issue-bound kernel.  Otherwise (a dead partner, mixed
// or MOTOR levels) -- and whenever a lane faults -- each row runs the scalar
// path.  Both paths are the same templates with explicitly rounded ops, so
// every row's result is bit-identical to the direct kernel's.
#ifndef SSB_PAIR_MINB
#define SSB_PAIR_MINB 8   // 128 regs: 16 warps per SM (measured best, profiles/tune_r01_v4.json)
#endif
// The paired kernel's per-thread body.  PF / RF: the launch's policy for the
// f2 pair and for a scalar row (NoLag, or the in-kernel circle feed, which
// puts every alive row at POS level).
// The paired kernels' per-thread work once rows r0 and r1 (flag bytes f0,
// f1) are in registers (R): the f2 lane pair or the scalar path per row.  C
// addresses the pair in global memory, C0 / C1 the single rows (stores, and
// the re-reads of a faulted row's launch inputs).
template <bool COMP, class PA, class PF, class RF>
__device__ __forceinline__ void pair_rows(uint8_t *__restrict__ flags, uint32_t *__restrict__ counters,
                                          uint64_t *__restrict__ fault_log, int64_t fault_cap, int overlay_active,
                                          uint32_t tick_base, const int64_t *tick_dev, const swarmstep_quad_params &P,
                                          const ssb::Derived &D, float dt, int K, int64_t r0, int64_t r1, uint8_t f0,
                                          uint8_t f1, const PA &C, const GlobalRow &C0, const GlobalRow &C1,
                                          RowT<ssb::f2> &R, PF pf, RF rf0, RF rf1)
{
    const bool a0 = f0 & SWARMSTEP_FLAG_ALIVE, a1 = f1 & SWARMSTEP_FLAG_ALIVE;
    const int l0 = PF::feed_on ? SWARMSTEP_LEVEL_POS : (f0 & SWARMSTEP_LEVEL_MASK) >> SWARMSTEP_LEVEL_SHIFT;
    const int l1 = PF::feed_on ? SWARMSTEP_LEVEL_POS : (f1 & SWARMSTEP_LEVEL_MASK) >> SWARMSTEP_LEVEL_SHIFT;
    const bool paired = a0 && a1 && l0 == l1 && l0 != SWARMSTEP_LEVEL_MOTOR;
    if (paired) pf.load();
    bool reload = false;
    if (paired) {
        const ssb::m2 hp{(f0 & SWARMSTEP_FLAG_HAS_PREV) != 0, (f1 & SWARMSTEP_FLAG_HAS_PREV) != 0};
        setup_level<PF>(C, l0, overlay_active, P, hp, R);
        if (run_level<COMP, false, false>(C, l0, overlay_active, P, D, dt, K, -1, R, pf) >= 0) {
            // a lane faulted: redo both rows on the scalar path from the
            // launch's inputs, still untouched in HBM
            reload = true;
        } else {
            store_state<COMP>(C, l0, R);
            pf.store();
            pf.store_cmd(C, K - 1);
            const uint8_t hpf = SWARMSTEP_FLAG_HAS_PREV;
            const uint8_t n0 = PF::feed_on ? (uint8_t)((f0 & ~SWARMSTEP_LEVEL_MASK) | hpf) : (uint8_t)(f0 | hpf);
            const uint8_t n1 = PF::feed_on ? (uint8_t)((f1 & ~SWARMSTEP_LEVEL_MASK) | hpf) : (uint8_t)(f1 | hpf);
            if (n0 != f0) flags[r0] = n0;
            if (n1 != f1) flags[r1] = n1;
            return;
        }
    }
    // scalar path per row: the loaded lanes (dead partner, mixed or MOTOR
    // levels) or a fresh load (after a fault in the pair)
    if (a0) {
        Row Rs = lane_row(R, 0);
        const uint8_t nf = step_row<COMP>(C0, f0, r0, overlay_active, P, D, dt, K, tick_base, tick_dev,
                                          counters, fault_log, fault_cap, Rs, !reload, rf0);
        if (nf != f0) flags[r0] = nf;
    }
    if (a1) {
        Row Rs = lane_row(R, 1);
        const uint8_t nf = step_row<COMP>(C1, f1, r1, overlay_active, P, D, dt, K, tick_base, tick_dev,
                                          counters, fault_log, fault_cap, Rs, !reload, rf1);
        if (nf != f1) flags[r1] = nf;
    }
}

// adjacent rows r0 = 2t, r0 + 1 of a tile loaded straight from HBM (one
// 8-byte load per column), then pair_rows.  Rows in [n, stride) are dead
// padding (flags 0), so the pair's second row needs no bound check.
template <bool COMP, class PF, class RF>
__device__ __forceinline__ void pair_body(float *__restrict__ cols, uint8_t *__restrict__ flags, int64_t n,
                                          uint32_t *__restrict__ counters, uint64_t *__restrict__ fault_log,
                                          int64_t fault_cap, int overlay_active, uint32_t tick_base,
                                          const int64_t *tick_dev, const swarmstep_quad_params &P,
                                          const ssb::Derived &D, float dt, int K, int64_t r0, PF pf, RF rf0, RF rf1)
{
    const int64_t r1 = r0 + 1;
    const uint16_t ff = *reinterpret_cast<const uint16_t *>(flags + r0);
    const uint8_t f0 = (uint8_t)(ff & 0xFFu), f1 = (uint8_t)(ff >> 8);
    float *base = cols + ssb::tile_base(r0);
    const VecPairRow C{base};
    const GlobalRow C0{base}, C1{base + 1};
    // both rows' loads in flight before any decision (see quad_step_kernel)
    RowT<ssb::f2> R;
    load_state<COMP>(C, R);
    __threadfence_block();
    pair_rows<COMP>(flags, counters, fault_log, fault_cap, overlay_active, tick_base, tick_dev, P, D, dt, K, r0, r1,
                    f0, f1, C, C0, C1, R, pf, rf0, rf1);
    (void)n;
}

template <bool COMP, bool AXI>
__global__ void __launch_bounds__(64, SSB_PAIR_MINB)
quad_step_pair_kernel(float *__restrict__ cols, uint8_t *__restrict__ flags, int64_t n,
                      uint32_t *__restrict__ counters, uint64_t *__restrict__ fault_log,
                      int64_t fault_cap, int overlay_active, uint32_t tick_base, const int64_t *tick_dev,
                      const swarmstep_quad_params P, const ssb::Derived D, float dt, int K, const ssbl::Pdl pdl)
{
    pdl_enter(pdl, blockIdx.x);
    const int64_t r0 = (int64_t)blockIdx.x * SWARMSTEP_TILE + 2 * threadIdx.x;
    if (r0 < n)
        pair_body<COMP>(cols, flags, n, counters, fault_log, fault_cap, overlay_active, tick_base, tick_dev, P, D, dt,
                        K, r0, NoLagT<AXI>(), NoLagT<AXI>(), NoLagT<AXI>());
    pdl_exit(pdl, blockIdx.x);
}

// the paired kernel with the opt-in rotor lag
template <bool COMP>
__global__ void __launch_bounds__(64, SSB_PAIR_MINB)
quad_step_pair_lag_kernel(float *__restrict__ cols, uint8_t *__restrict__ flags, float *__restrict__ motor, int64_t n,
                          uint32_t *__restrict__ counters, uint64_t *__restrict__ fault_log, int64_t fault_cap,
                          int overlay_active, uint32_t tick_base, const int64_t *tick_dev,
                          const swarmstep_quad_params P, const ssb::Derived D, float phi, float e_full, float dt,
                          int K)
{
    const int64_t r0 = (int64_t)blockIdx.x * SWARMSTEP_TILE + 2 * threadIdx.x;
    if (r0 >= n) return;
    float *m0 = motor + (r0 >> 7) * (4 * SWARMSTEP_TILE) + (r0 & (SWARMSTEP_TILE - 1)), *m1 = m0 + 1;
    pair_body<COMP>(cols, flags, n, counters, fault_log, fault_cap, overlay_active, tick_base, tick_dev, P, D, dt, K,
                    r0, MotorLagPair{m0, m1, phi, e_full, {}}, MotorLag{m0, phi, e_full, {}},
                    MotorLag{m1, phi, e_full, {}});
}

// the paired kernel with the in-kernel circle feed (every alive row at POS)
template <bool COMP, bool AXI>
__global__ void __launch_bounds__(64, SSB_PAIR_MINB)
quad_step_pair_circle_kernel(float *__restrict__ cols, uint8_t *__restrict__ flags, int64_t n,
                             uint32_t *__restrict__ counters, uint64_t *__restrict__ fault_log, int64_t fault_cap,
                             uint32_t tick_base, const int64_t *tick_dev, const swarmstep_quad_params P,
                             const ssb::Derived D, swarmstep_circle_feed feed, const ssbl::CircleRot rot, float dt,
                             int K, const ssbl::Pdl pdl)
{
    pdl_enter(pdl, blockIdx.x);
    const int64_t r0 = (int64_t)blockIdx.x * SWARMSTEP_TILE + 2 * threadIdx.x;
    if (r0 < n) {
        const int64_t tick0 = *tick_dev + (int64_t)tick_base;
        const CircleFeedRowT<AXI> c0{tick0, feed.dt, feed.radius, feed.omega, feed.z,
                                     feed.phase0 + feed.dphase * (double)r0, rot};
        const CircleFeedRowT<AXI> c1{tick0, feed.dt, feed.radius, feed.omega, feed.z,
                                     feed.phase0 + feed.dphase * (double)(r0 + 1), rot};
        pair_body<COMP>(cols, flags, n, counters, fault_log, fault_cap, 0, tick_base, tick_dev, P, D, dt, K, r0,
                        CircleFeedPairT<AXI>{c0, c1}, c0, c1);
    }
    pdl_exit(pdl, blockIdx.x);
}

// ---- TMA kernel: persistent CTAs, tiles staged through shared memory --------
// Each CTA walks tiles blockIdx.x, +gridDim.x, ...  One elected thread moves a
// tile's input columns HBM -> shared memory with one cp.async.bulk (TMA) per
// tile into a kStages-deep ring (mbarrier completion), so the next tiles'
// loads are in flight while this one is computed; results are written back
// into the same shared tile and leave with two bulk stores (cols [0, 22) and
// the stale setpoints [29, 33)).  No register holds an in-flight load.
#ifndef SSB_TMA_STAGES
#define SSB_TMA_STAGES 3
#endif
constexpr int kStages = SSB_TMA_STAGES;
constexpr int kTileFloats = SWARMSTEP_NCOL * SWARMSTEP_TILE;

struct TmaSmem {
    float tile[kStages][kTileFloats];
    uint8_t flags[kStages][SWARMSTEP_TILE];
    unsigned long long full[kStages];
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(unsigned long long *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long *bar, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "SSB_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra SSB_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, unsigned long long *bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, uint32_t bytes)
{
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
}

#ifndef SSB_TMA_MINB
#define SSB_TMA_MINB 4   // 3 x 18.6 KB stages per CTA: 4 CTAs fill the 228 KB of shared memory
#endif
template <bool COMP>
__global__ void __launch_bounds__(SWARMSTEP_TILE, SSB_TMA_MINB)
quad_step_tma_kernel(float *__restrict__ cols, uint8_t *__restrict__ flags, int64_t ntiles,
                     uint32_t *__restrict__ counters, uint64_t *__restrict__ fault_log, int64_t fault_cap,
                     int overlay_active, int motor_possible, uint32_t tick_base, const int64_t *tick_dev,
                     const swarmstep_quad_params P, const ssb::Derived D, float dt, int K)
{
    extern __shared__ __align__(128) unsigned char smem_raw[];
    TmaSmem &S = *reinterpret_cast<TmaSmem *>(smem_raw);
    const int tid = threadIdx.x;
    // input columns: [0, 29) always; the stale setpoints [29, 33) only if a
    // MOTOR row may exist; the overlay [33, 36) only on overlay ticks
    const int in_cols = overlay_active ? SWARMSTEP_NCOL : (motor_possible ? SWARMSTEP_COL_OVERLAY : SWARMSTEP_COL_SP);
    const uint32_t in_bytes = (uint32_t)in_cols * SWARMSTEP_TILE * 4u;
    if (tid == 0) {
        for (int s = 0; s < kStages; s++) mbar_init(&S.full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int64_t t0 = blockIdx.x, tstep = gridDim.x;
    auto issue = [&](int s, int64_t t) {
        mbar_expect_tx(&S.full[s], in_bytes + SWARMSTEP_TILE);
        bulk_g2s(S.tile[s], cols + t * kTileFloats, in_bytes, &S.full[s]);
        bulk_g2s(S.flags[s], flags + t * SWARMSTEP_TILE, SWARMSTEP_TILE, &S.full[s]);
    };
    if (tid == 0)
        for (int s = 0; s < kStages; s++)
            if (t0 + s * tstep < ntiles) issue(s, t0 + s * tstep);

    int64_t j = 0;
    for (int64_t t = t0; t < ntiles; t += tstep, j++) {
        const int s = (int)(j % kStages);
        mbar_wait(&S.full[s], (uint32_t)((j / kStages) & 1));
        float *T = S.tile[s];
        const uint8_t fl = S.flags[s][tid];
        const int64_t r = t * SWARMSTEP_TILE + tid;
        const SmemRow C{T + tid};
        if (fl & SWARMSTEP_FLAG_ALIVE) {
            Row Rs;
            const uint8_t nfl = step_row<COMP>(C, fl, r, overlay_active, P, D, dt, K, tick_base, tick_dev,
                                               counters, fault_log, fault_cap, Rs);
            if (nfl != fl) flags[r] = nfl;
        } else if (!motor_possible && !overlay_active) {
            // dead row, stale setpoints not staged: store zeros, not stale smem
#pragma unroll
            for (int i = 0; i < 4; i++) C.st(SWARMSTEP_COL_SP + i, 0.0f);
        }
        // make the generic-proxy smem writes visible to the bulk-copy engine
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (tid == 0) {
            float *g = cols + t * kTileFloats;
            bulk_s2g(g, T, SWARMSTEP_COL_CMD * SWARMSTEP_TILE * 4u);
            bulk_s2g(g + SWARMSTEP_COL_SP * SWARMSTEP_TILE, T + SWARMSTEP_COL_SP * SWARMSTEP_TILE,
                     4u * SWARMSTEP_TILE * 4u);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            // Refill the stage of the PREVIOUS tile (its stores were issued one
            // iteration ago, so waiting until all but the newest store group
            // have read shared memory rarely blocks): tile (j-1) + kStages.
            const int64_t tn = t + (kStages - 1) * tstep;
            if (j >= 1 && tn < ntiles) {
                asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                issue((int)((j - 1) % kStages), tn);
            }
        }
    }
    if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

}  // namespace
