// quad_math.cuh -- per-agent float32 device math for the quadrotor hot path.
//
// Each function restates one piece of the reference's batched numpy path for
// agents held in registers:
//   deriv / rk4_inplace  quad.py:222-310, 350-437  (_deriv_kernel, rk4_step)
//   mix_row              quad.py:143-168           (mix_to_motors)
//   motor_wrench         quad.py:130-140 + core.py:189-197
//   pid_row              control.py:136-187        (rate_pid_step)
//   outer_row            control.py:190-294        (position_outer_loop, _rotmats_to_quats)
//
// Every function is a template over the lane type T: `float` (one agent) or
// `f2` (two agents in the two halves of Blackwell's packed FP32x2 registers,
// so FFMA2 / FADD2 / FMUL2 do two agents' arithmetic per issued instruction).
// All arithmetic goes through explicitly rounded operations (no compiler
// contraction), so an agent's result is bit-identical whichever lane type
// computed it -- rows stay independent of their neighbours.
//
// Numerics (float32 against the float64 reference, target <= 1e-5 relative
// per step):
//  * the mixer returns the requested wrench unchanged for unsaturated rows
//    (G G^-1 w == w in R; a float32 round trip would inject |f_c| eps32 of
//    torque error -- SURVEY.md Appendix B);
//  * position can be carried as an unevaluated sum hi + lo (Fast2Sum) so the
//    reference's sub-ulp increments at |p| ~ 100 m are kept;
//  * sqrt / 1/x / 1/sqrt use the SFU (MUFU) approximations (<= 2 ulp) and
//    atan2 a degree-8 minimax polynomial (9e-8 relative): all well inside the
//    1e-5 budget, and free of the IEEE slow paths.
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include "swarmstep_b200.h"

namespace ssb {

// ---------------------------------------------------------------------------
// lane types
// ---------------------------------------------------------------------------
struct f2 {
    float2 v;
};
struct m2 {
    bool x, y;
};

template <class T> struct LaneMask;
template <> struct LaneMask<float> { using type = bool; };
template <> struct LaneMask<f2> { using type = m2; };
template <class T> using mask_t = typename LaneMask<T>::type;

template <class T> __device__ __forceinline__ T bc(float a);
template <> __device__ __forceinline__ float bc<float>(float a) { return a; }
template <> __device__ __forceinline__ f2 bc<f2>(float a) { return f2{make_float2(a, a)}; }

__device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ float fnma(float a, float b, float c) { return __fmaf_rn(-a, b, c); }  // c - a b
__device__ __forceinline__ float neg(float a) { return -a; }

__device__ __forceinline__ f2 add(f2 a, f2 b) { return f2{__fadd2_rn(a.v, b.v)}; }
__device__ __forceinline__ f2 sub(f2 a, f2 b) { return f2{__fadd2_rn(a.v, make_float2(-b.v.x, -b.v.y))}; }
__device__ __forceinline__ f2 mul(f2 a, f2 b) { return f2{__fmul2_rn(a.v, b.v)}; }

// mul_nc: a product whose result feeds an add / sub.  ptxas 12.9 contracts
// mul.rn.f32x2 + add.rn.f32x2 into FFMA2 despite the explicit rounding (it
// keeps scalar mul.rn / add.rn apart), which would make packed lanes round
// differently from scalar rows.  Such a product is issued as fma(a, b, -0):
// the same single rounding as mul.rn (round(a b) + -0 == round(a b), signed
// zeros included), and an FFMA2 result cannot be contracted further.  The -0
// lives in constant memory so ptxas cannot fold the FMA back into a multiply.
// Products that feed only multiplications, FMA multiplicands or addends,
// min / max or selects use plain mul (nothing to contract with).
static __constant__ float c_neg_zero = -0.0f;
__device__ __forceinline__ float mul_nc(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ f2 mul_nc(f2 a, f2 b) { return f2{__ffma2_rn(a.v, b.v, make_float2(c_neg_zero, c_neg_zero))}; }
// Operand order: an FFMA2 reading three vector registers issues at 2/3 rate
// (register-file read bandwidth; measured 49.5 vs 74.2 TFLOP/s with one
// operand uniform / immediate).  Only the second multiplicand and the addend
// can be uniform registers or immediates, so a * b + c is issued as b * a + c
// (exactly the same value): call sites put the per-type constant first.
__device__ __forceinline__ f2 fma(f2 a, f2 b, f2 c) { return f2{__ffma2_rn(b.v, a.v, c.v)}; }
__device__ __forceinline__ f2 fnma(f2 a, f2 b, f2 c) { return f2{__ffma2_rn(make_float2(-b.v.x, -b.v.y), a.v, c.v)}; }
__device__ __forceinline__ f2 neg(f2 a) { return f2{make_float2(-a.v.x, -a.v.y)}; }

// per-lane helpers
template <class F> __device__ __forceinline__ float lane1(float a, F f) { return f(a); }
template <class F> __device__ __forceinline__ f2 lane1(f2 a, F f) { return f2{make_float2(f(a.v.x), f(a.v.y))}; }

__device__ __forceinline__ float rsqrt1(float x)
{
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float sqrt1(float x)
{
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp1(float x)
{
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
template <class T> __device__ __forceinline__ T rsqrt_a(T x) { return lane1(x, rsqrt1); }
template <class T> __device__ __forceinline__ T sqrt_a(T x) { return lane1(x, sqrt1); }
template <class T> __device__ __forceinline__ T rcp_a(T x) { return lane1(x, rcp1); }

__device__ __forceinline__ float vmin(float a, float b) { return fminf(a, b); }
__device__ __forceinline__ float vmax(float a, float b) { return fmaxf(a, b); }
__device__ __forceinline__ float vabs(float a) { return fabsf(a); }
__device__ __forceinline__ f2 vmin(f2 a, f2 b) { return f2{make_float2(fminf(a.v.x, b.v.x), fminf(a.v.y, b.v.y))}; }
__device__ __forceinline__ f2 vmax(f2 a, f2 b) { return f2{make_float2(fmaxf(a.v.x, b.v.x), fmaxf(a.v.y, b.v.y))}; }
__device__ __forceinline__ f2 vabs(f2 a) { return f2{make_float2(fabsf(a.v.x), fabsf(a.v.y))}; }

// NaN-propagating min / max (PTX max.NaN / min.NaN, sm_80+): the same cost
// as fminf / fmaxf, but a NaN operand yields NaN instead of the other operand
__device__ __forceinline__ float vmax_nan(float a, float b)
{
    float r;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float vmin_nan(float a, float b)
{
    float r;
    asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ f2 vmax_nan(f2 a, f2 b) { return f2{make_float2(vmax_nan(a.v.x, b.v.x), vmax_nan(a.v.y, b.v.y))}; }
__device__ __forceinline__ f2 vmin_nan(f2 a, f2 b) { return f2{make_float2(vmin_nan(a.v.x, b.v.x), vmin_nan(a.v.y, b.v.y))}; }

__device__ __forceinline__ bool lt(float a, float b) { return a < b; }
__device__ __forceinline__ bool gt(float a, float b) { return a > b; }
__device__ __forceinline__ bool ge(float a, float b) { return a >= b; }
__device__ __forceinline__ bool le(float a, float b) { return a <= b; }
__device__ __forceinline__ bool eq(float a, float b) { return a == b; }
__device__ __forceinline__ m2 lt(f2 a, f2 b) { return m2{a.v.x < b.v.x, a.v.y < b.v.y}; }
__device__ __forceinline__ m2 gt(f2 a, f2 b) { return m2{a.v.x > b.v.x, a.v.y > b.v.y}; }
__device__ __forceinline__ m2 ge(f2 a, f2 b) { return m2{a.v.x >= b.v.x, a.v.y >= b.v.y}; }
__device__ __forceinline__ m2 le(f2 a, f2 b) { return m2{a.v.x <= b.v.x, a.v.y <= b.v.y}; }
__device__ __forceinline__ m2 eq(f2 a, f2 b) { return m2{a.v.x == b.v.x, a.v.y == b.v.y}; }

__device__ __forceinline__ bool mand(bool a, bool b) { return a && b; }
__device__ __forceinline__ bool mor(bool a, bool b) { return a || b; }
__device__ __forceinline__ bool mnot(bool a) { return !a; }
__device__ __forceinline__ bool any(bool a) { return a; }
__device__ __forceinline__ m2 mand(m2 a, m2 b) { return m2{a.x && b.x, a.y && b.y}; }
__device__ __forceinline__ m2 mor(m2 a, m2 b) { return m2{a.x || b.x, a.y || b.y}; }
__device__ __forceinline__ m2 mnot(m2 a) { return m2{!a.x, !a.y}; }
__device__ __forceinline__ bool any(m2 a) { return a.x || a.y; }

__device__ __forceinline__ float sel(bool m, float a, float b) { return m ? a : b; }
__device__ __forceinline__ f2 sel(m2 m, f2 a, f2 b) { return f2{make_float2(m.x ? a.v.x : b.v.x, m.y ? a.v.y : b.v.y)}; }

__device__ __forceinline__ float lane(float a, int) { return a; }
__device__ __forceinline__ float lane(f2 a, int i) { return i ? a.v.y : a.v.x; }

// double -> float, finite values beyond float32 range saturate at +-FLT_MAX
__device__ __forceinline__ float f32_sat(double x)
{
    return isfinite(x) ? (float)fmin(fmax(x, -3.4028234663852886e38), 3.4028234663852886e38) : (float)x;
}

// cos / sin of the yaw setpoint and of its half (the outer loop's heading and
// its quaternion factor), once per launch.  (Deriving the pair from the half
// angle by the double-angle formulas saves a sincos but measured 1 % slower per
// K = 10 launch: profiles/tune_r02/r02n_*.)
__device__ __forceinline__ void yaw_terms(float yaw, float &c, float &s, float &ch, float &sh)
{
    sincosf(yaw, &s, &c);
    sincosf(0.5f * yaw, &sh, &ch);
}

// np.clip semantics: NaN passes through
template <class T> __device__ __forceinline__ T clip(T x, T lo, T hi)
{
    return sel(lt(x, lo), lo, sel(gt(x, hi), hi, x));
}
// the same with NaN-propagating min / max (two ALU ops instead of two
// compares and two selects; a -0 input comes out as +0)
template <class T> __device__ __forceinline__ T clip_nan(T x, T lo, T hi)
{
    return vmin_nan(vmax_nan(x, lo), hi);
}

// ---------------------------------------------------------------------------
// Per-launch constants derived from the per-type struct on the host and passed
// as a kernel parameter (constant bank: no per-thread registers)
// ---------------------------------------------------------------------------
struct Derived {
    float g;
    float gx, gy, gz;        // (I_zz - I_yy) / I_xx, ... (gyroscopic coefficients)
    float kd_dt[3];          // kd / dt
    // RK4 step constants and 2: kernel parameters (uniform registers) rather
    // than values the kernel computes or materialises into vector registers,
    // so the FFMA2s using them read two vector registers (see fma below)
    float dt, half_dt, quarter_dt, sixth_dt, twelfth_dt, two;
    float dt2_sixth;         // dt^2 / 6: the position increment's acceleration weight
    // parameter combinations the per-tick code would otherwise recompute
    float two_inv_m, neg_g, two_m, m_amin, two_m_amin, amin_sq, neg_w_sp_max, g_inv2_abs;
    float neg_i_limit[3];
    // axisymmetric vehicle: I_xx == I_yy and every x / y gain pair equal (the
    // default quad).  Kernels instantiated for it (AXI) read the x constants
    // for y -- fewer distinct constants in the tick loop -- and drop the yaw
    // gyroscopic term, whose coefficient (I_yy - I_xx) / I_zz is exactly 0.
    int axisym;
};

__host__ __device__ __forceinline__ Derived derive(const swarmstep_quad_params &P, float dt)
{
    Derived d;
    const float inv_dt = 1.0f / dt;
    d.g = P.g;
    d.gx = (P.izz - P.iyy) * P.inv_ixx;
    d.gy = (P.ixx - P.izz) * P.inv_iyy;
    d.gz = (P.iyy - P.ixx) * P.inv_izz;
#pragma unroll
    for (int i = 0; i < 3; i++) d.kd_dt[i] = P.kd[i] * inv_dt;
    d.dt = dt;
    d.half_dt = 0.5f * dt;
    d.quarter_dt = 0.25f * dt;
    d.sixth_dt = dt * (1.0f / 6.0f);
    d.twelfth_dt = 0.5f * d.sixth_dt;
    d.two = 2.0f;
    d.dt2_sixth = (float)((double)dt * (double)dt / 6.0);
    d.two_inv_m = 2.0f * P.inv_m;
    d.neg_g = -P.g;
    d.two_m = 2.0f * P.m;
    d.m_amin = P.m * P.a_cmd_min;
    d.two_m_amin = 2.0f * P.m * P.a_cmd_min;
    d.amin_sq = P.a_cmd_min * P.a_cmd_min;
    d.neg_w_sp_max = -P.omega_sp_max;
    d.g_inv2_abs = fabsf(P.G_inv[2]);
    for (int i = 0; i < 3; i++) d.neg_i_limit[i] = -P.i_limit[i];
    d.axisym = P.ixx == P.iyy && P.inv_ixx == P.inv_iyy && P.kp[0] == P.kp[1] && P.ki[0] == P.ki[1] &&
               P.kd[0] == P.kd[1] && P.i_limit[0] == P.i_limit[1] && P.kp_pos[0] == P.kp_pos[1] &&
               P.kv[0] == P.kv[1] && P.k_att[0] == P.k_att[1];
    return d;
}

// d/dt of (v, 2 q, w) at (q, w) for a held wrench (quad.py:222-310):
//   vdot = (f_c/m) R(q) e_z - g e_z ; 2 qdot = q (x) (0, w) ;
//   wdot = tau/I - c (w_j w_k)  (gyroscopic term, diagonal inertia).
// fc2 = 2 f_c / m, fcg = f_c / m - g, tI = tau / I.  The quaternion rate is
// returned doubled (the RK4 stage weights carry the 1/2): all three stage
// inputs are then plain state values, and every product is the reference
// formula's scaled by an exact power of two.
// the constant index of axis i: y reads x's constants on an axisymmetric vehicle
template <bool AXI> __host__ __device__ constexpr int axc(int i) { return (AXI && i == 1) ? 0 : i; }

// thrust direction terms of R(q) e_z = (2 S0, 2 S1, 1 - 2 S2):
// S0 = qx qz + qw qy, S1 = qy qz - qw qx, S2 = qx^2 + qy^2
template <class T>
__device__ __forceinline__ void thrust_terms(const T q[4], T S[3])
{
    const T qw = q[0], qx = q[1], qy = q[2], qz = q[3];
    S[0] = fma(qx, qz, mul(qw, qy));
    S[1] = fnma(qw, qx, mul(qy, qz));
    S[2] = fma(qx, qx, mul(qy, qy));
}

// S: the thrust terms of q when the caller already has them (the outer loop
// computed them from the same quaternion), else null
// AXI: I_xx == I_yy, so D.gz == 0 exactly and wdot_z = tau_z / I_zz
template <bool AXI = false, class T>
__device__ __forceinline__ void deriv(const T q[4], const T w[3], T fc2, T fcg, const T tI[3], const Derived &D,
                                      T dv[3], T dq[4], T dw[3], const T *S = nullptr)
{
    const T qw = q[0], qx = q[1], qy = q[2], qz = q[3];
    const T wx = w[0], wy = w[1], wz = w[2];
    T St[3];
    if (S == nullptr) {
        thrust_terms(q, St);
        S = St;
    }
    dv[0] = mul_nc(fc2, S[0]);     // feed the RK4 stage sums
    dv[1] = mul_nc(fc2, S[1]);
    dv[2] = fnma(fc2, S[2], fcg);
    dq[0] = neg(fma(qx, wx, fma(qy, wy, mul(qz, wz))));
    dq[1] = fma(qw, wx, fnma(qz, wy, mul(qy, wz)));
    dq[2] = fma(qw, wy, fnma(qx, wz, mul(qz, wx)));
    dq[3] = fma(qw, wz, fnma(qy, wx, mul(qx, wy)));
    dw[0] = fnma(bc<T>(D.gx), mul(wy, wz), tI[0]);
    // axisymmetric: c_y = (I_xx - I_zz) / I_yy = -c_x exactly
    dw[1] = AXI ? fma(bc<T>(D.gx), mul(wz, wx), tI[1]) : fnma(bc<T>(D.gy), mul(wz, wx), tI[1]);
    dw[2] = AXI ? tI[2] : fnma(bc<T>(D.gz), mul(wx, wy), tI[2]);
}

// One classical RK4 step with the wrench held (quad.py:350-437), in place.
// Returns, per lane, whether the row stays finite (the reference's fault
// predicate, quad.py:404-430); a faulted lane's state is garbage and the
// caller restores its pre-step values.
//
// Position feeds no derivative and vdot depends on q alone, so the stage
// velocities v + c k are never needed: RK4's position increment
// dt/6 (v1 + 2 v2 + 2 v3 + v4) with v2 = v + dt/2 k1, v3 = v + dt/2 k2,
// v4 = v + dt k3 is exactly dt v + dt^2/6 (k1 + k2 + k3), accumulated as it
// goes (4 FMAs per axis instead of 7, and no stage-velocity registers).
// ACC (compensated position only): p_lo is a launch-local accumulator of
// the position increments against a p_hi held fixed for the whole launch
// (|acc| grows to about K |v| dt, rounding at ulp(acc) instead of a Fast2Sum
// per tick); the step kernels fold it back into (hi, lo) once per launch
// (fold_position).  Without ACC each tick ends with the Fast2Sum
// (the function-level rk4_step, ops.cu).
template <class T, bool COMP, bool ACC = false, bool AXI = false>
__device__ __forceinline__ mask_t<T> rk4_inplace(T p_hi[3], T p_lo[3], T v[3], T q[4], T w[3], T f_c,
                                                 const T tau[3], const swarmstep_quad_params &P,
                                                 const Derived &D, float dt, const T *S1 = nullptr)
{
    const T half = bc<T>(D.half_dt), h6 = bc<T>(D.sixth_dt), dtv = bc<T>(D.dt);
    const T qtr = bc<T>(D.quarter_dt), h12 = bc<T>(D.twelfth_dt);  // weights of the doubled quaternion rate
    const T two = bc<T>(D.two);
    // fc2 = 2 f_c / m (exact doubling of f_c / m); fcg = f_c / m - g in one FMA
    const T fc2 = mul(f_c, bc<T>(D.two_inv_m));
    const T fcg = fma(bc<T>(P.inv_m), f_c, bc<T>(D.neg_g));
    const T tI[3] = {mul(tau[0], bc<T>(P.inv_ixx)), mul(tau[1], bc<T>(AXI ? P.inv_ixx : P.inv_iyy)),
                     mul(tau[2], bc<T>(P.inv_izz))};
    T kv[3], kq[4], kw[3];
    T av[3], aq[4], aw[3];
    T sq[4], sw[3];
    // b = (lo +) dt v, then + dt^2/6 k_i for the first three stages
    const T d26 = bc<T>(D.dt2_sixth);
    T b[3];
#pragma unroll
    for (int i = 0; i < 3; i++) b[i] = COMP ? fma(dtv, v[i], p_lo[i]) : mul(dtv, v[i]);

    deriv<AXI>(q, w, fc2, fcg, tI, D, kv, kq, kw, S1);                   // k1
#pragma unroll
    for (int i = 0; i < 3; i++) { av[i] = kv[i]; aw[i] = kw[i]; }
#pragma unroll
    for (int i = 0; i < 4; i++) aq[i] = kq[i];
#pragma unroll
    for (int s = 0; s < 2; s++) {                                   // k2, k3 at y + h/2 k
#pragma unroll
        for (int i = 0; i < 3; i++) {
            sw[i] = fma(half, kw[i], w[i]);
            b[i] = fma(d26, kv[i], b[i]);
        }
#pragma unroll
        for (int i = 0; i < 4; i++) sq[i] = fma(qtr, kq[i], q[i]);
        deriv<AXI>(sq, sw, fc2, fcg, tI, D, kv, kq, kw);
#pragma unroll
        for (int i = 0; i < 3; i++) { av[i] = fma(two, kv[i], av[i]); aw[i] = fma(two, kw[i], aw[i]); }
#pragma unroll
        for (int i = 0; i < 4; i++) aq[i] = fma(two, kq[i], aq[i]);
    }
#pragma unroll
    for (int i = 0; i < 3; i++) {
        sw[i] = fma(dtv, kw[i], w[i]);
        b[i] = fma(d26, kv[i], b[i]);
    }
#pragma unroll
    for (int i = 0; i < 4; i++) sq[i] = fma(half, kq[i], q[i]);
    deriv<AXI>(sq, sw, fc2, fcg, tI, D, kv, kq, kw);                // k4
#pragma unroll
    for (int i = 0; i < 3; i++) { av[i] = add(av[i], kv[i]); aw[i] = add(aw[i], kw[i]); }
#pragma unroll
    for (int i = 0; i < 4; i++) aq[i] = add(aq[i], kq[i]);

    // y' = y + dt/6 (k1 + 2 k2 + 2 k3 + k4)
#pragma unroll
    for (int i = 0; i < 3; i++) {
        v[i] = fma(h6, av[i], v[i]);
        w[i] = fma(h6, aw[i], w[i]);
        const T b_i = b[i];
        if (COMP && ACC) {
            p_lo[i] = b_i;
        } else if (COMP) {
            // Fast2Sum of hi and b (the increment plus the carried lo): exact
            // when |hi| >= |b| (a position against one tick's displacement);
            // keeps |lo| <= ulp(hi)/2
            const T sum = add(p_hi[i], b_i);
            p_lo[i] = sub(b_i, sub(sum, p_hi[i]));
            p_hi[i] = sum;
        } else {
            p_hi[i] = add(p_hi[i], b_i);
        }
    }
#pragma unroll
    for (int i = 0; i < 4; i++) q[i] = fma(h12, aq[i], q[i]);

    // single post-step renormalisation; zero / non-finite norm is a fault
    const T nsq = fma(q[0], q[0], fma(q[1], q[1], fma(q[2], q[2], mul(q[3], q[3]))));
    const T inv = rsqrt_a(nsq);
#pragma unroll
    for (int i = 0; i < 4; i++) q[i] = mul(q[i], inv);
    // 0 * x is NaN exactly when x is inf / NaN, so one compare covers every
    // position / velocity / rate component (and nsq)
    T s = add(add(add(p_hi[0], p_hi[1]), add(p_hi[2], v[0])), add(add(v[1], v[2]), add(w[0], w[1])));
    s = add(s, add(w[2], nsq));
    if (COMP) s = add(s, add(add(p_lo[0], p_lo[1]), p_lo[2]));
    const T chk = mul(bc<T>(0.0f), s);
    return mand(gt(nsq, bc<T>(0.0f)), eq(chk, bc<T>(0.0f)));
}

// Fast2Sum of a launch-local accumulator back into (hi, lo), |lo| <= ulp(hi)/2
template <class T>
__device__ __forceinline__ void fold_position(T p_hi[3], T p_lo[3])
{
#pragma unroll
    for (int i = 0; i < 3; i++) {
        const T sum = add(p_hi[i], p_lo[i]);
        p_lo[i] = sub(p_lo[i], sub(sum, p_hi[i]));
        p_hi[i] = sum;
    }
}

// mix_to_motors (quad.py:143-168): realized wrench after per-motor clamp.
// G (quad.py:106-122) has mutually orthogonal rows, so G^-1 = G^T diag(c):
// motor i = c0 f + s_i1 c1 tau_x + s_i2 c2 tau_y + s_i3 c3 tau_z with the
// sign pattern of G's columns.  P.G_inv carries the exact inverse; the host
// checks the pattern (params.py) and the kernel uses c = |G_inv[0][:]|.
template <class T>
__device__ __forceinline__ void mix_row(T &f_c, T tau[3], const swarmstep_quad_params &P, const Derived &D)
{
    // c0 f +- c1 tau_x and c2 tau_y -+ c3 tau_z, one product folded into an FMA
    const T A = mul(bc<T>(P.G_inv[1]), tau[0]), C = mul(bc<T>(P.G_inv[3]), tau[2]);
    const T c0 = bc<T>(P.G_inv[0]), c2 = bc<T>(D.g_inv2_abs);
    const T FpA = fma(c0, f_c, A), FmA = fma(c0, f_c, neg(A)), BmC = fma(c2, tau[1], neg(C)), BpC = fma(c2, tau[1], C);
    T m[4] = {sub(FpA, BmC), sub(FmA, BpC), add(FmA, BpC), add(FpA, BmC)};
    const T lo = vmin(vmin(m[0], m[1]), vmin(m[2], m[3]));
    const T hi = vmax(vmax(m[0], m[1]), vmax(m[2], m[3]));
    const mask_t<T> sat = mor(lt(lo, bc<T>(0.0f)), gt(hi, bc<T>(P.f_max)));
    if (any(sat)) {
#pragma unroll
        for (int i = 0; i < 4; i++) m[i] = clip_nan(m[i], bc<T>(0.0f), bc<T>(P.f_max));
        // realized wrench G m (quad.py:160-168) on G's X structure: rows
        // (1 1 1 1), ls (1 -1 -1 1), lc (-1 -1 1 1), kr (1 -1 1 -1)
        const T s01 = add(m[0], m[1]), s23 = add(m[2], m[3]);
        const T s03 = add(m[0], m[3]), s12 = add(m[1], m[2]);
        const T s02 = add(m[0], m[2]), s13 = add(m[1], m[3]);
        f_c = sel(sat, add(s01, s23), f_c);
        tau[0] = sel(sat, mul(bc<T>(P.G[4]), sub(s03, s12)), tau[0]);
        tau[1] = sel(sat, mul(bc<T>(P.G[11]), sub(s23, s01)), tau[1]);
        tau[2] = sel(sat, mul(bc<T>(P.G[12]), sub(s02, s13)), tau[2]);
    }
}

// raw motor speeds -> wrench = G (k_t clip(rpm)^2)  (quad.py:130-140, core.py:189-197)
__device__ __forceinline__ void motor_wrench(const float rpm[4], const swarmstep_quad_params &P,
                                             float &f_c, float tau[3])
{
    float f[4];
#pragma unroll
    for (int i = 0; i < 4; i++) {
        const float c = clip(rpm[i], 0.0f, P.omega_max);
        f[i] = P.k_t * (c * c);
    }
    f_c = P.G[0] * f[0] + P.G[1] * f[1] + P.G[2] * f[2] + P.G[3] * f[3];
#pragma unroll
    for (int i = 0; i < 3; i++)
        tau[i] = P.G[(i + 1) * 4 + 0] * f[0] + P.G[(i + 1) * 4 + 1] * f[1] +
                 P.G[(i + 1) * 4 + 2] * f[2] + P.G[(i + 1) * 4 + 3] * f[3];
}

// ---- opt-in first-order motor lag (north_star; absent in the reference) ----
// Rotor thrusts f_i follow the commanded thrusts u_i (held over the tick):
// f' = (u - f) / tau_m, integrated exactly: f(t0 + s) = u + (f(t0) - u) e^(-s/tau_m).
// u = the mixer's clamped motor thrusts (quad.py:143-168), or k_t clip(rpm)^2
// for MOTOR rows (quad.py:130-140).  The rigid body integrates (rk4_inplace,
// wrench held) G fbar, fbar = u + (f(t0) - u) phi the tick-mean thrust,
// phi = (tau_m / dt)(1 - e^(-dt/tau_m)): exact thrust impulse per tick, and
// tau_m -> 0 recovers the reference's instantaneous mixer.

// clamped mixer motor thrusts m = clip(G^-1 [f_c, tau], 0, f_max) (quad.py:153-160)
template <class T>
__device__ __forceinline__ void mix_motors(T f_c, const T tau[3], const swarmstep_quad_params &P, const Derived &D,
                                           T m[4])
{
    const T A = mul(bc<T>(P.G_inv[1]), tau[0]), C = mul(bc<T>(P.G_inv[3]), tau[2]);
    const T c0 = bc<T>(P.G_inv[0]), c2 = bc<T>(D.g_inv2_abs);
    const T FpA = fma(c0, f_c, A), FmA = fma(c0, f_c, neg(A)), BmC = fma(c2, tau[1], neg(C)), BpC = fma(c2, tau[1], C);
    m[0] = sub(FpA, BmC); m[1] = sub(FmA, BpC); m[2] = add(FmA, BpC); m[3] = add(FpA, BmC);
#pragma unroll
    for (int i = 0; i < 4; i++) m[i] = clip(m[i], bc<T>(0.0f), bc<T>(P.f_max));
}

// wrench of four rotor thrusts: (f_c, tau) = G f (quad.py:138-140)
template <class T>
__device__ __forceinline__ void thrust_wrench(const T f[4], const swarmstep_quad_params &P, T &f_c, T tau[3])
{
    f_c = add(add(f[0], f[1]), add(f[2], f[3]));
#pragma unroll
    for (int i = 0; i < 3; i++)
        tau[i] = fma(bc<T>(P.G[(i + 1) * 4 + 0]), f[0], fma(bc<T>(P.G[(i + 1) * 4 + 1]), f[1],
                 fma(bc<T>(P.G[(i + 1) * 4 + 2]), f[2], mul(bc<T>(P.G[(i + 1) * 4 + 3]), f[3]))));
}

// rotor thrusts lagging towards u: u + (f - u) e (e = e^(-dt/tau_m) for the
// end of the tick, e = phi for the tick mean)
template <class T>
__device__ __forceinline__ void lag_thrust(const T f[4], const T u[4], T e, T out[4])
{
#pragma unroll
    for (int i = 0; i < 4; i++) out[i] = fma(sub(f[i], u[i]), e, u[i]);
}

// rate_pid_step for alive rows (control.py:136-187).  Dead rows never reach
// this (they are frozen: tau = 0, f_c = 0, state untouched).  A row without a
// previous sample has no D term (control.py:175-177): the caller sets
// prev := w for it before the first tick, making the difference exactly 0.
template <bool AXI = false, class T>
__device__ __forceinline__ void pid_row(const T w[3], const T w_sp[3], const swarmstep_quad_params &P,
                                        const Derived &D, float dt, T integ[3], T prev[3], T tau[3])
{
#pragma unroll
    for (int a = 0; a < 3; a++) {
        const T e = sub(w_sp[a], w[a]);
        // min/max clamp: a NaN error (NaN rate command) faults the row this
        // tick regardless (tau is NaN), so NaN need not be kept in the state
        const int c = axc<AXI>(a);
        integ[a] = vmin(vmax(fma(bc<T>(dt), e, integ[a]), bc<T>(D.neg_i_limit[c])), bc<T>(P.i_limit[c]));
        const T t = fma(bc<T>(P.kp[c]), e, mul(bc<T>(P.ki[c]), integ[a]));
        tau[a] = fnma(bc<T>(D.kd_dt[c]), sub(w[a], prev[a]), t);
        prev[a] = w[a];
    }
}

// 2 atan2(s, c) / s for s, c >= 0 (the axis-angle factor of control.py:283-285),
// finite at s = 0 (-> 2/c): atan(t) = t P(t^2) on [0, 1], degree-8 minimax.
// e0 < 0: the reference flips q_err to w >= 0 first (control.py:280-282),
// which negates the axis -- folded into the factor's constant 2.
template <class T>
__device__ __forceinline__ T axis_angle_factor(T s, T c, T e0)
{
    const mask_t<T> small = le(s, c);
    const T num = sel(small, s, c), den = sel(small, c, s);
    const T r = rcp_a(den);
    const T t = mul(num, r);
    const T u = mul(t, t);
    T p = bc<T>(0.002846542978659272f);
    p = fma(p, u, bc<T>(-0.01605575904250145f));
    p = fma(p, u, bc<T>(0.04267148673534393f));
    p = fma(p, u, bc<T>(-0.07502678036689758f));
    p = fma(p, u, bc<T>(0.10640215128660202f));
    p = fma(p, u, bc<T>(-0.14203472435474396f));
    p = fma(p, u, bc<T>(0.1999259889125824f));
    p = fma(p, u, bc<T>(-0.3333307206630707f));
    p = fma(p, u, bc<T>(1.0f));
    // small: atan2 = t p, factor = 2 t p / s = 2 p / c
    // large: atan2 = pi/2 - t p, factor = 2 (pi/2 - t p) / s
    const T big = fnma(t, p, bc<T>(1.5707963267948966f));
    const T two = sel(lt(e0, bc<T>(0.0f)), bc<T>(-2.0f), bc<T>(2.0f));
    return mul(mul(two, sel(small, p, big)), r);
}

// _rotmats_to_quats (control.py:190-213) for the desired frame R = [x y z],
// x = y x z, up to a positive scale: branch 0 (tr > 0), 1 (m00 largest),
// 2 (m11 >= m22) or 3; branch k has t = 1 + (+-m00 +- m11 +- m22), s =
// 2 sqrt(t), its own component s/4 and the others (m_ij +- m_ji)/s.  Any
// positive scale of q_des leaves the outer loop's result unchanged (q_err is
// linear in q_des and the axis-angle vector is scale invariant), so the
// branch quaternion is formed scaled by s -- (t, m_ij +- m_ji) -- with no
// square root.
template <class T>
__device__ __forceinline__ void frame_quat(const T yd[3], const T z[3], T qd[4])
{
    const T zero = bc<T>(0.0f), one = bc<T>(1.0f);
    const T m00 = fnma(yd[2], z[1], mul(yd[1], z[2]));
    const T m10 = fnma(yd[0], z[2], mul(yd[2], z[0]));
    const T m20 = fnma(yd[1], z[0], mul(yd[0], z[1]));
    const T m01 = yd[0], m11 = yd[1], m21 = yd[2];
    const T m02 = z[0], m12 = z[1], m22 = z[2];
    const T tr = add(add(m00, m11), m22);
    const mask_t<T> b0 = gt(tr, zero);
    const mask_t<T> b1 = mand(mnot(b0), mand(ge(m00, m11), ge(m00, m22)));
    const mask_t<T> b2 = mand(mand(mnot(b0), mnot(b1)), ge(m11, m22));
    const mask_t<T> b3 = mand(mand(mnot(b0), mnot(b1)), mnot(b2));
    const T s00 = sel(mor(b0, b1), m00, neg(m00));
    const T s11 = sel(mor(b0, b2), m11, neg(m11));
    const T s22 = sel(mor(b0, b3), m22, neg(m22));
    const T t = vmax(add(add(add(one, s00), s11), s22), bc<T>(1e-30f));
    const T d21 = sub(m21, m12), d02 = sub(m02, m20), d10 = sub(m10, m01);
    const T a01 = add(m01, m10), a02 = add(m02, m20), a12 = add(m12, m21);
    qd[0] = sel(b0, t, sel(b1, d21, sel(b2, d02, d10)));
    qd[1] = sel(b1, t, sel(b0, d21, sel(b2, a01, a02)));
    qd[2] = sel(b2, t, sel(b0, d02, sel(b1, a01, a12)));
    qd[3] = sel(b3, t, sel(b0, d10, sel(b1, a02, a12)));
}

// Desired quaternion of the degenerate-heading fallback (control.py:256-262):
// x_alt = y_c x z with y_c = (-sy, cy, 0); y = z x x_alt / |x_alt|.
template <class T>
__device__ __forceinline__ void fallback_quat(const T z[3], T cy, T sy, T qd[4])
{
    const T xa0 = mul(cy, z[2]), xa1 = mul(sy, z[2]), xa2 = fnma(sy, z[1], neg(mul(cy, z[0])));
    const T ix = rsqrt_a(fma(xa0, xa0, fma(xa1, xa1, mul(xa2, xa2))));
    const T x0 = mul(xa0, ix), x1 = mul(xa1, ix), x2 = mul(xa2, ix);
    T yd[3];
    yd[0] = fnma(z[2], x1, mul(z[1], x2));
    yd[1] = fnma(z[0], x2, mul(z[2], x0));
    yd[2] = fnma(z[1], x0, mul(z[0], x1));
    frame_quat(yd, z, qd);
}

// position_outer_loop for alive rows (control.py:222-294): PD position loop
// -> desired frame (z_des, yaw) with the degenerate-heading fallback ->
// desired quaternion (control.py:190-213) -> axis-angle attitude error ->
// clipped rate setpoint.  cy / sy = cos / sin(yaw_sp) and ch / sh =
// cos / sin(yaw_sp / 2) are hoisted by the caller (per launch).
//
// The desired frame (x_c = (cy, sy, 0), y = z x x_c / |z x x_c|, x = y x z)
// is R = Rz(yaw) Rx(phi) Ry(theta): its y axis Rz Rx e_y is orthogonal to
// x_c = Rz e_x, and with z' = Rz(-yaw) z = (sin th, -sin ph cos th,
// cos ph cos th) the angles come from z' directly (cos th = |z x x_c|).  So
// q_des = q_z(yaw) (x) q_x(phi) (x) q_y(theta) in closed form, each factor
// from its (cos, sin) pair by the half-angle identity up to a positive scale
// -- (1 + c, s) or (s, 1 - c) -- instead of building R and selecting a
// branch of _rotmats_to_quats: the same rotation, 21 FP32 operations and
// three selects instead of 27 and ~24 selects / compares per agent-tick.
template <bool AXI = false, class T>
__device__ __forceinline__ void outer_row(const T p_err[3], const T v[3], const T q[4], const T v_sp[3],
                                          T cy, T sy, T ch, T sh, const swarmstep_quad_params &P,
                                          const Derived &D, T w_sp[3], T &f_c_sp, T S[3])
{
    const T zero = bc<T>(0.0f), one = bc<T>(1.0f);
    T a[3], z[3];
#pragma unroll
    for (int i = 0; i < 3; i++)
        a[i] = fma(bc<T>(P.kp_pos[axc<AXI>(i)]), p_err[i], mul(bc<T>(P.kv[axc<AXI>(i)]), sub(v_sp[i], v[i])));
    a[2] = add(a[2], bc<T>(P.g));
    const T asq = fma(a[0], a[0], fma(a[1], a[1], mul(a[2], a[2])));
    const T qw = q[0], qx = q[1], qy = q[2], qz = q[3];
    // body z axis R(q) e_z = (2 S0, 2 S1, 1 - 2 S2); the RK4's first stage
    // reuses S (same quaternion)
    thrust_terms(q, S);
    // free-fall floor (control.py:243-247): |a| < a_min -> z_des = e_z, |a| := a_min;
    // else m |a| (z_body . a/|a|) = m (z_body . a) = m (a2 + 2 (S0 a0 + S1 a1 - S2 a2))
    const mask_t<T> low = lt(asq, bc<T>(D.amin_sq));
    const T ia = rsqrt_a(asq);
    z[0] = sel(low, zero, mul(a[0], ia));
    z[1] = sel(low, zero, mul(a[1], ia));
    z[2] = sel(low, one, mul(a[2], ia));
    const T za = fma(S[0], a[0], fnma(S[2], a[2], mul(S[1], a[1])));
    const T fc = sel(low, fnma(bc<T>(D.two_m_amin), S[2], bc<T>(D.m_amin)),
                     fma(bc<T>(D.two_m), za, mul(bc<T>(P.m), a[2])));
    f_c_sp = vmin(vmax(fc, zero), bc<T>(P.fc_max));

    // z in the yaw frame; |z x x_c|^2 = z'1^2 + z'2^2 = cos^2 th
    const T zp0 = fma(cy, z[0], mul(sy, z[1]));
    const T nzp1 = fnma(cy, z[1], mul(sy, z[0]));      // -z'1 = cos th sin ph
    const T zp2 = z[2];
    const T nysq = fma(nzp1, nzp1, mul(zp2, zp2));
    const T ct = sqrt_a(nysq);
    // roll: cos th (1 + cos ph, sin ph) while z'2 >= 0, else cos th (sin ph, 1 - cos ph)
    const mask_t<T> up = ge(zp2, zero);
    const T ax = sel(up, add(ct, zp2), nzp1);
    const T bx = sel(up, nzp1, sub(ct, zp2));
    // pitch: (1 + cos th, sin th), cos th >= 0
    const T ay = add(one, ct), by = zp0;
    // q_err = conj(q) (x) q_des (quat.py:75-92) with q_des = q_z (x) q_x (x) q_y,
    // multiplied left to right: each factor has two non-zero components
    T e0, e1, e2, e3;
    {
        // conj(q) (x) (ch, 0, 0, sh)
        const T p0 = fma(qw, ch, mul(qz, sh)), p1 = fnma(qx, ch, neg(mul(qy, sh)));
        const T p2 = fma(qx, sh, neg(mul(qy, ch))), p3 = fnma(qz, ch, mul(qw, sh));
        // (x) (ax, bx, 0, 0)
        const T t0 = fnma(bx, p1, mul(ax, p0)), t1 = fma(bx, p0, mul(ax, p1));
        const T t2 = fma(bx, p3, mul(ax, p2)), t3 = fnma(bx, p2, mul(ax, p3));
        // (x) (ay, 0, by, 0)
        e0 = fnma(by, t2, mul(ay, t0));
        e1 = fnma(by, t3, mul(ay, t1));
        e2 = fma(by, t0, mul(ay, t2));
        e3 = fma(by, t1, mul(ay, t3));
    }
    const mask_t<T> degen = mnot(ge(nysq, bc<T>(1e-12f)));
    if (any(degen)) {
        T qa[4];
        fallback_quat(z, cy, sy, qa);
        e0 = sel(degen, fma(qw, qa[0], fma(qx, qa[1], fma(qy, qa[2], mul(qz, qa[3])))), e0);
        e1 = sel(degen, fma(qw, qa[1], fnma(qx, qa[0], fnma(qy, qa[3], mul(qz, qa[2])))), e1);
        e2 = sel(degen, fma(qw, qa[2], fma(qx, qa[3], fnma(qy, qa[0], neg(mul(qz, qa[1]))))), e2);
        e3 = sel(degen, fma(qw, qa[3], fnma(qx, qa[2], fnma(qz, qa[0], mul(qy, qa[1])))), e3);
    }
    // the w >= 0 flip of q_err becomes |e_w| and a sign on the rate setpoint
    const T ssq = fma(e1, e1, fma(e2, e2, mul(e3, e3)));
    const T factor = axis_angle_factor(sqrt_a(ssq), vabs(e0), e0);
    // |w_sp| <= omega_sp_max, NaN propagating (np.clip): a NaN setpoint that
    // reached the device (the bulk feed does not screen) faults its row
    // through the PID and RK4 instead of flying a clamped garbage command
    const T wm = bc<T>(P.omega_sp_max), nwm = bc<T>(D.neg_w_sp_max);
    w_sp[0] = vmin_nan(vmax_nan(mul(bc<T>(P.k_att[0]), mul(e1, factor)), nwm), wm);
    w_sp[1] = vmin_nan(vmax_nan(mul(bc<T>(P.k_att[axc<AXI>(1)]), mul(e2, factor)), nwm), wm);
    w_sp[2] = vmin_nan(vmax_nan(mul(bc<T>(P.k_att[2]), mul(e3, factor)), nwm), wm);
}

}  // namespace ssb
