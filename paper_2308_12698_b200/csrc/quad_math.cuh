// quad_math.cuh -- per-agent float32 device math for the quadrotor hot path.
//
// Each function restates one piece of the reference's batched numpy path for
// a single agent held in registers:
//   deriv / rk4_row  quad.py:222-310, 350-437  (_deriv_kernel, rk4_step)
//   mix_row          quad.py:143-168           (mix_to_motors)
//   motor_wrench     quad.py:130-140 + core.py:189-197
//   pid_row          control.py:136-187        (rate_pid_step)
//   outer_row        control.py:190-294        (position_outer_loop, _rotmats_to_quats)
//
// Numerics (float32 against the float64 reference, target <= 1e-5 relative
// per step):
//  * clamps are compare-selects so NaN propagates like np.clip;
//  * the mixer returns the requested wrench unchanged for unsaturated rows
//    (G G^-1 w == w in R; a float32 round trip would inject |f_c| eps32 of
//    torque error -- SURVEY.md Appendix B);
//  * position can be carried as an unevaluated sum hi + lo (TwoSum update) so
//    the reference's sub-ulp increments at |p| ~ 100 m are kept;
//  * sqrt / 1/x / 1/sqrt use the SFU (MUFU) approximations (<= 2 ulp) and
//    atan2 a degree-8 minimax polynomial (9e-8 relative): all well inside the
//    1e-5 budget, and branch-free of the IEEE slow paths.
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include "swarmstep_b200.h"

namespace ssb {

__device__ __forceinline__ float clip(float x, float lo, float hi)
{
    // np.clip semantics: NaN passes through
    return x < lo ? lo : (x > hi ? hi : x);
}

__device__ __forceinline__ float rsqrt_a(float x)
{
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float sqrt_a(float x)
{
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float rcp_a(float x)
{
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Per-tick constants derived from the per-type struct (hoisted out of the
// substep loop by the caller).
struct Derived {
    float g;
    float gx, gy, gz;        // gyroscopic coefficients (I_zz-I_yy)/I_xx, ...
    float kd_dt[3];          // kd / dt
};

__device__ __forceinline__ Derived derive(const swarmstep_quad_params &P, float inv_dt)
{
    Derived d;
    d.g = P.g;
    d.gx = 4.0f * (P.izz - P.iyy) * P.inv_ixx;   // x4: products of half rates
    d.gy = 4.0f * (P.ixx - P.izz) * P.inv_iyy;
    d.gz = 4.0f * (P.iyy - P.ixx) * P.inv_izz;
#pragma unroll
    for (int i = 0; i < 3; i++) d.kd_dt[i] = P.kd[i] * inv_dt;
    return d;
}

// d/dt of (v, q, w) at (q, w) for a held wrench (quad.py:222-310):
//   vdot = (f_c/m) R(q) e_z - g e_z ; qdot = q (x) (0, w) / 2 ;
//   wdot = I^-1 (tau - w x (I w)) = tau/I - (gyro coefficient) w_j w_k.
// fc2 = 2 f_c / m, fcg = f_c / m - g, tI = tau / I (per axis).
// h = w / 2 is carried instead of w (saves the halving per stage); the
// gyroscopic coefficients are pre-multiplied by 4 accordingly.
__device__ __forceinline__ void deriv(const float q[4], const float h[3], float fc2, float fcg,
                                      const float tI[3], const Derived &D,
                                      float dv[3], float dq[4], float dw[3])
{
    const float qw = q[0], qx = q[1], qy = q[2], qz = q[3];
    const float hx = h[0], hy = h[1], hz = h[2];
    dv[0] = fc2 * fmaf(qx, qz, qw * qy);
    dv[1] = fc2 * fmaf(qy, qz, -qw * qx);
    dv[2] = fmaf(-fc2, fmaf(qx, qx, qy * qy), fcg);
    dq[0] = -fmaf(qx, hx, fmaf(qy, hy, qz * hz));
    dq[1] = fmaf(qw, hx, fmaf(qy, hz, -qz * hy));
    dq[2] = fmaf(qw, hy, fmaf(qz, hx, -qx * hz));
    dq[3] = fmaf(qw, hz, fmaf(qx, hy, -qy * hx));
    dw[0] = fmaf(-D.gx, hy * hz, tI[0]);
    dw[1] = fmaf(-D.gy, hz * hx, tI[1]);
    dw[2] = fmaf(-D.gz, hx * hy, tI[2]);
}

// One classical RK4 step with the wrench held (quad.py:350-437), in place.
// Returns false when the row turns non-finite (the reference's fault
// predicate, quad.py:404-430); the state is then garbage and the caller
// restores the pre-step values (by deterministic re-execution, see
// swarmstep_b200.cu).  Position feeds no derivative, so only its final
// combination is formed: dp = dt/6 (v + 2 v2 + 2 v3 + v4).
template <bool COMP>
__device__ __forceinline__ bool rk4_inplace(float p_hi[3], float p_lo[3], float v[3], float q[4],
                                            float w[3], float f_c, const float tau[3],
                                            const swarmstep_quad_params &P, const Derived &D, float dt)
{
    const float half = 0.5f * dt;
    const float h6 = dt * (1.0f / 6.0f);
    const float fcm = f_c * P.inv_m;
    const float fc2 = 2.0f * fcm;
    const float fcg = fcm - D.g;
    const float tI[3] = {tau[0] * P.inv_ixx, tau[1] * P.inv_iyy, tau[2] * P.inv_izz};
    float kv[3], kq[4], kw[3];
    float av[3], aq[4], aw[3], ap[3];
    float sv[3], sq[4], sw[3];
    const float hw[3] = {0.5f * w[0], 0.5f * w[1], 0.5f * w[2]};
    const float qtr = 0.5f * half, hdt = 0.5f * dt;  // stage steps on half rates

    deriv(q, hw, fc2, fcg, tI, D, kv, kq, kw);                      // k1
#pragma unroll
    for (int i = 0; i < 3; i++) { av[i] = kv[i]; aw[i] = kw[i]; ap[i] = v[i]; }
#pragma unroll
    for (int i = 0; i < 4; i++) aq[i] = kq[i];
#pragma unroll
    for (int s = 0; s < 2; s++) {                                   // k2, k3 at y + h/2 k
#pragma unroll
        for (int i = 0; i < 3; i++) { sv[i] = fmaf(half, kv[i], v[i]); sw[i] = fmaf(qtr, kw[i], hw[i]); }
#pragma unroll
        for (int i = 0; i < 4; i++) sq[i] = fmaf(half, kq[i], q[i]);
#pragma unroll
        for (int i = 0; i < 3; i++) ap[i] = fmaf(2.0f, sv[i], ap[i]);
        deriv(sq, sw, fc2, fcg, tI, D, kv, kq, kw);
#pragma unroll
        for (int i = 0; i < 3; i++) { av[i] = fmaf(2.0f, kv[i], av[i]); aw[i] = fmaf(2.0f, kw[i], aw[i]); }
#pragma unroll
        for (int i = 0; i < 4; i++) aq[i] = fmaf(2.0f, kq[i], aq[i]);
    }
#pragma unroll
    for (int i = 0; i < 3; i++) { sv[i] = fmaf(dt, kv[i], v[i]); sw[i] = fmaf(hdt, kw[i], hw[i]); }
#pragma unroll
    for (int i = 0; i < 4; i++) sq[i] = fmaf(dt, kq[i], q[i]);
#pragma unroll
    for (int i = 0; i < 3; i++) ap[i] += sv[i];
    deriv(sq, sw, fc2, fcg, tI, D, kv, kq, kw);                     // k4
#pragma unroll
    for (int i = 0; i < 3; i++) { av[i] += kv[i]; aw[i] += kw[i]; }
#pragma unroll
    for (int i = 0; i < 4; i++) aq[i] += kq[i];

    // y' = y + dt/6 (k1 + 2 k2 + 2 k3 + k4)
#pragma unroll
    for (int i = 0; i < 3; i++) {
        v[i] = fmaf(h6, av[i], v[i]);
        w[i] = fmaf(h6, aw[i], w[i]);
        const float dp = h6 * ap[i];
        if (COMP) {
            // Fast2Sum: exact when |hi| >= |dp + lo| (a position against one
            // tick's displacement); keeps |lo| <= ulp(hi)/2
            const float b = dp + p_lo[i];
            const float sum = p_hi[i] + b;
            p_lo[i] = b - (sum - p_hi[i]);
            p_hi[i] = sum;
        } else {
            p_hi[i] += dp;
        }
    }
#pragma unroll
    for (int i = 0; i < 4; i++) q[i] = fmaf(h6, aq[i], q[i]);

    // single post-step renormalisation; zero / non-finite norm is a fault
    const float nsq = fmaf(q[0], q[0], fmaf(q[1], q[1], fmaf(q[2], q[2], q[3] * q[3])));
    const float inv = rsqrt_a(nsq);
#pragma unroll
    for (int i = 0; i < 4; i++) q[i] *= inv;
    // 0 * x is NaN exactly when x is inf / NaN (IEEE; no fast-math here), so
    // one compare covers every position / velocity / rate component
    const float chk = 0.0f * (((p_hi[0] + p_hi[1]) + (p_hi[2] + v[0])) + ((v[1] + v[2]) + (w[0] + w[1])) +
                              (w[2] + (COMP ? (p_lo[0] + p_lo[1]) + p_lo[2] : 0.0f)));
    return isfinite(nsq) && nsq > 0.0f && chk == 0.0f;
}

// mix_to_motors (quad.py:143-168): realized wrench after per-motor clamp.
// G (quad.py:106-122) has mutually orthogonal rows, so G^-1 = G^T diag(c):
// motor i = c0 f + s_i1 c1 tau_x + s_i2 c2 tau_y + s_i3 c3 tau_z with the
// sign pattern of G's columns.  P.G_inv carries the exact inverse; the host
// checks the pattern (params.py) and the kernel uses c = |G_inv[0][:]|.
__device__ __forceinline__ void mix_row(float &f_c, float tau[3], const swarmstep_quad_params &P)
{
    const float F = P.G_inv[0] * f_c, A = P.G_inv[1] * tau[0];
    const float B = fabsf(P.G_inv[2]) * tau[1], C = P.G_inv[3] * tau[2];
    const float FpA = F + A, FmA = F - A, BmC = B - C, BpC = B + C;
    float m[4] = {FpA - BmC, FmA - BpC, FmA + BpC, FpA + BmC};
    const float lo = fminf(fminf(m[0], m[1]), fminf(m[2], m[3]));
    const float hi = fmaxf(fmaxf(m[0], m[1]), fmaxf(m[2], m[3]));
    if (lo < 0.0f || hi > P.f_max) {
#pragma unroll
        for (int i = 0; i < 4; i++) m[i] = clip(m[i], 0.0f, P.f_max);
        f_c = (m[0] + m[1]) + (m[2] + m[3]);
#pragma unroll
        for (int i = 0; i < 3; i++)
            tau[i] = fmaf(P.G[(i + 1) * 4 + 0], m[0], fmaf(P.G[(i + 1) * 4 + 1], m[1],
                     fmaf(P.G[(i + 1) * 4 + 2], m[2], P.G[(i + 1) * 4 + 3] * m[3])));
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

// rate_pid_step for one alive row (control.py:136-187).  Dead rows never
// reach this (they are frozen: tau = 0, f_c = 0, state untouched).
__device__ __forceinline__ void pid_row(const float w[3], const float w_sp[3],
                                        const swarmstep_quad_params &P, const Derived &D, float dt,
                                        float integ[3], float prev[3], float tau[3])
{
    // (no previous sample -> no D term, control.py:175-177: the caller sets
    // prev := w for such rows before the first tick, making the difference 0)
#pragma unroll
    for (int a = 0; a < 3; a++) {
        const float pv = prev[a];
        const float e = w_sp[a] - w[a];
        // min/max clamp: a NaN error (NaN rate command) faults the row this
        // tick regardless (tau is NaN), so NaN need not be kept in the state
        integ[a] = fminf(fmaxf(fmaf(e, dt, integ[a]), -P.i_limit[a]), P.i_limit[a]);
        const float t = fmaf(P.kp[a], e, P.ki[a] * integ[a]);
        tau[a] = fmaf(-D.kd_dt[a], w[a] - pv, t);
        prev[a] = w[a];
    }
}

// 2 atan2(s, c) / s for s, c >= 0 (the axis-angle factor of control.py:283-285),
// finite at s = 0 (-> 2/c): atan(t) = t P(t^2) on [0, 1], degree-8 minimax.
__device__ __forceinline__ float axis_angle_factor(float s, float c)
{
    const bool small = s <= c;
    const float num = small ? s : c, den = small ? c : s;
    const float r = rcp_a(den);
    const float t = num * r;
    const float u = t * t;
    float p = 0.002846542978659272f;
    p = fmaf(p, u, -0.01605575904250145f);
    p = fmaf(p, u, 0.04267148673534393f);
    p = fmaf(p, u, -0.07502678036689758f);
    p = fmaf(p, u, 0.10640215128660202f);
    p = fmaf(p, u, -0.14203472435474396f);
    p = fmaf(p, u, 0.1999259889125824f);
    p = fmaf(p, u, -0.3333307206630707f);
    p = fmaf(p, u, 1.0f);
    // small: atan2 = t p, factor = 2 t p / s = 2 p / c
    // large: atan2 = pi/2 - t p, factor = 2 (pi/2 - t p) / s
    return small ? 2.0f * p * r : 2.0f * fmaf(-t, p, 1.5707963267948966f) * r;
}

// position_outer_loop for one alive row (control.py:222-294): PD position
// loop -> desired frame (z_des, yaw) with the degenerate-heading fallback ->
// desired quaternion from the one selected branch of _rotmats_to_quats
// (control.py:190-213) -> axis-angle attitude error -> clipped rate setpoint.
// cy / sy = cos / sin(yaw_sp) are hoisted by the caller.
__device__ __forceinline__ void outer_row(const float p_err[3], const float v[3], const float q[4],
                                          const float v_sp[3], float cy, float sy,
                                          const swarmstep_quad_params &P,
                                          float w_sp[3], float &f_c_sp)
{
    float a[3], z[3];
#pragma unroll
    for (int i = 0; i < 3; i++) a[i] = fmaf(P.kp_pos[i], p_err[i], P.kv[i] * (v_sp[i] - v[i]));
    a[2] += P.g;
    const float asq = fmaf(a[0], a[0], fmaf(a[1], a[1], a[2] * a[2]));
    const float qw = q[0], qx = q[1], qy = q[2], qz = q[3];
    const float zb0 = 2.0f * fmaf(qx, qz, qw * qy);
    const float zb1 = 2.0f * fmaf(qy, qz, -qw * qx);
    const float zb2 = fmaf(-2.0f, fmaf(qx, qx, qy * qy), 1.0f);
    const float amin = P.a_cmd_min;
    float fc;
    if (asq < amin * amin) {            // free-fall floor: z_des = e_z, |a| := a_min
        z[0] = 0.0f; z[1] = 0.0f; z[2] = 1.0f;
        fc = P.m * amin * zb2;
    } else {                            // m |a| (z_body . a/|a|) = m (z_body . a)
        const float ia = rsqrt_a(asq);
        z[0] = a[0] * ia; z[1] = a[1] * ia; z[2] = a[2] * ia;
        fc = P.m * fmaf(zb0, a[0], fmaf(zb1, a[1], zb2 * a[2]));
    }
    f_c_sp = fminf(fmaxf(fc, 0.0f), P.fc_max);

    // y = z x x_c / |z x x_c| with x_c = (cy, sy, 0); degenerate fallback from y_c
    float yd[3];
    const float yr0 = -z[2] * sy, yr1 = z[2] * cy, yr2 = fmaf(z[0], sy, -z[1] * cy);
    const float nysq = fmaf(yr0, yr0, fmaf(yr1, yr1, yr2 * yr2));
    if (nysq >= 1e-12f) {
        const float iy = rsqrt_a(nysq);
        yd[0] = yr0 * iy; yd[1] = yr1 * iy; yd[2] = yr2 * iy;
    } else {
        // x_alt = y_c x z, y_c = (-sy, cy, 0); y = z x x_alt / |x_alt|
        const float xa0 = cy * z[2], xa1 = sy * z[2], xa2 = fmaf(-sy, z[1], -cy * z[0]);
        const float ix = rsqrt_a(fmaf(xa0, xa0, fmaf(xa1, xa1, xa2 * xa2)));
        const float x0 = xa0 * ix, x1 = xa1 * ix, x2 = xa2 * ix;
        yd[0] = fmaf(z[1], x2, -z[2] * x1);
        yd[1] = fmaf(z[2], x0, -z[0] * x2);
        yd[2] = fmaf(z[0], x1, -z[1] * x0);
    }
    // x = y x z ;  R = [x y z] (columns)
    const float m00 = fmaf(yd[1], z[2], -yd[2] * z[1]);
    const float m10 = fmaf(yd[2], z[0], -yd[0] * z[2]);
    const float m20 = fmaf(yd[0], z[1], -yd[1] * z[0]);
    const float m01 = yd[0], m11 = yd[1], m21 = yd[2];
    const float m02 = z[0], m12 = z[1], m22 = z[2];
    const float tr = m00 + m11 + m22;
    // _rotmats_to_quats selects branch 0 (tr > 0), 1 (m00 largest), 2 (m11 >=
    // m22) or 3; branch k has t = 1 + (+-m00 +- m11 +- m22), s = 2 sqrt(t), its
    // own component s/4 = sqrt(t)/2 and the others (m_ij +- m_ji)/s.  Evaluated
    // branch-free with selects (agents in a warp pick different branches).
    const bool b0 = tr > 0.0f;
    const bool b1 = !b0 && (m00 >= m11 && m00 >= m22);
    const bool b2 = !b0 && !b1 && (m11 >= m22);
    const bool b3 = !b0 && !b1 && !b2;
    const float s00 = (b0 || b1) ? m00 : -m00;
    const float s11 = (b0 || b2) ? m11 : -m11;
    const float s22 = (b0 || b3) ? m22 : -m22;
    // Any positive scale of q_des leaves the result unchanged: q_err is
    // linear in q_des, and the axis-angle vector e_xyz * 2 atan2(|e_xyz|,
    // e_w) / |e_xyz| is invariant to a positive scale of q_err.  So the
    // branch quaternion is formed scaled by s = 2 sqrt(t) -- (t, m_ij +- m_ji)
    // -- with no square root, and neither q_des nor q_err is renormalised
    // (the reference renormalises both; identical in R).
    const float t = fmaxf(1.0f + s00 + s11 + s22, 1e-30f);
    const float d21 = m21 - m12, d02 = m02 - m20, d10 = m10 - m01;
    const float a01 = m01 + m10, a02 = m02 + m20, a12 = m12 + m21;
    float qd[4];
    qd[0] = b0 ? t : (b1 ? d21 : (b2 ? d02 : d10));
    qd[1] = b1 ? t : (b0 ? d21 : (b2 ? a01 : a02));
    qd[2] = b2 ? t : (b0 ? d02 : (b1 ? a01 : a12));
    qd[3] = b3 ? t : (b0 ? d10 : (b1 ? a02 : a12));
    // q_err = conj(q) (x) q_des (quat.py:75-92); the w >= 0 flip becomes |e_w|
    // and a sign on the rate setpoint
    const float e0 = fmaf(qw, qd[0], fmaf(qx, qd[1], fmaf(qy, qd[2], qz * qd[3])));
    const float e1 = fmaf(qw, qd[1], fmaf(-qx, qd[0], fmaf(-qy, qd[3], qz * qd[2])));
    const float e2 = fmaf(qw, qd[2], fmaf(qx, qd[3], fmaf(-qy, qd[0], -qz * qd[1])));
    const float e3 = fmaf(qw, qd[3], fmaf(-qx, qd[2], fmaf(qy, qd[1], -qz * qd[0])));
    const float ssq = fmaf(e1, e1, fmaf(e2, e2, e3 * e3));
    float factor = axis_angle_factor(sqrt_a(ssq), fabsf(e0));
    factor = e0 < 0.0f ? -factor : factor;
    // |w_sp| <= omega_sp_max.  min/max (not NaN-propagating) is safe here:
    // non-finite outer-loop inputs are rejected before launch (InvalidState).
    const float wm = P.omega_sp_max;
    w_sp[0] = fminf(fmaxf(P.k_att[0] * (e1 * factor), -wm), wm);
    w_sp[1] = fminf(fmaxf(P.k_att[1] * (e2 * factor), -wm), wm);
    w_sp[2] = fminf(fmaxf(P.k_att[2] * (e3 * factor), -wm), wm);
}

}  // namespace ssb
