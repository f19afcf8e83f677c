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
    d.gx = (P.izz - P.iyy) * P.inv_ixx;
    d.gy = (P.ixx - P.izz) * P.inv_iyy;
    d.gz = (P.iyy - P.ixx) * P.inv_izz;
#pragma unroll
    for (int i = 0; i < 3; i++) d.kd_dt[i] = P.kd[i] * inv_dt;
    return d;
}

// d/dt of (v, q, w) at (q, w) for a held wrench (quad.py:222-310):
//   vdot = (f_c/m) R(q) e_z - g e_z ; qdot = q (x) (0, w) / 2 ;
//   wdot = I^-1 (tau - w x (I w)) = tau/I - (gyro coefficient) w_j w_k.
// fc2 = 2 f_c / m, fcg = f_c / m - g, tI = tau / I (per axis).
__device__ __forceinline__ void deriv(const float q[4], const float w[3], float fc2, float fcg,
                                      const float tI[3], const Derived &D,
                                      float dv[3], float dq[4], float dw[3])
{
    const float qw = q[0], qx = q[1], qy = q[2], qz = q[3];
    const float hx = 0.5f * w[0], hy = 0.5f * w[1], hz = 0.5f * w[2];
    dv[0] = fc2 * fmaf(qx, qz, qw * qy);
    dv[1] = fc2 * fmaf(qy, qz, -qw * qx);
    dv[2] = fmaf(-fc2, fmaf(qx, qx, qy * qy), fcg);
    dq[0] = -fmaf(qx, hx, fmaf(qy, hy, qz * hz));
    dq[1] = fmaf(qw, hx, fmaf(qy, hz, -qz * hy));
    dq[2] = fmaf(qw, hy, fmaf(qz, hx, -qx * hz));
    dq[3] = fmaf(qw, hz, fmaf(qx, hy, -qy * hx));
    dw[0] = fmaf(-D.gx, w[1] * w[2], tI[0]);
    dw[1] = fmaf(-D.gy, w[2] * w[0], tI[1]);
    dw[2] = fmaf(-D.gz, w[0] * w[1], tI[2]);
}

__device__ __forceinline__ void two_sum(float a, float b, float &s, float &e)
{
    s = a + b;
    const float bb = s - a;
    e = (a - (s - bb)) + (b - bb);
}

// One classical RK4 step with the wrench held (quad.py:350-437).  Writes the
// candidate state into the *_n arrays and returns true when the row stays
// finite (the reference's fault predicate, quad.py:404-430).  Position does
// not feed any derivative, so only its final combination is formed.
__device__ __forceinline__ bool rk4_row(const float p_hi[3], const float p_lo[3], const float v[3],
                                        const float q[4], const float w[3], float f_c,
                                        const float tau[3], const swarmstep_quad_params &P,
                                        const Derived &D, float dt, bool compensated,
                                        float p_hi_n[3], float p_lo_n[3], float v_n[3],
                                        float q_n[4], float w_n[3])
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

    deriv(q, w, fc2, fcg, tI, D, kv, kq, kw);                       // k1
#pragma unroll
    for (int i = 0; i < 3; i++) { av[i] = kv[i]; aw[i] = kw[i]; ap[i] = v[i]; }
#pragma unroll
    for (int i = 0; i < 4; i++) aq[i] = kq[i];
#pragma unroll
    for (int s = 0; s < 2; s++) {                                   // k2, k3 at y + h/2 k
#pragma unroll
        for (int i = 0; i < 3; i++) { sv[i] = fmaf(half, kv[i], v[i]); sw[i] = fmaf(half, kw[i], w[i]); }
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
    for (int i = 0; i < 3; i++) { sv[i] = fmaf(dt, kv[i], v[i]); sw[i] = fmaf(dt, kw[i], w[i]); }
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
        v_n[i] = fmaf(h6, av[i], v[i]);
        w_n[i] = fmaf(h6, aw[i], w[i]);
        const float dp = h6 * ap[i];
        if (compensated) {
            float s, e;
            two_sum(p_hi[i], dp + p_lo[i], s, e);
            const float hi2 = s + e;          // renormalise: |lo| <= ulp(hi)/2
            p_lo_n[i] = e - (hi2 - s);
            p_hi_n[i] = hi2;
        } else {
            p_hi_n[i] = p_hi[i] + dp;
            p_lo_n[i] = 0.0f;
        }
    }
#pragma unroll
    for (int i = 0; i < 4; i++) q_n[i] = fmaf(h6, aq[i], q[i]);

    // single post-step renormalisation; zero / non-finite norm is a fault
    const float nsq = fmaf(q_n[0], q_n[0], fmaf(q_n[1], q_n[1], fmaf(q_n[2], q_n[2], q_n[3] * q_n[3])));
    const float inv = rsqrt_a(nsq);
    bool ok = isfinite(nsq) && nsq > 0.0f;
#pragma unroll
    for (int i = 0; i < 4; i++) q_n[i] *= inv;
    // 0 * x is NaN exactly when x is inf / NaN (IEEE; no fast-math here), so
    // one compare covers every position / velocity / rate component
    const float chk = 0.0f * (((p_hi_n[0] + p_hi_n[1]) + (p_hi_n[2] + p_lo_n[0])) +
                              ((p_lo_n[1] + p_lo_n[2]) + (v_n[0] + v_n[1])) +
                              ((v_n[2] + w_n[0]) + (w_n[1] + w_n[2])));
    ok = ok && (chk == 0.0f);
    return ok;
}

// mix_to_motors (quad.py:143-168): realized wrench after per-motor clamp.
__device__ __forceinline__ void mix_row(float &f_c, float tau[3], const swarmstep_quad_params &P)
{
    const float w4[4] = {f_c, tau[0], tau[1], tau[2]};
    float m[4];
    bool sat = false;
#pragma unroll
    for (int i = 0; i < 4; i++) {
        m[i] = fmaf(P.G_inv[i * 4 + 0], w4[0], fmaf(P.G_inv[i * 4 + 1], w4[1],
               fmaf(P.G_inv[i * 4 + 2], w4[2], P.G_inv[i * 4 + 3] * w4[3])));
        sat = sat || (m[i] < 0.0f) || (m[i] > P.f_max);
    }
    if (sat) {
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
                                        float integ[3], float prev[3], bool &has_prev, float tau[3])
{
#pragma unroll
    for (int a = 0; a < 3; a++) {
        const float e = w_sp[a] - w[a];
        integ[a] = clip(fmaf(e, dt, integ[a]), -P.i_limit[a], P.i_limit[a]);
        float t = fmaf(P.kp[a], e, P.ki[a] * integ[a]);
        if (has_prev) t = fmaf(-D.kd_dt[a], w[a] - prev[a], t);
        tau[a] = t;
        prev[a] = w[a];
    }
    has_prev = true;
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
    f_c_sp = clip(fc, 0.0f, P.fc_max);

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
    const float t = fmaxf(1.0f + s00 + s11 + s22, 1e-30f);
    const float rt = rsqrt_a(t);
    const float big = 0.5f * (t * rt), hr = 0.5f * rt;
    const float d21 = m21 - m12, d02 = m02 - m20, d10 = m10 - m01;
    const float a01 = m01 + m10, a02 = m02 + m20, a12 = m12 + m21;
    float qd[4];
    qd[0] = b0 ? big : hr * (b1 ? d21 : (b2 ? d02 : d10));
    qd[1] = b1 ? big : hr * (b0 ? d21 : (b2 ? a01 : a02));
    qd[2] = b2 ? big : hr * (b0 ? d02 : (b1 ? a01 : a12));
    qd[3] = b3 ? big : hr * (b0 ? d10 : (b1 ? a02 : a12));
    {
        const float in = rsqrt_a(fmaf(qd[0], qd[0], fmaf(qd[1], qd[1], fmaf(qd[2], qd[2], qd[3] * qd[3]))));
        qd[0] *= in; qd[1] *= in; qd[2] *= in; qd[3] *= in;
    }
    // q_err = conj(q) (x) q_des, renormalised (quat.py:75-92), sign so w >= 0
    float e0 = fmaf(qw, qd[0], fmaf(qx, qd[1], fmaf(qy, qd[2], qz * qd[3])));
    float e1 = fmaf(qw, qd[1], fmaf(-qx, qd[0], fmaf(-qy, qd[3], qz * qd[2])));
    float e2 = fmaf(qw, qd[2], fmaf(qx, qd[3], fmaf(-qy, qd[0], -qz * qd[1])));
    float e3 = fmaf(qw, qd[3], fmaf(-qx, qd[2], fmaf(qy, qd[1], -qz * qd[0])));
    {
        float in = rsqrt_a(fmaf(e0, e0, fmaf(e1, e1, fmaf(e2, e2, e3 * e3))));
        in = e0 < 0.0f ? -in : in;
        e0 *= in; e1 *= in; e2 *= in; e3 *= in;
    }
    const float ssq = fmaf(e1, e1, fmaf(e2, e2, e3 * e3));
    const float factor = axis_angle_factor(sqrt_a(ssq), e0);
    w_sp[0] = clip(P.k_att[0] * (e1 * factor), -P.omega_sp_max, P.omega_sp_max);
    w_sp[1] = clip(P.k_att[1] * (e2 * factor), -P.omega_sp_max, P.omega_sp_max);
    w_sp[2] = clip(P.k_att[2] * (e3 * factor), -P.omega_sp_max, P.omega_sp_max);
}

}  // namespace ssb
