// quad_math.cuh -- per-agent float32 device math for the quadrotor hot path.
//
// Each function restates one piece of the reference's batched numpy path for
// a single agent held in registers:
//   deriv            quad.py:222-310   (_deriv_kernel)
//   rk4_row          quad.py:350-437   (rk4_step, one row)
//   mix_row          quad.py:143-168   (mix_to_motors)
//   motor_wrench     quad.py:130-140 + core.py:189-197
//   pid_row          control.py:136-187 (rate_pid_step)
//   outer_row        control.py:190-294 (position_outer_loop, _rotmats_to_quats)
//
// Numerics (float32 against the float64 reference):
//  * clamps are written as compare-selects so NaN propagates like np.clip;
//  * the mixer returns the requested wrench unchanged for unsaturated rows
//    (G * G^-1 * w == w exactly in R; the reference's float64 round trip
//    differs by ~1 ulp, a float32 round trip would inject |f_c| * eps32 of
//    torque error -- SURVEY.md Appendix B);
//  * position may be carried as an unevaluated sum hi + lo (TwoSum update),
//    so that the float64 reference's sub-ulp increments at |p| ~ 100 m are
//    kept.
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

// d/dt of (v, q, w); p-dot = v is handled by the caller.
// fc_m = f_c / m.  quad.py:222-310.
__device__ __forceinline__ void deriv(const float q[4], const float w[3], float fc_m,
                                      const float tau[3], const swarmstep_quad_params &P,
                                      float dv[3], float dq[4], float dw[3])
{
    const float qw = q[0], qx = q[1], qy = q[2], qz = q[3];
    const float ox = w[0], oy = w[1], oz = w[2];
    dv[0] = 2.0f * (qx * qz + qw * qy) * fc_m;
    dv[1] = 2.0f * (qy * qz - qw * qx) * fc_m;
    dv[2] = (1.0f - 2.0f * (qx * qx + qy * qy)) * fc_m - P.g;
    dq[0] = -0.5f * (qx * ox + qy * oy + qz * oz);
    dq[1] = 0.5f * (qw * ox + qy * oz - qz * oy);
    dq[2] = 0.5f * (qw * oy + qz * ox - qx * oz);
    dq[3] = 0.5f * (qw * oz + qx * oy - qy * ox);
    // I^-1 (tau - w x (I w)), diagonal inertia
    dw[0] = (tau[0] - (oy * (P.izz * oz) - oz * (P.iyy * oy))) * P.inv_ixx;
    dw[1] = (tau[1] - (oz * (P.ixx * ox) - ox * (P.izz * oz))) * P.inv_iyy;
    dw[2] = (tau[2] - (ox * (P.iyy * oy) - oy * (P.ixx * ox))) * P.inv_izz;
}

__device__ __forceinline__ void two_sum(float a, float b, float &s, float &e)
{
    s = a + b;
    float bb = s - a;
    e = (a - (s - bb)) + (b - bb);
}

// One classical RK4 step with the wrench held (quad.py:350-437).  Writes the
// candidate state into the *_n arrays and returns true when the row stays
// finite (the reference's fault predicate, quad.py:404-430).
__device__ __forceinline__ bool rk4_row(const float p_hi[3], const float p_lo[3], const float v[3],
                                        const float q[4], const float w[3], float f_c,
                                        const float tau[3], const swarmstep_quad_params &P,
                                        float dt, bool compensated,
                                        float p_hi_n[3], float p_lo_n[3], float v_n[3],
                                        float q_n[4], float w_n[3])
{
    const float half = 0.5f * dt;
    const float h6 = dt * (1.0f / 6.0f);
    const float fc_m = f_c * P.inv_m;
    float kv[3], kq[4], kw[3];
    float av[3], aq[4], aw[3], ap[3];
    float sv[3], sq[4], sw[3];

    // k1
    deriv(q, w, fc_m, tau, P, kv, kq, kw);
#pragma unroll
    for (int i = 0; i < 3; i++) { av[i] = kv[i]; aw[i] = kw[i]; ap[i] = v[i]; }
#pragma unroll
    for (int i = 0; i < 4; i++) aq[i] = kq[i];
    // k2 at y + h/2 k1
#pragma unroll
    for (int i = 0; i < 3; i++) { sv[i] = fmaf(half, kv[i], v[i]); sw[i] = fmaf(half, kw[i], w[i]); }
#pragma unroll
    for (int i = 0; i < 4; i++) sq[i] = fmaf(half, kq[i], q[i]);
#pragma unroll
    for (int i = 0; i < 3; i++) ap[i] = fmaf(2.0f, sv[i], ap[i]);
    deriv(sq, sw, fc_m, tau, P, kv, kq, kw);
#pragma unroll
    for (int i = 0; i < 3; i++) { av[i] = fmaf(2.0f, kv[i], av[i]); aw[i] = fmaf(2.0f, kw[i], aw[i]); }
#pragma unroll
    for (int i = 0; i < 4; i++) aq[i] = fmaf(2.0f, kq[i], aq[i]);
    // k3 at y + h/2 k2
#pragma unroll
    for (int i = 0; i < 3; i++) { sv[i] = fmaf(half, kv[i], v[i]); sw[i] = fmaf(half, kw[i], w[i]); }
#pragma unroll
    for (int i = 0; i < 4; i++) sq[i] = fmaf(half, kq[i], q[i]);
#pragma unroll
    for (int i = 0; i < 3; i++) ap[i] = fmaf(2.0f, sv[i], ap[i]);
    deriv(sq, sw, fc_m, tau, P, kv, kq, kw);
#pragma unroll
    for (int i = 0; i < 3; i++) { av[i] = fmaf(2.0f, kv[i], av[i]); aw[i] = fmaf(2.0f, kw[i], aw[i]); }
#pragma unroll
    for (int i = 0; i < 4; i++) aq[i] = fmaf(2.0f, kq[i], aq[i]);
    // k4 at y + h k3
#pragma unroll
    for (int i = 0; i < 3; i++) { sv[i] = fmaf(dt, kv[i], v[i]); sw[i] = fmaf(dt, kw[i], w[i]); }
#pragma unroll
    for (int i = 0; i < 4; i++) sq[i] = fmaf(dt, kq[i], q[i]);
#pragma unroll
    for (int i = 0; i < 3; i++) ap[i] += sv[i];
    deriv(sq, sw, fc_m, tau, P, kv, kq, kw);
#pragma unroll
    for (int i = 0; i < 3; i++) { av[i] += kv[i]; aw[i] += kw[i]; }
#pragma unroll
    for (int i = 0; i < 4; i++) aq[i] += kq[i];

    // combine: y' = y + dt/6 (k1 + 2k2 + 2k3 + k4)
#pragma unroll
    for (int i = 0; i < 3; i++) {
        v_n[i] = fmaf(h6, av[i], v[i]);
        w_n[i] = fmaf(h6, aw[i], w[i]);
        const float dp = h6 * ap[i];
        if (compensated) {
            float s, e;
            two_sum(p_hi[i], dp + p_lo[i], s, e);
            // renormalise so |lo| <= ulp(hi)/2
            float hi2 = s + e;
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
    const float nsq = q_n[0] * q_n[0] + q_n[1] * q_n[1] + q_n[2] * q_n[2] + q_n[3] * q_n[3];
    const float nrm = sqrtf(nsq);
    bool ok = isfinite(nrm) && nrm > 0.0f;
    const float inv = 1.0f / nrm;
#pragma unroll
    for (int i = 0; i < 4; i++) q_n[i] *= inv;
#pragma unroll
    for (int i = 0; i < 3; i++)
        ok = ok && isfinite(p_hi_n[i] + p_lo_n[i]) && isfinite(v_n[i]) && isfinite(w_n[i]);
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
        m[i] = P.G_inv[i * 4 + 0] * w4[0] + P.G_inv[i * 4 + 1] * w4[1] +
               P.G_inv[i * 4 + 2] * w4[2] + P.G_inv[i * 4 + 3] * w4[3];
        sat = sat || (m[i] < 0.0f) || (m[i] > P.f_max);
    }
    if (sat) {
#pragma unroll
        for (int i = 0; i < 4; i++) m[i] = clip(m[i], 0.0f, P.f_max);
        f_c = P.G[0] * m[0] + P.G[1] * m[1] + P.G[2] * m[2] + P.G[3] * m[3];
#pragma unroll
        for (int i = 0; i < 3; i++)
            tau[i] = P.G[(i + 1) * 4 + 0] * m[0] + P.G[(i + 1) * 4 + 1] * m[1] +
                     P.G[(i + 1) * 4 + 2] * m[2] + P.G[(i + 1) * 4 + 3] * m[3];
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
                                        const swarmstep_quad_params &P, float dt, float inv_dt,
                                        float integ[3], float prev[3], bool &has_prev, float tau[3])
{
#pragma unroll
    for (int a = 0; a < 3; a++) {
        const float e = w_sp[a] - w[a];
        integ[a] = clip(integ[a] + e * dt, -P.i_limit[a], P.i_limit[a]);
        float t = fmaf(P.kp[a], e, P.ki[a] * integ[a]);
        if (has_prev) t -= ((w[a] - prev[a]) * inv_dt) * P.kd[a];
        tau[a] = t;
        prev[a] = w[a];
    }
    has_prev = true;
}

__device__ __forceinline__ void cross3(const float a[3], const float b[3], float c[3])
{
    c[0] = a[1] * b[2] - a[2] * b[1];
    c[1] = a[2] * b[0] - a[0] * b[2];
    c[2] = a[0] * b[1] - a[1] * b[0];
}

// position_outer_loop for one alive row (control.py:222-294) with the
// desired-attitude quaternion from the one selected branch of
// _rotmats_to_quats (control.py:190-213).  cy/sy = cos/sin(yaw_sp) are
// hoisted by the caller (constant over fused substeps).
__device__ __forceinline__ void outer_row(const float p_err[3], const float v[3], const float q[4],
                                          const float v_sp[3], float cy, float sy,
                                          const swarmstep_quad_params &P,
                                          float w_sp[3], float &f_c_sp)
{
    float a[3], z[3];
#pragma unroll
    for (int i = 0; i < 3; i++) a[i] = fmaf(P.kp_pos[i], p_err[i], P.kv[i] * (v_sp[i] - v[i]));
    a[2] += P.g;
    const float an = sqrtf(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]);
    const bool low = an < P.a_cmd_min;
    const float eff = low ? P.a_cmd_min : an;   // np.maximum; NaN stays NaN
    if (low) {
        z[0] = 0.0f; z[1] = 0.0f; z[2] = 1.0f;
    } else {
        const float ie = 1.0f / eff;
        z[0] = a[0] * ie; z[1] = a[1] * ie; z[2] = a[2] * ie;
    }
    const float qw = q[0], qx = q[1], qy = q[2], qz = q[3];
    const float zb0 = 2.0f * (qx * qz + qw * qy);
    const float zb1 = 2.0f * (qy * qz - qw * qx);
    const float zb2 = 1.0f - 2.0f * (qx * qx + qy * qy);
    f_c_sp = clip(P.m * eff * (zb0 * z[0] + zb1 * z[1] + zb2 * z[2]), 0.0f, P.fc_max);

    // desired frame: y = z x x_c / |.|, degenerate fallback from y_c
    float yd[3], xd[3];
    const float xc[3] = {cy, sy, 0.0f};
    float yr[3];
    cross3(z, xc, yr);
    const float ny = sqrtf(yr[0] * yr[0] + yr[1] * yr[1] + yr[2] * yr[2]);
    if (!(ny < 1e-6f)) {
        const float iy = 1.0f / ny;
        yd[0] = yr[0] * iy; yd[1] = yr[1] * iy; yd[2] = yr[2] * iy;
    } else {
        const float yc[3] = {-sy, cy, 0.0f};
        float xa[3];
        cross3(yc, z, xa);
        const float ix = 1.0f / sqrtf(xa[0] * xa[0] + xa[1] * xa[1] + xa[2] * xa[2]);
        xa[0] *= ix; xa[1] *= ix; xa[2] *= ix;
        cross3(z, xa, yd);
    }
    cross3(yd, z, xd);
    // R = [xd yd z] (columns); rotmat -> quaternion, one branch
    const float m00 = xd[0], m01 = yd[0], m02 = z[0];
    const float m10 = xd[1], m11 = yd[1], m12 = z[1];
    const float m20 = xd[2], m21 = yd[2], m22 = z[2];
    const float tr = m00 + m11 + m22;
    float qd[4];
    if (tr > 0.0f) {
        const float s = sqrtf(fmaxf(tr + 1.0f, 1e-30f)) * 2.0f, is = 1.0f / s;
        qd[0] = 0.25f * s; qd[1] = (m21 - m12) * is; qd[2] = (m02 - m20) * is; qd[3] = (m10 - m01) * is;
    } else if (m00 >= m11 && m00 >= m22) {
        const float s = sqrtf(fmaxf(1.0f + m00 - m11 - m22, 1e-30f)) * 2.0f, is = 1.0f / s;
        qd[0] = (m21 - m12) * is; qd[1] = 0.25f * s; qd[2] = (m01 + m10) * is; qd[3] = (m02 + m20) * is;
    } else if (m11 >= m22) {
        const float s = sqrtf(fmaxf(1.0f + m11 - m00 - m22, 1e-30f)) * 2.0f, is = 1.0f / s;
        qd[0] = (m02 - m20) * is; qd[1] = (m01 + m10) * is; qd[2] = 0.25f * s; qd[3] = (m12 + m21) * is;
    } else {
        const float s = sqrtf(fmaxf(1.0f + m22 - m00 - m11, 1e-30f)) * 2.0f, is = 1.0f / s;
        qd[0] = (m10 - m01) * is; qd[1] = (m02 + m20) * is; qd[2] = (m12 + m21) * is; qd[3] = 0.25f * s;
    }
    {
        const float in = 1.0f / sqrtf(qd[0] * qd[0] + qd[1] * qd[1] + qd[2] * qd[2] + qd[3] * qd[3]);
        qd[0] *= in; qd[1] *= in; qd[2] *= in; qd[3] *= in;
    }
    // q_err = conj(q) * q_des, renormalised (quat.py:75-92), w >= 0
    float e0 = qw * qd[0] + qx * qd[1] + qy * qd[2] + qz * qd[3];
    float e1 = qw * qd[1] - qx * qd[0] - qy * qd[3] + qz * qd[2];
    float e2 = qw * qd[2] + qx * qd[3] - qy * qd[0] - qz * qd[1];
    float e3 = qw * qd[3] - qx * qd[2] + qy * qd[1] - qz * qd[0];
    {
        float in = 1.0f / sqrtf(e0 * e0 + e1 * e1 + e2 * e2 + e3 * e3);
        if (e0 < 0.0f) in = -in;
        e0 *= in; e1 *= in; e2 *= in; e3 *= in;
    }
    const float s = sqrtf(e1 * e1 + e2 * e2 + e3 * e3);
    const float angle = 2.0f * atan2f(s, e0);
    const float factor = s > 1e-12f ? angle / s : 2.0f;
    w_sp[0] = clip(P.k_att[0] * (e1 * factor), -P.omega_sp_max, P.omega_sp_max);
    w_sp[1] = clip(P.k_att[1] * (e2 * factor), -P.omega_sp_max, P.omega_sp_max);
    w_sp[2] = clip(P.k_att[2] * (e3 * factor), -P.omega_sp_max, P.omega_sp_max);
}

}  // namespace ssb
