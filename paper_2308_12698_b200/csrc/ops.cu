// ops.cu -- the reference's function-level hot-path API on the GPU.
//
// The group kernels (swarmstep_b200.cu) fuse the whole QuadGroup.step; the
// reference also exposes each stage as a batched function that its own tests
// and callers use directly (SURVEY.md 8(b) "kernel-level functions"):
//   dynamics_deriv      quad.py:320-335     swarmstep_op_deriv
//   rk4_step            quad.py:350-437     swarmstep_op_rk4
//   mix_to_motors       quad.py:143-168     swarmstep_op_mix
//   rotor_thrust_torque quad.py:130-140     swarmstep_op_rotor
//   rate_pid_step       control.py:136-187  swarmstep_op_pid
//   position_outer_loop control.py:222-294  swarmstep_op_outer
// Same per-row math as the fused kernels (quad_math.cuh), on the reference's
// own row-major layout: (n, 3) / (n, 4) float32 arrays, u8 flags, one thread
// per row.  Positions may carry a float32 low word (pos_lo, nullable) so a
// float64 host position survives the round trip, as in the group.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "common.cuh"
#include "quad_math.cuh"

namespace {

constexpr int kT = 256;

unsigned blocks(int64_t n) { return (unsigned)((n + kT - 1) / kT); }

__device__ __forceinline__ int64_t row_id() { return (int64_t)blockIdx.x * kT + threadIdx.x; }

// dynamics_deriv: derivative of every alive row, exactly zero for dead rows
__global__ void op_deriv_kernel(int64_t n, const float *pos, const float *vel, const float *quat,
                                const float *omega, const uint8_t *alive, const float *f_c, const float *tau,
                                const swarmstep_quad_params P, const ssb::Derived D, float *dpos, float *dvel,
                                float *dquat, float *domega)
{
    const int64_t r = row_id();
    if (r >= n) return;
    float dv[3] = {0, 0, 0}, dq[4] = {0, 0, 0, 0}, dw[3] = {0, 0, 0}, dp[3] = {0, 0, 0};
    if (!alive || alive[r]) {
        const float q[4] = {quat[4 * r], quat[4 * r + 1], quat[4 * r + 2], quat[4 * r + 3]};
        const float w[3] = {omega[3 * r], omega[3 * r + 1], omega[3 * r + 2]};
        const float fc = f_c[r];
        const float fc2 = ssb::mul(fc, 2.0f * P.inv_m), fcg = ssb::fma(fc, P.inv_m, -D.g);
        const float tI[3] = {ssb::mul(tau[3 * r], P.inv_ixx), ssb::mul(tau[3 * r + 1], P.inv_iyy),
                             ssb::mul(tau[3 * r + 2], P.inv_izz)};
        ssb::deriv(q, w, fc2, fcg, tI, D, dv, dq, dw);
        for (int i = 0; i < 4; i++) dq[i] = 0.5f * dq[i];   // deriv returns 2 qdot (exact halving)
        for (int i = 0; i < 3; i++) dp[i] = vel[3 * r + i];
    }
    for (int i = 0; i < 3; i++) {
        dpos[3 * r + i] = dp[i];
        dvel[3 * r + i] = dv[i];
        domega[3 * r + i] = dw[i];
    }
    for (int i = 0; i < 4; i++) dquat[4 * r + i] = dq[i];
}

// rk4_step: one step per alive row with the wrench held; a row that turns
// non-finite keeps its pre-step state, dies and is flagged
template <bool COMP>
__global__ void op_rk4_kernel(int64_t n, float *pos, float *pos_lo, float *vel, float *quat, float *omega,
                              uint8_t *alive, const float *f_c, const float *tau, const swarmstep_quad_params P,
                              const ssb::Derived D, float dt, uint8_t *fault)
{
    const int64_t r = row_id();
    if (r >= n) return;
    fault[r] = 0;
    if (!alive[r]) return;
    float ph[3], pl[3], v[3], q[4], w[3];
    for (int i = 0; i < 3; i++) {
        ph[i] = pos[3 * r + i];
        pl[i] = COMP ? pos_lo[3 * r + i] : 0.0f;
        v[i] = vel[3 * r + i];
        w[i] = omega[3 * r + i];
    }
    for (int i = 0; i < 4; i++) q[i] = quat[4 * r + i];
    const float t[3] = {tau[3 * r], tau[3 * r + 1], tau[3 * r + 2]};
    if (!ssb::rk4_inplace<float, COMP>(ph, pl, v, q, w, f_c[r], t, P, D, dt)) {
        alive[r] = 0;
        fault[r] = 1;
        return;
    }
    for (int i = 0; i < 3; i++) {
        pos[3 * r + i] = ph[i];
        if (COMP) pos_lo[3 * r + i] = pl[i];
        vel[3 * r + i] = v[i];
        omega[3 * r + i] = w[i];
    }
    for (int i = 0; i < 4; i++) quat[4 * r + i] = q[i];
}

// mix_to_motors: clamped motor thrusts, saturation flag, realized wrench
// (the requested wrench itself for unsaturated rows: G G^-1 w == w)
__global__ void op_mix_kernel(int64_t n, const float *f_c, const float *tau, const swarmstep_quad_params P,
                              float *motors, float *realized, uint8_t *saturated)
{
    const int64_t r = row_id();
    if (r >= n) return;
    const float t[3] = {tau[3 * r], tau[3 * r + 1], tau[3 * r + 2]};
    const float A = ssb::mul(P.G_inv[1], t[0]), C = ssb::mul(P.G_inv[3], t[2]);
    const float c0 = P.G_inv[0], c2 = fabsf(P.G_inv[2]);
    const float FpA = ssb::fma(c0, f_c[r], A), FmA = ssb::fma(c0, f_c[r], -A);
    const float BmC = ssb::fma(c2, t[1], -C), BpC = ssb::fma(c2, t[1], C);
    float m[4] = {ssb::sub(FpA, BmC), ssb::sub(FmA, BpC), ssb::add(FmA, BpC), ssb::add(FpA, BmC)};
    bool sat = false;
    for (int i = 0; i < 4; i++) {
        sat = sat || m[i] < 0.0f || m[i] > P.f_max;      // NaN compares false (numpy)
        m[i] = ssb::clip(m[i], 0.0f, P.f_max);
        motors[4 * r + i] = m[i];
    }
    saturated[r] = sat;
    float w[4] = {f_c[r], t[0], t[1], t[2]};
    if (sat) {
        w[0] = ssb::add(ssb::add(m[0], m[1]), ssb::add(m[2], m[3]));
        for (int i = 0; i < 3; i++)
            w[i + 1] = ssb::fma(P.G[(i + 1) * 4 + 0], m[0], ssb::fma(P.G[(i + 1) * 4 + 1], m[1],
                       ssb::fma(P.G[(i + 1) * 4 + 2], m[2], ssb::mul(P.G[(i + 1) * 4 + 3], m[3]))));
    }
    for (int i = 0; i < 4; i++) realized[4 * r + i] = w[i];
}

// rotor_thrust_torque: k_t O^2, k_q O^2 with O clamped to [0, omega_max]
__global__ void op_rotor_kernel(int64_t n, const float *rpm, float k_t, float k_q, float omega_max, float *thrust,
                                float *torque, uint8_t *saturated)
{
    const int64_t i = row_id();
    if (i >= n) return;
    const float o = rpm[i];
    saturated[i] = (o < 0.0f) || (o > omega_max);
    const float c = ssb::clip(o, 0.0f, omega_max);
    const float sq = ssb::mul(c, c);
    thrust[i] = ssb::mul(k_t, sq);
    torque[i] = ssb::mul(k_q, sq);
}

// rate_pid_step in the reference's operation order, NaN-propagating clip of
// the integral state (np.clip), dead rows: state frozen, zero output
__global__ void op_pid_kernel(int64_t n, const float *omega, const float *omega_sp, const float *f_c_sp,
                              const swarmstep_quad_params P, float dt, float *integral, float *prev,
                              uint8_t *has_prev, const uint8_t *alive, float *tau_out, float *f_c_out)
{
    const int64_t r = row_id();
    if (r >= n) return;
    const bool a = alive[r] != 0, hp = has_prev[r] != 0;
    for (int i = 0; i < 3; i++) {
        const float w = omega[3 * r + i];
        const float e = ssb::sub(omega_sp[3 * r + i], w);
        float I = integral[3 * r + i];
        if (a) I = ssb::add(I, ssb::mul(e, dt));
        I = ssb::clip(I, -P.i_limit[i], P.i_limit[i]);
        integral[3 * r + i] = I;
        float t = ssb::add(ssb::mul(e, P.kp[i]), ssb::mul(I, P.ki[i]));
        if (a && hp) t = ssb::sub(t, ssb::mul(__fdiv_rn(ssb::sub(w, prev[3 * r + i]), dt), P.kd[i]));
        if (a) prev[3 * r + i] = w;
        tau_out[3 * r + i] = a ? t : 0.0f;
    }
    if (a) has_prev[r] = 1;
    f_c_out[r] = a ? f_c_sp[r] : 0.0f;
}

// position_outer_loop for every row (dead rows: zero setpoints, no low flag)
template <bool COMP>
__global__ void op_outer_kernel(int64_t n, const float *pos, const float *pos_lo, const float *vel,
                                const float *quat, const uint8_t *alive, const float *p_sp, const float *v_sp,
                                const float *yaw_sp, const swarmstep_quad_params P, float *omega_sp, float *f_c_sp,
                                uint8_t *low)
{
    const int64_t r = row_id();
    if (r >= n) return;
    float w_sp[3] = {0, 0, 0}, f = 0.0f;
    bool lo = false;
    if (alive[r]) {
        float pe[3], v[3], vs[3], q[4];
        for (int i = 0; i < 3; i++) {
            pe[i] = ssb::sub(p_sp[3 * r + i], pos[3 * r + i]);
            if (COMP) pe[i] = ssb::sub(pe[i], pos_lo[3 * r + i]);
            v[i] = vel[3 * r + i];
            vs[i] = v_sp[3 * r + i];
        }
        for (int i = 0; i < 4; i++) q[i] = quat[4 * r + i];
        float s, c, sh, ch;
        ssb::yaw_terms(yaw_sp[r], c, s, ch, sh);
        float S[3];
        ssb::outer_row(pe, v, q, vs, c, s, ch, sh, P, ssb::derive(P, 1.0f), w_sp, f, S);
        float asq = 0.0f;
        for (int i = 0; i < 3; i++) {
            float ai = ssb::fma(P.kp_pos[i], pe[i], ssb::mul(P.kv[i], ssb::sub(vs[i], v[i])));
            if (i == 2) ai = ssb::add(ai, P.g);
            asq = ssb::fma(ai, ai, asq);
        }
        lo = asq < P.a_cmd_min * P.a_cmd_min;
    }
    for (int i = 0; i < 3; i++) omega_sp[3 * r + i] = w_sp[i];
    f_c_sp[r] = f;
    low[r] = lo;
}

int bad(const char *m) { return ssb::set_err(SWARMSTEP_EINVAL, m); }

}  // namespace

extern "C" {

int swarmstep_op_deriv(int64_t n, const float *pos, const float *vel, const float *quat, const float *omega,
                       const uint8_t *alive, const float *f_c, const float *tau, const swarmstep_quad_params *p,
                       float *dpos, float *dvel, float *dquat, float *domega, void *stream)
{
    if (n < 0 || !p) return bad("bad arguments");
    if (n == 0) return SWARMSTEP_OK;
    if (!pos || !vel || !quat || !omega || !f_c || !tau || !dpos || !dvel || !dquat || !domega)
        return bad("null argument");
    op_deriv_kernel<<<blocks(n), kT, 0, (cudaStream_t)stream>>>(n, pos, vel, quat, omega, alive, f_c, tau, *p,
                                                                ssb::derive(*p, 1.0f), dpos, dvel, dquat, domega);
    return ssb::cuda_status("op_deriv_kernel");
}

int swarmstep_op_rk4(int64_t n, float *pos, float *pos_lo, float *vel, float *quat, float *omega, uint8_t *alive,
                     const float *f_c, const float *tau, const swarmstep_quad_params *p, float dt, uint8_t *fault,
                     void *stream)
{
    if (n < 0 || !p) return bad("bad arguments");
    if (!(dt > 0.0f)) return bad("dt must be positive");
    if (n == 0) return SWARMSTEP_OK;
    if (!pos || !vel || !quat || !omega || !alive || !f_c || !tau || !fault) return bad("null argument");
    const ssb::Derived D = ssb::derive(*p, dt);
    if (pos_lo)
        op_rk4_kernel<true><<<blocks(n), kT, 0, (cudaStream_t)stream>>>(n, pos, pos_lo, vel, quat, omega, alive,
                                                                       f_c, tau, *p, D, dt, fault);
    else
        op_rk4_kernel<false><<<blocks(n), kT, 0, (cudaStream_t)stream>>>(n, pos, nullptr, vel, quat, omega, alive,
                                                                        f_c, tau, *p, D, dt, fault);
    return ssb::cuda_status("op_rk4_kernel");
}

int swarmstep_op_mix(int64_t n, const float *f_c, const float *tau, const swarmstep_quad_params *p, float *motors,
                     float *realized, uint8_t *saturated, void *stream)
{
    if (n < 0 || !p) return bad("bad arguments");
    if (n == 0) return SWARMSTEP_OK;
    if (!f_c || !tau || !motors || !realized || !saturated) return bad("null argument");
    op_mix_kernel<<<blocks(n), kT, 0, (cudaStream_t)stream>>>(n, f_c, tau, *p, motors, realized, saturated);
    return ssb::cuda_status("op_mix_kernel");
}

int swarmstep_op_rotor(int64_t count, const float *rpm, float k_t, float k_q, float omega_max, float *thrust,
                       float *torque, uint8_t *saturated, void *stream)
{
    if (count < 0) return bad("bad count");
    if (count == 0) return SWARMSTEP_OK;
    if (!rpm || !thrust || !torque || !saturated) return bad("null argument");
    op_rotor_kernel<<<blocks(count), kT, 0, (cudaStream_t)stream>>>(count, rpm, k_t, k_q, omega_max, thrust, torque,
                                                                    saturated);
    return ssb::cuda_status("op_rotor_kernel");
}

int swarmstep_op_pid(int64_t n, const float *omega, const float *omega_sp, const float *f_c_sp,
                     const swarmstep_quad_params *p, float dt, float *integral, float *prev_omega, uint8_t *has_prev,
                     const uint8_t *alive, float *tau_out, float *f_c_out, void *stream)
{
    if (n < 0 || !p) return bad("bad arguments");
    if (!(dt > 0.0f)) return bad("dt must be positive");
    if (n == 0) return SWARMSTEP_OK;
    if (!omega || !omega_sp || !f_c_sp || !integral || !prev_omega || !has_prev || !alive || !tau_out || !f_c_out)
        return bad("null argument");
    op_pid_kernel<<<blocks(n), kT, 0, (cudaStream_t)stream>>>(n, omega, omega_sp, f_c_sp, *p, dt,
                                                              integral, prev_omega, has_prev, alive, tau_out, f_c_out);
    return ssb::cuda_status("op_pid_kernel");
}

int swarmstep_op_outer(int64_t n, const float *pos, const float *pos_lo, const float *vel, const float *quat,
                       const uint8_t *alive, const float *p_sp, const float *v_sp, const float *yaw_sp,
                       const swarmstep_quad_params *p, float *omega_sp, float *f_c_sp, uint8_t *low, void *stream)
{
    if (n < 0 || !p) return bad("bad arguments");
    if (n == 0) return SWARMSTEP_OK;
    if (!pos || !vel || !quat || !alive || !p_sp || !v_sp || !yaw_sp || !omega_sp || !f_c_sp || !low)
        return bad("null argument");
    if (pos_lo)
        op_outer_kernel<true><<<blocks(n), kT, 0, (cudaStream_t)stream>>>(n, pos, pos_lo, vel, quat, alive, p_sp,
                                                                         v_sp, yaw_sp, *p, omega_sp, f_c_sp, low);
    else
        op_outer_kernel<false><<<blocks(n), kT, 0, (cudaStream_t)stream>>>(n, pos, nullptr, vel, quat, alive, p_sp,
                                                                          v_sp, yaw_sp, *p, omega_sp, f_c_sp, low);
    return ssb::cuda_status("op_outer_kernel");
}

}  // extern "C"
