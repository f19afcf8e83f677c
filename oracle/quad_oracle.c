/*
 * quad_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A float64, scalar-per-agent C restatement of the reference's quadrotor hot
 * path (swarmstep, /root/reference/pkg/src/swarmstep).  It is the checker the
 * CUDA path is compared against; it is never linked into, loaded by, or used
 * as a fallback for the product package (paper_2308_12698_b200).  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load it.
 *
 * Parity pin: tests/test_oracle.py checks every entry point below against
 * golden vectors produced by importing the reference itself
 * (tests/golden/make_golden.py) and against the reference's own known-answer
 * tests (test_quad.py, test_control.py, test_acceptance.py).
 *
 * Operation order follows the reference's numpy ufunc sequence so that the
 * float64 results agree to a few ulp; compile with -ffp-contract=off.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    /* QuadParams (quad.py:39-69) */
    double m, ixx, iyy, izz, g, k_t, k_q, arm_length, arm_angle, omega_max;
    double f_max;      /* k_t * omega_max^2 (quad.py:62-63) */
    double G[16];      /* allocation matrix, row-major (quad.py:106-122) */
    double Ginv[16];   /* np.linalg.inv(G), row-major, filled by the caller */
    /* PidGains (control.py:40-53) */
    double kp[3], ki[3], kd[3], i_limit[3];
    /* OuterGains (control.py:56-68) */
    double kp_pos[3], kv[3], k_att[3], omega_sp_max, a_cmd_min;
} oracle_params;

enum { LVL_POS = 0, LVL_RATE = 1, LVL_MOTOR = 2 }; /* core.py:73 */

/* ---- dynamics: quad.py:222-310 (_deriv_kernel) ------------------------- */
/* s = (px,py,pz, vx,vy,vz, qw,qx,qy,qz, ox,oy,oz) */
void oracle_deriv(const double *s, double f_c, const double *tau,
                  const oracle_params *p, double *d)
{
    double qw = s[6], qx = s[7], qy = s[8], qz = s[9];
    double ox = s[10], oy = s[11], oz = s[12];
    double t0, t1;
    d[0] = s[3]; d[1] = s[4]; d[2] = s[5];
    t0 = qx * qz; t1 = qw * qy; t0 = t0 + t1; t0 = t0 * 2.0; t0 = t0 * f_c; d[3] = t0 / p->m;
    t0 = qy * qz; t1 = qw * qx; t0 = t0 - t1; t0 = t0 * 2.0; t0 = t0 * f_c; d[4] = t0 / p->m;
    t0 = qx * qx; t1 = qy * qy; t0 = t0 + t1; t0 = t0 * -2.0; t0 = t0 + 1.0; t0 = t0 * f_c;
    d[5] = t0 / p->m; d[5] = d[5] - p->g;

    t0 = qx * ox; t1 = qy * oy; t0 = t0 + t1; t1 = qz * oz; t0 = t0 + t1; d[6] = t0 * -0.5;
    t0 = qw * ox; t1 = qy * oz; t0 = t0 + t1; t1 = qz * oy; t0 = t0 - t1; d[7] = t0 * 0.5;
    t0 = qw * oy; t1 = qz * ox; t0 = t0 + t1; t1 = qx * oz; t0 = t0 - t1; d[8] = t0 * 0.5;
    t0 = qw * oz; t1 = qx * oy; t0 = t0 + t1; t1 = qy * ox; t0 = t0 - t1; d[9] = t0 * 0.5;

    t0 = oz * p->izz; t0 = oy * t0; t1 = oy * p->iyy; t1 = oz * t1; t0 = t0 - t1;
    t0 = tau[0] - t0; d[10] = t0 / p->ixx;
    t0 = ox * p->ixx; t0 = oz * t0; t1 = oz * p->izz; t1 = ox * t1; t0 = t0 - t1;
    t0 = tau[1] - t0; d[11] = t0 / p->iyy;
    t0 = oy * p->iyy; t0 = ox * t0; t1 = ox * p->ixx; t1 = oy * t1; t0 = t0 - t1;
    t0 = tau[2] - t0; d[12] = t0 / p->izz;
}

/* ---- integrator: quad.py:350-437 (rk4_step), one row ------------------
 * Returns 1 if the row is ok, 0 on a fault (non-finite pos/vel/omega, or a
 * non-finite / non-positive quaternion norm).  `out` receives the candidate
 * post-step state; the caller decides whether to commit it (alive rows
 * without fault) exactly as rk4_step's masked copy-back does.          */
int oracle_rk4_row(const double *y, double f_c, const double *tau,
                   const oracle_params *p, double dt, double *out)
{
    double k1[13], k2[13], k3[13], k4[13], st[13];
    double half = 0.5 * dt, h6 = dt / 6.0;
    int i;
    oracle_deriv(y, f_c, tau, p, k1);
    for (i = 0; i < 13; i++) { st[i] = k1[i] * half; st[i] = st[i] + y[i]; }
    oracle_deriv(st, f_c, tau, p, k2);
    for (i = 0; i < 13; i++) { st[i] = k2[i] * half; st[i] = st[i] + y[i]; }
    oracle_deriv(st, f_c, tau, p, k3);
    for (i = 0; i < 13; i++) { st[i] = k3[i] * dt; st[i] = st[i] + y[i]; }
    oracle_deriv(st, f_c, tau, p, k4);
    for (i = 0; i < 13; i++) {
        double s = k2[i] * 2.0;
        double k3x2;
        s = s + k1[i];
        k3x2 = k3[i] * 2.0;
        s = s + k3x2;
        s = s + k4[i];
        s = s * h6;
        out[i] = s + y[i];
    }
    {
        double t0 = out[6] * out[6], t1;
        int ok;
        t1 = out[7] * out[7]; t0 = t0 + t1;
        t1 = out[8] * out[8]; t0 = t0 + t1;
        t1 = out[9] * out[9]; t0 = t0 + t1;
        t0 = sqrt(t0);
        ok = isfinite(t0) && t0 > 0.0;
        for (i = 6; i < 10; i++) out[i] = out[i] / t0;
        for (i = 0; i < 6; i++) ok = ok && isfinite(out[i]);
        for (i = 10; i < 13; i++) ok = ok && isfinite(out[i]);
        return ok;
    }
}

/* ---- opt-in first-order rotor lag (north star; ABSENT in the reference) --
 * Parity unpinned: the reference has no rotor dynamics, so this
 * restates the model DESIGN.md defines, not reference code.  Rotor thrusts f
 * follow the commanded thrusts u, held over the tick, exactly:
 * f(t + s) = u + (f(t) - u) exp(-s / tau_m).  The rigid body integrates
 * (quad.py:350-437, wrench held) the wrench of the tick-mean thrust
 * fbar = u + (f(t) - u) phi, phi = (tau_m / dt)(1 - exp(-dt / tau_m)): the
 * thrust impulse over the tick is exact, and tau_m -> 0 gives fbar = u, the
 * reference's instantaneous mixer. */
/* wrench of rotor thrusts f: G f (quad.py:138-140) */
static void thrust_wrench(const double *f, const oracle_params *p, double *wrench)
{
    int i, j;
    for (i = 0; i < 4; i++) {
        double acc = 0.0;
        for (j = 0; j < 4; j++) acc += f[j] * p->G[i * 4 + j];
        wrench[i] = acc;
    }
}

/* ---- mixer: quad.py:143-168 (mix_to_motors), one row ------------------ */
int oracle_mix_row(double f_c, const double *tau, const oracle_params *p,
                   double *motors, double *realized)
{
    double w[4] = {f_c, tau[0], tau[1], tau[2]};
    int i, j, sat = 0;
    for (i = 0; i < 4; i++) {
        double acc = 0.0;
        for (j = 0; j < 4; j++) acc += w[j] * p->Ginv[i * 4 + j];
        motors[i] = acc;
    }
    for (i = 0; i < 4; i++) {
        if (motors[i] < 0.0 || motors[i] > p->f_max) sat = 1;
        motors[i] = motors[i] < 0.0 ? 0.0 : (motors[i] > p->f_max ? p->f_max : motors[i]);
    }
    for (i = 0; i < 4; i++) {
        double acc = 0.0;
        for (j = 0; j < 4; j++) acc += motors[j] * p->G[i * 4 + j];
        realized[i] = acc;
    }
    return sat;
}

/* ---- rotor model + MOTOR override: quad.py:130-140, core.py:189-197 ----- */
void oracle_motor_wrench(const double *rpm, const oracle_params *p, double *wrench)
{
    double f[4];
    int i, j;
    for (i = 0; i < 4; i++) {
        double c = rpm[i] < 0.0 ? 0.0 : (rpm[i] > p->omega_max ? p->omega_max : rpm[i]);
        f[i] = p->k_t * (c * c);
    }
    for (i = 0; i < 4; i++) {
        double acc = 0.0;
        for (j = 0; j < 4; j++) acc += f[j] * p->G[i * 4 + j];
        wrench[i] = acc;
    }
}

/* ---- inner loop: control.py:136-187 (rate_pid_step), one row ----------- */
void oracle_pid_row(const double *omega, const double *omega_sp, double f_c_sp,
                    const oracle_params *p, double dt, int alive,
                    double *integral, double *prev_omega, uint8_t *has_prev,
                    double *tau, double *f_c)
{
    int a;
    int use_d = (*has_prev) && alive;
    for (a = 0; a < 3; a++) {
        double e = omega_sp[a] - omega[a];
        double t;
        if (alive) integral[a] = integral[a] + e * dt;
        integral[a] = integral[a] < -p->i_limit[a] ? -p->i_limit[a]
                    : (integral[a] > p->i_limit[a] ? p->i_limit[a] : integral[a]);
        t = e * p->kp[a];
        t = t + integral[a] * p->ki[a];
        if (use_d) {
            double dd = omega[a] - prev_omega[a];
            dd = dd / dt;
            dd = dd * p->kd[a];
            t = t - dd;
        }
        tau[a] = alive ? t : 0.0;
    }
    if (alive) { prev_omega[0] = omega[0]; prev_omega[1] = omega[1]; prev_omega[2] = omega[2]; }
    *has_prev = (uint8_t)((*has_prev) || alive);
    *f_c = alive ? f_c_sp : 0.0;
}

/* ---- outer loop: control.py:190-294, one row ---------------------------- */
static void cross3(const double *a, const double *b, double *c)
{
    c[0] = a[1] * b[2] - a[2] * b[1];
    c[1] = a[2] * b[0] - a[0] * b[2];
    c[2] = a[0] * b[1] - a[1] * b[0];
}

static double norm3(const double *v) { return sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]); }

static double safe_sqrt(double x) { return sqrt(x > 1e-30 ? x : 1e-30); }

/* control.py:190-213 (_rotmats_to_quats), row-major r[i][j] */
static void rotmat_to_quat(const double r[3][3], double *q)
{
    double m00 = r[0][0], m01 = r[0][1], m02 = r[0][2];
    double m10 = r[1][0], m11 = r[1][1], m12 = r[1][2];
    double m20 = r[2][0], m21 = r[2][1], m22 = r[2][2];
    double tr = m00 + m11 + m22, s, n;
    if (tr > 0.0) {
        s = safe_sqrt(tr + 1.0) * 2.0;
        q[0] = 0.25 * s; q[1] = (m21 - m12) / s; q[2] = (m02 - m20) / s; q[3] = (m10 - m01) / s;
    } else if (m00 >= m11 && m00 >= m22) {
        s = safe_sqrt(1.0 + m00 - m11 - m22) * 2.0;
        q[0] = (m21 - m12) / s; q[1] = 0.25 * s; q[2] = (m01 + m10) / s; q[3] = (m02 + m20) / s;
    } else if (m11 >= m22) {
        s = safe_sqrt(1.0 + m11 - m00 - m22) * 2.0;
        q[0] = (m02 - m20) / s; q[1] = (m01 + m10) / s; q[2] = 0.25 * s; q[3] = (m12 + m21) / s;
    } else {
        s = safe_sqrt(1.0 + m22 - m00 - m11) * 2.0;
        q[0] = (m10 - m01) / s; q[1] = (m02 + m20) / s; q[2] = (m12 + m21) / s; q[3] = 0.25 * s;
    }
    n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    q[0] /= n; q[1] /= n; q[2] /= n; q[3] /= n;
}

/* Returns 1 if the row is "low thrust" (free-fall floor engaged), and -1 if
 * quat_mul would have raised InvalidStateError on non-finite input
 * (quat.py:84, 69-72). */
int oracle_outer_row(const double *pos, const double *vel, const double *quat, int alive,
                     const double *p_sp, const double *v_sp, double yaw,
                     const oracle_params *p, double *omega_sp, double *f_c_out)
{
    double a[3], z_des[3], z_body[3], x_c[3], y_raw[3], y_des[3], x_des[3];
    double a_norm, eff, f_c, ny, r[3][3], q_des[4], qc[4], qe[4], nq, s, angle, factor;
    int low, i, degenerate, bad = 0;
    double qw = quat[0], qx = quat[1], qy = quat[2], qz = quat[3];

    for (i = 0; i < 3; i++)
        a[i] = p->kp_pos[i] * (p_sp[i] - pos[i]) + p->kv[i] * (v_sp[i] - vel[i]);
    a[2] += p->g;
    a_norm = norm3(a);
    low = a_norm < p->a_cmd_min;
    eff = a_norm > p->a_cmd_min ? a_norm : p->a_cmd_min;
    if (isnan(a_norm)) eff = a_norm; /* np.maximum propagates NaN */
    for (i = 0; i < 3; i++) z_des[i] = a[i] / eff;
    if (low) { z_des[0] = 0.0; z_des[1] = 0.0; z_des[2] = 1.0; }

    z_body[0] = 2.0 * (qx * qz + qw * qy);
    z_body[1] = 2.0 * (qy * qz - qw * qx);
    z_body[2] = 1.0 - 2.0 * (qx * qx + qy * qy);
    f_c = p->m * eff * (z_body[0] * z_des[0] + z_body[1] * z_des[1] + z_body[2] * z_des[2]);
    f_c = f_c < 0.0 ? 0.0 : (f_c > 4.0 * p->f_max ? 4.0 * p->f_max : f_c);

    x_c[0] = cos(yaw); x_c[1] = sin(yaw); x_c[2] = 0.0;
    cross3(z_des, x_c, y_raw);
    ny = norm3(y_raw);
    degenerate = ny < 1e-6;
    for (i = 0; i < 3; i++) y_des[i] = y_raw[i] / (degenerate ? 1.0 : ny);
    if (degenerate) {
        double y_c[3] = {-sin(yaw), cos(yaw), 0.0}, x_alt[3], nx;
        cross3(y_c, z_des, x_alt);
        nx = norm3(x_alt);
        for (i = 0; i < 3; i++) x_alt[i] /= nx;
        cross3(z_des, x_alt, y_des);
    }
    cross3(y_des, z_des, x_des);
    for (i = 0; i < 3; i++) { r[i][0] = x_des[i]; r[i][1] = y_des[i]; r[i][2] = z_des[i]; }
    rotmat_to_quat(r, q_des);

    /* quat_mul(quat_conj(q), q_des), renormalized (quat.py:75-92) */
    for (i = 0; i < 4; i++) if (!isfinite(quat[i]) || !isfinite(q_des[i])) bad = 1;
    qc[0] = qw; qc[1] = -qx; qc[2] = -qy; qc[3] = -qz;
    qe[0] = qc[0] * q_des[0] - qc[1] * q_des[1] - qc[2] * q_des[2] - qc[3] * q_des[3];
    qe[1] = qc[0] * q_des[1] + qc[1] * q_des[0] + qc[2] * q_des[3] - qc[3] * q_des[2];
    qe[2] = qc[0] * q_des[2] - qc[1] * q_des[3] + qc[2] * q_des[0] + qc[3] * q_des[1];
    qe[3] = qc[0] * q_des[3] + qc[1] * q_des[2] - qc[2] * q_des[1] + qc[3] * q_des[0];
    nq = sqrt(qe[0] * qe[0] + qe[1] * qe[1] + qe[2] * qe[2] + qe[3] * qe[3]);
    for (i = 0; i < 4; i++) qe[i] /= nq;
    if (qe[0] < 0.0) for (i = 0; i < 4; i++) qe[i] = -qe[i];
    s = norm3(qe + 1);
    angle = 2.0 * atan2(s, qe[0]);
    factor = s > 1e-12 ? angle / s : 2.0;
    for (i = 0; i < 3; i++) {
        double w = p->k_att[i] * (qe[1 + i] * factor);
        omega_sp[i] = w < -p->omega_sp_max ? -p->omega_sp_max : (w > p->omega_sp_max ? p->omega_sp_max : w);
    }
    *f_c_out = f_c;
    if (!alive) {
        *f_c_out = 0.0;
        omega_sp[0] = omega_sp[1] = omega_sp[2] = 0.0;
        low = 0;
    }
    return bad ? -1 : low;
}

/* ---- group step: core.py:166-202 (QuadGroup.step), rows [lo, hi) --------
 * Array shapes mirror the reference's numpy columns (row-major):
 *   pos/vel/omega (n,3), quat (n,4), alive (n,) u8,
 *   integral/prev_omega (n,3), has_prev (n,) u8,
 *   omega_sp (n,3), f_c_sp (n,)         -- QuadGroup.omega_sp / f_c_sp
 *   cmd_level (n,) u8, cmd_values (n,7) -- QuadGroup command store
 *   v_overlay (n,3) or NULL             -- QuadGroup.v_overlay (active iff non-NULL)
 *   fault (n,) u8 out                   -- 1 where rk4 faulted this step
 * Returns the number of faulted rows; sets *bad if quat_mul would raise.  */
typedef struct {
    int64_t lo, hi;
    double dt;
    const oracle_params *p;
    double *pos, *vel, *quat, *omega;
    uint8_t *alive;
    double *integral, *prev_omega;
    uint8_t *has_prev;
    double *omega_sp, *f_c_sp;
    const uint8_t *cmd_level;
    const double *cmd_values;
    const double *v_overlay;
    uint8_t *fault;
    double *motor;           /* (n,4) rotor thrusts, or NULL: no rotor lag */
    double phi, e_full;      /* (tau_m / dt)(1 - exp(-dt / tau_m)), exp(-dt / tau_m) */
    int any_pos;
    int64_t n_fault;
    int bad;
} step_job;

static void step_rows(step_job *j)
{
    const oracle_params *p = j->p;
    int64_t r;
    for (r = j->lo; r < j->hi; r++) {
        int alive = j->alive[r] != 0;
        int lvl = j->cmd_level[r];
        const double *cv = j->cmd_values + r * 7;
        double tau[3], f_c, motors[4], realized[4], y[13], out[13];
        int i, ok;
        j->fault[r] = 0;
        /* setpoint selection (core.py:171-182) */
        if (lvl == LVL_POS || j->any_pos) {
            /* the reference evaluates the outer loop for all rows whenever any
             * POS row exists, and quat_mul's finiteness check covers all rows */
            double vsp[3], osp[3], fsp;
            int lowflag;
            for (i = 0; i < 3; i++)
                vsp[i] = j->v_overlay ? cv[3 + i] + j->v_overlay[r * 3 + i] : cv[3 + i];
            lowflag = oracle_outer_row(j->pos + r * 3, j->vel + r * 3, j->quat + r * 4, alive,
                                       cv, vsp, cv[6], p, osp, &fsp);
            if (lowflag < 0) j->bad = 1;
            if (lvl == LVL_POS) {
                for (i = 0; i < 3; i++) j->omega_sp[r * 3 + i] = osp[i];
                j->f_c_sp[r] = fsp;
            }
        }
        if (lvl == LVL_RATE) {
            for (i = 0; i < 3; i++) j->omega_sp[r * 3 + i] = cv[i];
            j->f_c_sp[r] = cv[3];
        }
        /* inner loop + mixer (core.py:184-188) */
        oracle_pid_row(j->omega + r * 3, j->omega_sp + r * 3, j->f_c_sp[r], p, j->dt, alive,
                       j->integral + r * 3, j->prev_omega + r * 3, j->has_prev + r,
                       tau, &f_c);
        oracle_mix_row(f_c, tau, p, motors, realized);
        f_c = realized[0]; tau[0] = realized[1]; tau[1] = realized[2]; tau[2] = realized[3];
        /* raw motor override (core.py:189-197) */
        if (lvl == LVL_MOTOR && alive) {
            double wr[4];
            oracle_motor_wrench(cv, p, wr);
            f_c = wr[0]; tau[0] = wr[1]; tau[1] = wr[2]; tau[2] = wr[3];
        }
        /* rk4 (quad.py:350-437) */
        if (!alive) continue;
        for (i = 0; i < 3; i++) { y[i] = j->pos[r * 3 + i]; y[3 + i] = j->vel[r * 3 + i]; y[10 + i] = j->omega[r * 3 + i]; }
        for (i = 0; i < 4; i++) y[6 + i] = j->quat[r * 4 + i];
        if (j->motor) {
            /* rotor lag: commanded thrusts u = clamped mixer motors, or
             * k_t clip(rpm)^2 for MOTOR rows (quad.py:134-137) */
            double u[4], fbar[4], f1[4], wr[4], *f0 = j->motor + r * 4;
            for (i = 0; i < 4; i++) {
                if (lvl == LVL_MOTOR) {
                    double c = cv[i] < 0.0 ? 0.0 : (cv[i] > p->omega_max ? p->omega_max : cv[i]);
                    u[i] = p->k_t * (c * c);
                } else {
                    u[i] = motors[i];
                }
                fbar[i] = u[i] + (f0[i] - u[i]) * j->phi;
                f1[i] = u[i] + (f0[i] - u[i]) * j->e_full;
            }
            thrust_wrench(fbar, p, wr);
            ok = oracle_rk4_row(y, wr[0], wr + 1, p, j->dt, out);
            if (ok) for (i = 0; i < 4; i++) f0[i] = f1[i];
        } else {
            ok = oracle_rk4_row(y, f_c, tau, p, j->dt, out);
        }
        if (!ok) {
            j->alive[r] = 0;
            j->fault[r] = 1;
            j->n_fault++;
            continue;
        }
        for (i = 0; i < 3; i++) { j->pos[r * 3 + i] = out[i]; j->vel[r * 3 + i] = out[3 + i]; j->omega[r * 3 + i] = out[10 + i]; }
        for (i = 0; i < 4; i++) j->quat[r * 4 + i] = out[6 + i];
    }
}

static void *step_thread(void *arg) { step_rows((step_job *)arg); return NULL; }

/* Returns #faults, or -1 if quat_mul would have raised (the reference then
 * raises InvalidStateError before touching any state; this oracle has already
 * stepped, so callers treat -1 as "group crashed").  nthreads >= 1 shards the
 * rows contiguously across POSIX threads; results are identical for any
 * thread count because rows are independent (core.py determinism,
 * test_core.py:314-339). */
static int64_t group_step(int64_t n, double dt, const oracle_params *p,
                          double *pos, double *vel, double *quat, double *omega, uint8_t *alive,
                          double *integral, double *prev_omega, uint8_t *has_prev,
                          double *omega_sp, double *f_c_sp,
                          const uint8_t *cmd_level, const double *cmd_values,
                          const double *v_overlay, uint8_t *fault, int nthreads,
                          double *motor, double tau_m)
{
    step_job jobs[256];
    pthread_t th[256];
    int64_t total = 0, r;
    int t, any_pos = 0, bad = 0;
    if (!(dt > 0.0)) return -2;
    for (r = 0; r < n; r++) if (cmd_level[r] == LVL_POS) { any_pos = 1; break; }
    /* The reference raises InvalidStateError from quat_mul before touching
     * any state (control.py:279 -> quat.py:84) when any row's outer-loop
     * input is non-finite; the outer loop covers every row (dead ones too)
     * whenever a POS row exists.  Pre-check the inputs so this oracle, too,
     * leaves the state untouched in that case. */
    if (any_pos) {
        for (r = 0; r < n && !bad; r++) {
            int i;
            for (i = 0; i < 7; i++) if (!isfinite(cmd_values[r * 7 + i])) bad = 1;
            for (i = 0; i < 4; i++) if (!isfinite(quat[r * 4 + i])) bad = 1;
            for (i = 0; i < 3; i++)
                if (!isfinite(pos[r * 3 + i]) || !isfinite(vel[r * 3 + i]) ||
                    (v_overlay && !isfinite(v_overlay[r * 3 + i]))) bad = 1;
        }
        if (bad) return -1;
    }
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    if ((int64_t)nthreads > n) nthreads = (int)(n > 0 ? n : 1);
    for (t = 0; t < nthreads; t++) {
        step_job *j = &jobs[t];
        j->lo = n * t / nthreads;
        j->hi = n * (t + 1) / nthreads;
        j->dt = dt; j->p = p;
        j->pos = pos; j->vel = vel; j->quat = quat; j->omega = omega; j->alive = alive;
        j->integral = integral; j->prev_omega = prev_omega; j->has_prev = has_prev;
        j->omega_sp = omega_sp; j->f_c_sp = f_c_sp;
        j->cmd_level = cmd_level; j->cmd_values = cmd_values; j->v_overlay = v_overlay;
        j->fault = fault; j->any_pos = any_pos; j->n_fault = 0; j->bad = 0;
        j->motor = motor;
        j->phi = motor ? -(tau_m / dt) * expm1(-dt / tau_m) : 0.0;
        j->e_full = motor ? exp(-dt / tau_m) : 0.0;
    }
    if (nthreads == 1) {
        step_rows(&jobs[0]);
    } else {
        for (t = 0; t < nthreads; t++) pthread_create(&th[t], NULL, step_thread, &jobs[t]);
        for (t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
    }
    for (t = 0; t < nthreads; t++) { total += jobs[t].n_fault; bad |= jobs[t].bad; }
    return bad ? -1 : total;
}

int64_t oracle_group_step(int64_t n, double dt, const oracle_params *p,
                          double *pos, double *vel, double *quat, double *omega, uint8_t *alive,
                          double *integral, double *prev_omega, uint8_t *has_prev,
                          double *omega_sp, double *f_c_sp,
                          const uint8_t *cmd_level, const double *cmd_values,
                          const double *v_overlay, uint8_t *fault, int nthreads)
{
    return group_step(n, dt, p, pos, vel, quat, omega, alive, integral, prev_omega, has_prev, omega_sp,
                      f_c_sp, cmd_level, cmd_values, v_overlay, fault, nthreads, NULL, 0.0);
}

/* QuadGroup.step with the opt-in rotor lag (parity unpinned, see above);
 * motor (n,4) rotor thrusts are updated in place for rows that step without
 * fault.  tau_m <= 0 -> -2. */
int64_t oracle_group_step_lag(int64_t n, double dt, const oracle_params *p,
                              double *pos, double *vel, double *quat, double *omega, uint8_t *alive,
                              double *integral, double *prev_omega, uint8_t *has_prev,
                              double *omega_sp, double *f_c_sp,
                              const uint8_t *cmd_level, const double *cmd_values,
                              const double *v_overlay, uint8_t *fault, int nthreads,
                              double *motor, double tau_m)
{
    if (!(tau_m > 0.0) || !motor) return -2;
    return group_step(n, dt, p, pos, vel, quat, omega, alive, integral, prev_omega, has_prev, omega_sp,
                      f_c_sp, cmd_level, cmd_values, v_overlay, fault, nthreads, motor, tau_m);
}

/* ---- batched per-function entry points for golden pinning -------------- */
void oracle_deriv_batch(int64_t n, const double *state13, const double *f_c, const double *tau,
                        const oracle_params *p, double *out13)
{
    int64_t r;
    for (r = 0; r < n; r++) oracle_deriv(state13 + r * 13, f_c[r], tau + r * 3, p, out13 + r * 13);
}

/* rk4_step semantics on (n,13) rows: faulted alive rows are reverted and
 * killed, dead rows untouched; returns #faults. */
int64_t oracle_rk4_batch(int64_t n, double *state13, uint8_t *alive, const double *f_c,
                         const double *tau, const oracle_params *p, double dt, uint8_t *fault)
{
    int64_t r, nf = 0;
    for (r = 0; r < n; r++) {
        double out[13];
        int ok = oracle_rk4_row(state13 + r * 13, f_c[r], tau + r * 3, p, dt, out);
        fault[r] = 0;
        if (!alive[r]) continue;
        if (!ok) { alive[r] = 0; fault[r] = 1; nf++; continue; }
        memcpy(state13 + r * 13, out, sizeof(out));
    }
    return nf;
}

void oracle_mix_batch(int64_t n, const double *f_c, const double *tau, const oracle_params *p,
                      double *motors, double *realized, uint8_t *sat)
{
    int64_t r;
    for (r = 0; r < n; r++) sat[r] = (uint8_t)oracle_mix_row(f_c[r], tau + r * 3, p, motors + r * 4, realized + r * 4);
}

void oracle_pid_batch(int64_t n, const double *omega, const double *omega_sp, const double *f_c_sp,
                      const oracle_params *p, double dt, const uint8_t *alive,
                      double *integral, double *prev_omega, uint8_t *has_prev,
                      double *tau, double *f_c)
{
    int64_t r;
    for (r = 0; r < n; r++)
        oracle_pid_row(omega + r * 3, omega_sp + r * 3, f_c_sp[r], p, dt, alive[r] != 0,
                       integral + r * 3, prev_omega + r * 3, has_prev + r, tau + r * 3, f_c + r);
}

int oracle_outer_batch(int64_t n, const double *pos, const double *vel, const double *quat,
                       const uint8_t *alive, const double *p_sp, const double *v_sp,
                       const double *yaw, const oracle_params *p,
                       double *omega_sp, double *f_c, uint8_t *low)
{
    int64_t r;
    int bad = 0;
    for (r = 0; r < n; r++) {
        int l = oracle_outer_row(pos + r * 3, vel + r * 3, quat + r * 4, alive[r] != 0,
                                 p_sp + r * 3, v_sp + r * 3, yaw[r], p, omega_sp + r * 3, f_c + r);
        if (l < 0) { bad = 1; l = 0; }
        low[r] = (uint8_t)l;
    }
    return bad;
}
