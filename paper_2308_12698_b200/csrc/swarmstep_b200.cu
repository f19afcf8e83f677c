// swarmstep_b200.cu -- the C ABI (include/swarmstep_b200.h): argument checks
// and dispatch to the step kernels (step_pair.cu, step_direct.cu via
// step_launch.h), plus the command / bookkeeping kernels.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>

#include "swarmstep_b200.h"
#include "circle.cuh"
#include "common.cuh"
#include "quad_math.cuh"
#include "step_launch.h"


namespace {

using ssb::cuda_status;
using ssb::set_err;

int check_view(const swarmstep_group_view *g)
{
    if (!g || !g->cols || !g->flags) return set_err(SWARMSTEP_EINVAL, "null group view");
    if (g->n < 0 || g->stride < g->n || (g->stride % SWARMSTEP_TILE) != 0)
        return set_err(SWARMSTEP_EINVAL, "bad n/stride (stride must be >= n and a multiple of 128)");
    if ((reinterpret_cast<uintptr_t>(g->cols) & 15u) != 0)
        return set_err(SWARMSTEP_EINVAL, "cols must be 16-byte aligned");
    if ((reinterpret_cast<uintptr_t>(g->flags) & 1u) != 0)    // the paired kernels read two flag bytes at once
        return set_err(SWARMSTEP_EINVAL, "flags must be 2-byte aligned");
    return SWARMSTEP_OK;
}

// ---------------------------------------------------------------------------
// Command / bookkeeping kernels (off the per-tick hot loop).
// ---------------------------------------------------------------------------
__global__ void apply_commands_kernel(float *cols, uint8_t *flags, int64_t stride,
                                      const int64_t *rows, const uint8_t *levels,
                                      const float *values, int64_t count)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const int64_t r = rows[i];
    const uint8_t fl = flags[r];
    if (!(fl & SWARMSTEP_FLAG_ALIVE)) return;
    flags[r] = (uint8_t)((fl & ~SWARMSTEP_LEVEL_MASK) | ((levels[i] & 3u) << SWARMSTEP_LEVEL_SHIFT));
#pragma unroll
    for (int c = 0; c < 7; c++) cols[ssb::at(SWARMSTEP_COL_CMD + c, r)] = values[i * 7 + c];
}

__global__ void set_setpoints_kernel(float *cols, uint8_t *flags, int64_t stride, int64_t row0,
                                     int64_t count, int level, const float *values, int64_t ld)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const int64_t r = row0 + i;
    const uint8_t fl = flags[r];
    if (!(fl & SWARMSTEP_FLAG_ALIVE)) return;
    const uint8_t nfl = (uint8_t)((fl & ~SWARMSTEP_LEVEL_MASK) | ((level & 3) << SWARMSTEP_LEVEL_SHIFT));
    if (nfl != fl) flags[r] = nfl;
    const int nv = level == SWARMSTEP_LEVEL_POS ? 7 : 4;
    for (int c = 0; c < 7; c++)
        cols[ssb::at(SWARMSTEP_COL_CMD + c, r)] = c < nv ? values[(int64_t)c * ld + i] : 0.0f;
}

__global__ void mark_dead_kernel(uint8_t *flags, const int64_t *rows, uint8_t *was_alive, int64_t count)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const int64_t r = rows[i];
    const uint8_t fl = flags[r];
    if (was_alive) was_alive[i] = (fl & SWARMSTEP_FLAG_ALIVE) ? 1 : 0;
    flags[r] = (uint8_t)(fl & ~SWARMSTEP_FLAG_ALIVE);
}

__device__ __forceinline__ double norm3_rn(double x, double y, double z)
{
    return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z)));
}

// World._apply_viewer_input for ATTRACT / REPEL (core.py:445-453) with
// viewer_velocity_offsets (wire.py:320-340) evaluated per row in float64 in
// the reference's operation order, added to the one-tick overlay in float32
// like add_velocity_overlay's host path.  counters[2] counts rows whose
// offset is non-zero (the reference's `offsets.any()` gate).
__global__ void viewer_overlay_kernel(float *cols, const uint8_t *flags, int64_t n, int64_t stride,
                                      int compensated, double px, double py, double pz, double radius,
                                      double gain, uint32_t *counters)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool hit = false;
    if (r < n && (flags[r] & SWARMSTEP_FLAG_ALIVE)) {
        double p[3];
        for (int i = 0; i < 3; i++) {
            p[i] = (double)cols[ssb::at(SWARMSTEP_COL_POS + i, r)];
            if (compensated) p[i] += (double)ssb::pos_lo(cols, r, i);
        }
        const double delta[3] = {__dadd_rn(px, -p[0]), __dadd_rn(py, -p[1]), __dadd_rn(pz, -p[2])};
        const double d = norm3_rn(delta[0], delta[1], delta[2]);
        if (d < radius && d > 1e-12) {
            // sign * strength * (1.0 - d / radius) / d
            const double scale = __ddiv_rn(__dmul_rn(gain, __dadd_rn(1.0, -__ddiv_rn(d, radius))), d);
            for (int i = 0; i < 3; i++) {
                const double o = __dmul_rn(delta[i], scale);
                hit |= o != 0.0;
                const int64_t at = ssb::at(SWARMSTEP_COL_OVERLAY + i, r);
                cols[at] = __fadd_rn(cols[at], (float)o);
            }
        }
    }
    const unsigned hits = __ballot_sync(0xffffffffu, hit);
    if (hits && (threadIdx.x & 31) == 0) atomicAdd(&counters[2], (uint32_t)__popc(hits));
}

__global__ void retarget_kernel(float *cols, uint8_t *flags, int64_t n, int64_t stride, int compensated,
                                double px, double py, double pz, double radius, uint32_t *counters)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const uint8_t fl = flags[r];
    if (!(fl & SWARMSTEP_FLAG_ALIVE)) return;
    double p[3];
    for (int i = 0; i < 3; i++) {
        p[i] = (double)cols[ssb::at(SWARMSTEP_COL_POS + i, r)];
        if (compensated) p[i] += (double)ssb::pos_lo(cols, r, i);
    }
    // np.linalg.norm(pos - point, axis=1): ((dx^2 + dy^2) + dz^2), no contraction
    const double d = norm3_rn(__dadd_rn(p[0], -px), __dadd_rn(p[1], -py), __dadd_rn(p[2], -pz));
    if (!(d < radius)) return;
    const double w = cols[ssb::at(SWARMSTEP_COL_QUAT + 0, r)];
    const double x = cols[ssb::at(SWARMSTEP_COL_QUAT + 1, r)];
    const double y = cols[ssb::at(SWARMSTEP_COL_QUAT + 2, r)];
    const double z = cols[ssb::at(SWARMSTEP_COL_QUAT + 3, r)];
    const double yaw = atan2(2.0 * (w * z + x * y), 1.0 - 2.0 * (y * y + z * z));  // quat.py:139-143
    flags[r] = (uint8_t)(fl & ~SWARMSTEP_LEVEL_MASK);  // POS level
    // a point beyond float32 range saturates (like the host command store)
    const float vals[7] = {ssb::f32_sat(px), ssb::f32_sat(py), ssb::f32_sat(pz), 0.0f, 0.0f, 0.0f, (float)yaw};
    for (int c = 0; c < 7; c++) cols[ssb::at(SWARMSTEP_COL_CMD + c, r)] = vals[c];
    atomicAdd(&counters[1], 1u);
}

__global__ void pack_f64_kernel(const float *cols, const uint8_t *flags, int64_t n, int64_t stride,
                                int compensated, double *pos, double *vel, double *quat,
                                double *omega, uint8_t *alive)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    for (int i = 0; i < 3; i++) {
        if (pos) {
            double p = cols[ssb::at(SWARMSTEP_COL_POS + i, r)];
            if (compensated) p += (double)ssb::pos_lo(cols, r, i);
            pos[r * 3 + i] = p;
        }
        if (vel) vel[r * 3 + i] = cols[ssb::at(SWARMSTEP_COL_VEL + i, r)];
        if (omega) omega[r * 3 + i] = cols[ssb::at(SWARMSTEP_COL_OMEGA + i, r)];
    }
    if (quat)
        for (int i = 0; i < 4; i++) quat[r * 4 + i] = cols[ssb::at(SWARMSTEP_COL_QUAT + i, r)];
    if (alive) alive[r] = (flags[r] & SWARMSTEP_FLAG_ALIVE) ? 1 : 0;
}

__global__ void unpack_f64_kernel(float *cols, uint8_t *flags, int64_t n, int64_t stride, int compensated,
                                  const double *pos, const double *vel, const double *quat,
                                  const double *omega, const uint8_t *alive)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    if (pos) {
        float hi[3], lo[3];
        for (int i = 0; i < 3; i++) {
            const double p = pos[r * 3 + i];
            hi[i] = (float)p;
            lo[i] = compensated ? (float)(p - (double)hi[i]) : 0.0f;
            cols[ssb::at(SWARMSTEP_COL_POS + i, r)] = hi[i];
        }
        cols[ssb::at(SWARMSTEP_COL_POS_LO, r)] = __uint_as_float(ssb::pos_lo_encode(lo, hi));
    }
    for (int i = 0; i < 3; i++) {
        if (vel) cols[ssb::at(SWARMSTEP_COL_VEL + i, r)] = (float)vel[r * 3 + i];
        if (omega) cols[ssb::at(SWARMSTEP_COL_OMEGA + i, r)] = (float)omega[r * 3 + i];
    }
    if (quat)
        for (int i = 0; i < 4; i++) cols[ssb::at(SWARMSTEP_COL_QUAT + i, r)] = (float)quat[r * 4 + i];
    if (alive) {
        const uint8_t fl = flags[r];
        // the PID's has_prev survives a host-state push: the reference never
        // resets pid_state.has_prev when batch state is edited (control.py:100-114)
        flags[r] = (uint8_t)((fl & (SWARMSTEP_LEVEL_MASK | SWARMSTEP_FLAG_HAS_PREV)) |
                             (alive[r] ? SWARMSTEP_FLAG_ALIVE : 0u));
    }
}

inline unsigned grid_for(int64_t n, int block) { return (unsigned)((n + block - 1) / block); }

}  // namespace

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" int swarmstep_feed_preload(void);

extern "C" {

int swarmstep_abi_version(void) { return SWARMSTEP_ABI_VERSION; }

const char *swarmstep_last_error(void) { return ssb::err_buf(); }

int swarmstep_device_info(int *sm_count, int *cc_major, int *cc_minor)
{
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return cuda_status("cudaGetDevice");
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess) return cuda_status("cudaGetDeviceProperties");
    if (sm_count) *sm_count = prop.multiProcessorCount;
    if (cc_major) *cc_major = prop.major;
    if (cc_minor) *cc_minor = prop.minor;
    if (prop.major != 10) return set_err(SWARMSTEP_ENODEV, "device is not sm_100 (B200)");
    return SWARMSTEP_OK;
}

int swarmstep_quad_params_init(swarmstep_quad_params *p, const swarmstep_quad_physics *phys,
                               const swarmstep_quad_gains *gains)
{
    if (!p || !phys || !gains) return set_err(SWARMSTEP_EINVAL, "null argument");
    const double vals[] = {phys->m, phys->ixx, phys->iyy, phys->izz, phys->g, phys->k_t, phys->k_q,
                           phys->arm_length, phys->arm_angle, phys->omega_max};
    for (double v : vals)
        if (!(v > 0.0) || !isfinite(v))     // quad.py:56-60
            return set_err(SWARMSTEP_EINVAL, "all quadrotor parameters must be strictly positive and finite");
    // G (quad.py:106-122): rows mutually orthogonal, so G^-1 = G^T diag(1 / |row|^2)
    const double ls = phys->arm_length * sin(phys->arm_angle), lc = phys->arm_length * cos(phys->arm_angle);
    const double kr = phys->k_q / phys->k_t;
    const double G[16] = {1, 1, 1, 1, ls, -ls, -ls, ls, -lc, -lc, lc, lc, kr, -kr, kr, -kr};
    const double det = 256.0 * ls * ls * lc * lc * kr * kr;     // |det G| = prod |row| (orthogonal rows)
    if (!(fabs(det) > 1e-12)) return set_err(SWARMSTEP_EINVAL, "allocation matrix is singular (degenerate arm angle)");
    memset(p, 0, sizeof(*p));
    p->m = (float)phys->m;
    p->inv_m = (float)(1.0 / phys->m);
    p->g = (float)phys->g;
    p->ixx = (float)phys->ixx; p->iyy = (float)phys->iyy; p->izz = (float)phys->izz;
    p->inv_ixx = (float)(1.0 / phys->ixx); p->inv_iyy = (float)(1.0 / phys->iyy); p->inv_izz = (float)(1.0 / phys->izz);
    p->k_t = (float)phys->k_t;
    p->omega_max = (float)phys->omega_max;
    const double f_max = phys->k_t * phys->omega_max * phys->omega_max;
    p->f_max = (float)f_max;
    p->fc_max = (float)(4.0 * f_max);
    const double rsq[4] = {4.0, 4.0 * ls * ls, 4.0 * lc * lc, 4.0 * kr * kr};
    for (int i = 0; i < 4; i++)
        for (int j = 0; j < 4; j++) {
            p->G[i * 4 + j] = (float)G[i * 4 + j];
            p->G_inv[i * 4 + j] = (float)(G[j * 4 + i] / rsq[j]);
        }
    for (int i = 0; i < 3; i++) {
        p->kp[i] = (float)gains->kp[i]; p->ki[i] = (float)gains->ki[i]; p->kd[i] = (float)gains->kd[i];
        p->i_limit[i] = (float)gains->i_limit[i];
        p->kp_pos[i] = (float)gains->kp_pos[i]; p->kv[i] = (float)gains->kv[i]; p->k_att[i] = (float)gains->k_att[i];
    }
    p->omega_sp_max = (float)gains->omega_sp_max;
    p->a_cmd_min = (float)gains->a_cmd_min;
    return SWARMSTEP_OK;
}

int swarmstep_memcpy_async(void *dst, const void *src, uint64_t bytes, void *stream)
{
    if (bytes == 0) return SWARMSTEP_OK;
    if (!dst || !src) return set_err(SWARMSTEP_EINVAL, "null pointer");
    if (cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDefault, (cudaStream_t)stream) != cudaSuccess)
        return cuda_status("cudaMemcpyAsync");
    return SWARMSTEP_OK;
}

int swarmstep_stream_sync(void *stream)
{
    if (cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess) return cuda_status("cudaStreamSynchronize");
    return cuda_status("stream work");
}

int swarmstep_preload(void)
{
    // force-load every kernel (lazy module loading must not happen inside a
    // CUDA graph capture)
    int st = ssbl::preload_pair();
    if (!st) st = ssbl::preload_direct();
    if (st) return st;
    cudaFuncAttributes attr;
    const void *fns[] = {(const void *)apply_commands_kernel, (const void *)set_setpoints_kernel,
                         (const void *)mark_dead_kernel, (const void *)retarget_kernel,
                         (const void *)viewer_overlay_kernel,
                         (const void *)pack_f64_kernel, (const void *)unpack_f64_kernel};
    for (const void *f : fns)
        if (cudaFuncGetAttributes(&attr, f) != cudaSuccess) return cuda_status("cudaFuncGetAttributes");
    return swarmstep_feed_preload();
}

int swarmstep_quad_step(const swarmstep_group_view *g, const swarmstep_quad_params *p, float dt,
                        int k_substeps, int launch_flags, uint32_t tick_base, const int64_t *tick_dev,
                        void *stream)
{
    int st = check_view(g);
    if (st) return st;
    if (!p) return set_err(SWARMSTEP_EINVAL, "null params");
    if (!(dt > 0.0f)) return set_err(SWARMSTEP_EINVAL, "dt must be positive");
    if (k_substeps < 1) return set_err(SWARMSTEP_EINVAL, "k_substeps must be >= 1");
    if (!g->counters) return set_err(SWARMSTEP_EINVAL, "null counters");
    if (g->n == 0) return SWARMSTEP_OK;
    const ssb::Derived D = ssb::derive(*p, dt);
    const bool axi = D.axisym != 0;   // the axisymmetric-vehicle step kernels (NoLagT<true>)
    const int overlay = launch_flags & SWARMSTEP_STEP_OVERLAY;
    const int motor = (launch_flags & SWARMSTEP_STEP_MOTOR) ? 1 : 0;
    const bool use_tma = (launch_flags & SWARMSTEP_STEP_FORCE_DIRECT) ? false
                       : (launch_flags & SWARMSTEP_STEP_FORCE_TMA) ? true
                       : k_substeps <= SSB_TMA_MAX_K;
    const ssbl::StepArgs args{g->cols, g->flags, g->n, g->counters, g->fault_log, g->fault_log ? g->fault_cap : 0,
                              overlay, tick_base, tick_dev, dt, k_substeps, g->compensated != 0};
    if (use_tma) return ssbl::launch_tma(args, motor, *p, D, (cudaStream_t)stream);
    if (!(launch_flags & SWARMSTEP_STEP_FORCE_DIRECT) &&
        ((launch_flags & SWARMSTEP_STEP_FORCE_PAIR) || k_substeps >= SSB_PAIR_MIN_K))
        return ssbl::launch_pair(args, axi, *p, D, (cudaStream_t)stream);
    return ssbl::launch_direct(args, axi, *p, D, (cudaStream_t)stream);
}

int swarmstep_quad_step_overlapped(const swarmstep_group_view *g, const swarmstep_quad_params *p, float dt,
                                   int k_substeps, int launch_flags, uint32_t tick_base, uint32_t *tile_epoch,
                                   uint32_t wait_epoch, uint32_t set_epoch, void *stream)
{
    int st = check_view(g);
    if (st) return st;
    if (!p || !tile_epoch) return set_err(SWARMSTEP_EINVAL, "null params / tile_epoch");
    if (!(dt > 0.0f)) return set_err(SWARMSTEP_EINVAL, "dt must be positive");
    if (k_substeps < 1) return set_err(SWARMSTEP_EINVAL, "k_substeps must be >= 1");
    if (!g->counters) return set_err(SWARMSTEP_EINVAL, "null counters");
    if (set_epoch == 0 || (int32_t)(set_epoch - wait_epoch) <= 0)
        return set_err(SWARMSTEP_EINVAL, "set_epoch must be non-zero and follow wait_epoch");
    if (launch_flags & SWARMSTEP_STEP_FORCE_TMA)
        return set_err(SWARMSTEP_EINVAL, "the TMA-staged kernel does not overlap launches");
    if (g->n == 0) return SWARMSTEP_OK;
    const ssb::Derived D = ssb::derive(*p, dt);
    const bool axi = D.axisym != 0;
    const ssbl::StepArgs args{g->cols, g->flags, g->n, g->counters, g->fault_log, g->fault_log ? g->fault_cap : 0,
                              launch_flags & SWARMSTEP_STEP_OVERLAY, tick_base, nullptr, dt, k_substeps,
                              g->compensated != 0};
    const ssbl::Pdl pdl{tile_epoch, wait_epoch, set_epoch};
    if (!(launch_flags & SWARMSTEP_STEP_FORCE_DIRECT) &&
        ((launch_flags & SWARMSTEP_STEP_FORCE_PAIR) || k_substeps >= SSB_PAIR_MIN_K))
        return ssbl::launch_pair(args, axi, *p, D, (cudaStream_t)stream, pdl);
    return ssbl::launch_direct(args, axi, *p, D, (cudaStream_t)stream, pdl);
}

int swarmstep_quad_step_collect(const swarmstep_group_view *g, const swarmstep_quad_params *p, float dt,
                                int k_substeps, int launch_flags, uint32_t tick_base, uint32_t *counters_host,
                                void *stream)
{
    // the World-facing synchronous tick in one call: launch, fault counter to
    // pinned host memory, wait (three host API calls, one crossing of the FFI)
    int st = swarmstep_quad_step(g, p, dt, k_substeps, launch_flags, tick_base, nullptr, stream);
    if (st) return st;
    if (!counters_host) return set_err(SWARMSTEP_EINVAL, "null counters_host");
    if (cudaMemcpyAsync(counters_host, g->counters, 4 * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                        (cudaStream_t)stream) != cudaSuccess)
        return cuda_status("cudaMemcpyAsync");
    if (cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess) return cuda_status("cudaStreamSynchronize");
    return cuda_status("quad step");
}

int swarmstep_quad_step_lag(const swarmstep_group_view *g, const swarmstep_quad_params *p, float *motor,
                            float tau_m, float dt, int k_substeps, int launch_flags, uint32_t tick_base,
                            const int64_t *tick_dev, void *stream)
{
    int st = check_view(g);
    if (st) return st;
    if (!p || !motor) return set_err(SWARMSTEP_EINVAL, "null params / motor");
    if (!(dt > 0.0f)) return set_err(SWARMSTEP_EINVAL, "dt must be positive");
    if (!(tau_m > 0.0f) || !isfinite(tau_m))
        return set_err(SWARMSTEP_EINVAL, "tau_m must be positive and finite (tau_m = 0 is swarmstep_quad_step)");
    if (k_substeps < 1) return set_err(SWARMSTEP_EINVAL, "k_substeps must be >= 1");
    if (!g->counters) return set_err(SWARMSTEP_EINVAL, "null counters");
    if ((reinterpret_cast<uintptr_t>(motor) & 15u) != 0) return set_err(SWARMSTEP_EINVAL, "motor must be 16-byte aligned");
    if (g->n == 0) return SWARMSTEP_OK;
    const ssb::Derived D = ssb::derive(*p, dt);
    const float phi = (float)(-((double)tau_m / (double)dt) * expm1(-(double)dt / (double)tau_m));
    const float e_full = (float)exp(-(double)dt / (double)tau_m);
    const int overlay = launch_flags & SWARMSTEP_STEP_OVERLAY;
    const ssbl::StepArgs args{g->cols, g->flags, g->n, g->counters, g->fault_log, g->fault_log ? g->fault_cap : 0,
                              overlay, tick_base, tick_dev, dt, k_substeps, g->compensated != 0};
    if (!(launch_flags & SWARMSTEP_STEP_FORCE_DIRECT) &&
        ((launch_flags & SWARMSTEP_STEP_FORCE_PAIR) || k_substeps >= SSB_PAIR_MIN_K))
        return ssbl::launch_pair_lag(args, motor, phi, e_full, *p, D, (cudaStream_t)stream);
    return ssbl::launch_lag(args, motor, phi, e_full, *p, D, (cudaStream_t)stream);
}

static int quad_step_circle(const swarmstep_group_view *g, const swarmstep_quad_params *p, float dt, int k_substeps,
                            int launch_flags, uint32_t tick_base, const int64_t *tick_dev,
                            const swarmstep_circle_feed *feed, const ssbl::Pdl &pdl, void *stream)
{
    int st = check_view(g);
    if (st) return st;
    if (!p || !feed || !tick_dev) return set_err(SWARMSTEP_EINVAL, "null params / feed / tick");
    if (!(dt > 0.0f)) return set_err(SWARMSTEP_EINVAL, "dt must be positive");
    if (!(feed->radius > 0.0)) return set_err(SWARMSTEP_EINVAL, "circle radius must be positive");
    if (!(feed->dt > 0.0)) return set_err(SWARMSTEP_EINVAL, "feed dt must be positive");
    if (k_substeps < 1) return set_err(SWARMSTEP_EINVAL, "k_substeps must be >= 1");
    if (!g->counters) return set_err(SWARMSTEP_EINVAL, "null counters");
    if (g->n == 0) return SWARMSTEP_OK;
    const ssb::Derived D = ssb::derive(*p, dt);
    const ssbl::StepArgs args{g->cols, g->flags, g->n, g->counters, g->fault_log, g->fault_log ? g->fault_cap : 0,
                              0, tick_base, tick_dev, dt, k_substeps, g->compensated != 0};
    if (!(launch_flags & SWARMSTEP_STEP_FORCE_DIRECT) &&
        ((launch_flags & SWARMSTEP_STEP_FORCE_PAIR) || k_substeps >= SSB_PAIR_MIN_K))
        return ssbl::launch_pair_circle(args, *feed, *p, D, (cudaStream_t)stream, pdl);
    return ssbl::launch_circle(args, *feed, *p, D, (cudaStream_t)stream, pdl);
}

int swarmstep_quad_step_circle(const swarmstep_group_view *g, const swarmstep_quad_params *p, float dt,
                               int k_substeps, int launch_flags, uint32_t tick_base, const int64_t *tick_dev,
                               const swarmstep_circle_feed *feed, void *stream)
{
    return quad_step_circle(g, p, dt, k_substeps, launch_flags, tick_base, tick_dev, feed, ssbl::Pdl{nullptr, 0, 0},
                            stream);
}

int swarmstep_quad_step_circle_overlapped(const swarmstep_group_view *g, const swarmstep_quad_params *p, float dt,
                                          int k_substeps, int launch_flags, uint32_t tick_base,
                                          const int64_t *tick_dev, const swarmstep_circle_feed *feed,
                                          uint32_t *tile_epoch, uint32_t wait_epoch, uint32_t set_epoch,
                                          void *stream)
{
    if (!tile_epoch) return set_err(SWARMSTEP_EINVAL, "null tile_epoch");
    if (set_epoch == 0 || (int32_t)(set_epoch - wait_epoch) <= 0)
        return set_err(SWARMSTEP_EINVAL, "set_epoch must be non-zero and follow wait_epoch");
    return quad_step_circle(g, p, dt, k_substeps, launch_flags, tick_base, tick_dev, feed,
                            ssbl::Pdl{tile_epoch, wait_epoch, set_epoch}, stream);
}

int swarmstep_quad_apply_commands(const swarmstep_group_view *g, const int64_t *rows, const uint8_t *levels,
                                  const float *values, int64_t count, void *stream)
{
    int st = check_view(g);
    if (st) return st;
    if (count < 0) return set_err(SWARMSTEP_EINVAL, "negative count");
    if (count == 0) return SWARMSTEP_OK;
    if (!rows || !levels || !values) return set_err(SWARMSTEP_EINVAL, "null command arrays");
    apply_commands_kernel<<<grid_for(count, 256), 256, 0, (cudaStream_t)stream>>>(
        g->cols, g->flags, g->stride, rows, levels, values, count);
    return cuda_status("apply_commands_kernel");
}

int swarmstep_quad_set_setpoints(const swarmstep_group_view *g, int64_t row0, int64_t count, int level,
                                 const float *values, int64_t ld, void *stream)
{
    int st = check_view(g);
    if (st) return st;
    if (row0 < 0 || count < 0 || row0 + count > g->n) return set_err(SWARMSTEP_EINVAL, "row range out of bounds");
    if (level < 0 || level > 2) return set_err(SWARMSTEP_EINVAL, "bad level");
    if (count == 0) return SWARMSTEP_OK;
    if (!values || ld < count) return set_err(SWARMSTEP_EINVAL, "bad values / ld");
    set_setpoints_kernel<<<grid_for(count, 256), 256, 0, (cudaStream_t)stream>>>(
        g->cols, g->flags, g->stride, row0, count, level, values, ld);
    return cuda_status("set_setpoints_kernel");
}

int swarmstep_quad_mark_dead(const swarmstep_group_view *g, const int64_t *rows, uint8_t *was_alive,
                             int64_t count, void *stream)
{
    int st = check_view(g);
    if (st) return st;
    if (count <= 0) return count < 0 ? set_err(SWARMSTEP_EINVAL, "negative count") : SWARMSTEP_OK;
    if (!rows) return set_err(SWARMSTEP_EINVAL, "null rows");
    mark_dead_kernel<<<grid_for(count, 256), 256, 0, (cudaStream_t)stream>>>(g->flags, rows, was_alive, count);
    return cuda_status("mark_dead_kernel");
}

int swarmstep_quad_retarget_waypoint(const swarmstep_group_view *g, const double *point3, double radius,
                                     void *stream)
{
    int st = check_view(g);
    if (st) return st;
    if (!point3 || !g->counters) return set_err(SWARMSTEP_EINVAL, "null point / counters");
    if (g->n == 0) return SWARMSTEP_OK;
    retarget_kernel<<<grid_for(g->n, 256), 256, 0, (cudaStream_t)stream>>>(
        g->cols, g->flags, g->n, g->stride, g->compensated, point3[0], point3[1], point3[2], radius, g->counters);
    return cuda_status("retarget_kernel");
}

int swarmstep_quad_viewer_overlay(const swarmstep_group_view *g, const double *point3, double radius,
                                  double gain, void *stream)
{
    int st = check_view(g);
    if (st) return st;
    if (!point3 || !g->counters) return set_err(SWARMSTEP_EINVAL, "null point / counters");
    if (g->n == 0 || !(radius > 0.0)) return SWARMSTEP_OK;   // wire.py:331-332
    viewer_overlay_kernel<<<grid_for(g->n, 256), 256, 0, (cudaStream_t)stream>>>(
        g->cols, g->flags, g->n, g->stride, g->compensated, point3[0], point3[1], point3[2], radius, gain,
        g->counters);
    return cuda_status("viewer_overlay_kernel");
}

int swarmstep_quad_pack_f64(const swarmstep_group_view *g, double *pos, double *vel, double *quat,
                            double *omega, uint8_t *alive, void *stream)
{
    int st = check_view(g);
    if (st) return st;
    if (g->n == 0) return SWARMSTEP_OK;
    pack_f64_kernel<<<grid_for(g->n, 256), 256, 0, (cudaStream_t)stream>>>(
        g->cols, g->flags, g->n, g->stride, g->compensated, pos, vel, quat, omega, alive);
    return cuda_status("pack_f64_kernel");
}

int swarmstep_quad_unpack_f64(const swarmstep_group_view *g, const double *pos, const double *vel,
                              const double *quat, const double *omega, const uint8_t *alive, void *stream)
{
    int st = check_view(g);
    if (st) return st;
    if (g->n == 0) return SWARMSTEP_OK;
    unpack_f64_kernel<<<grid_for(g->n, 256), 256, 0, (cudaStream_t)stream>>>(
        g->cols, g->flags, g->n, g->stride, g->compensated, pos, vel, quat, omega, alive);
    return cuda_status("unpack_f64_kernel");
}

}  // extern "C"
