// swarmstep_b200.cu -- sm_100a kernels and the C ABI (include/swarmstep_b200.h).
//
// Hot path: quad_step_kernel = K fused QuadGroup.step(dt) calls
// (core.py:166-202) per launch, one agent per thread, state register-resident
// across the K substeps.  Columns are float32 SoA (one column per scalar
// component), so every warp-wide load/store of a component is one fully
// coalesced 128-byte line.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "swarmstep_b200.h"
#include "common.cuh"
#include "quad_math.cuh"

namespace {

using ssb::cuda_status;
using ssb::set_err;

int check_view(const swarmstep_group_view *g)
{
    if (!g || !g->cols || !g->flags) return set_err(SWARMSTEP_EINVAL, "null group view");
    if (g->n < 0 || g->stride < g->n || (g->stride % 32) != 0)
        return set_err(SWARMSTEP_EINVAL, "bad n/stride (stride must be >= n and a multiple of 32)");
    if ((reinterpret_cast<uintptr_t>(g->cols) & 15u) != 0)
        return set_err(SWARMSTEP_EINVAL, "cols must be 16-byte aligned");
    return SWARMSTEP_OK;
}

#ifndef SSB_STEP_BLOCK
#define SSB_STEP_BLOCK 128
#endif
#ifndef SSB_STEP_MINB
#define SSB_STEP_MINB 5
#endif
// 128-thread CTAs, >= 5 resident per SM: caps the step kernel at 102
// registers (no spills) for 20 warps per SM.
constexpr int kBlock = SSB_STEP_BLOCK;

struct Cols {
    float *c;
    int64_t s;
    __device__ __forceinline__ float *col(int k) const { return c + (int64_t)k * s; }
};

// ---------------------------------------------------------------------------
// The fused step kernel.
// ---------------------------------------------------------------------------
#ifndef SSB_TICK_UNROLL
#define SSB_TICK_UNROLL 1
#endif
constexpr int kTickUnroll = SSB_TICK_UNROLL;

// One agent's registers for a launch.
struct Row {
    float p_hi[3], p_lo[3], v[3], q[4], w[3], integ[3], prev[3];
    // u[]: per-launch setpoint registers, shared by the three levels
    //   POS:   p_sp xyz, v_sp xyz (+ overlay on tick 0), cos(yaw), sin(yaw)
    //   MOTOR: rotor-model wrench f_c, tau xyz (core.py:189-197)
    float u[8];
    float w_sp[3], f_sp;   // inner-loop setpoints (stale ones for MOTOR rows)
    bool has_prev;
};

template <bool COMP>
__device__ __forceinline__ void load_state(const Cols &C, int64_t r, Row &R)
{
#pragma unroll
    for (int i = 0; i < 3; i++) {
        R.p_hi[i] = __ldcs(C.col(SWARMSTEP_COL_POS + i) + r);
        R.v[i] = __ldcs(C.col(SWARMSTEP_COL_VEL + i) + r);
        R.w[i] = __ldcs(C.col(SWARMSTEP_COL_OMEGA + i) + r);
        R.integ[i] = __ldcs(C.col(SWARMSTEP_COL_INTEGRAL + i) + r);
        R.prev[i] = __ldcs(C.col(SWARMSTEP_COL_PREV + i) + r);
        R.p_lo[i] = COMP ? __ldcs(C.col(SWARMSTEP_COL_POS_LO + i) + r) : 0.0f;
    }
#pragma unroll
    for (int i = 0; i < 4; i++) R.q[i] = __ldcs(C.col(SWARMSTEP_COL_QUAT + i) + r);
#pragma unroll
    for (int i = 0; i < 7; i++) R.u[i] = __ldcs(C.col(SWARMSTEP_COL_CMD + i) + r);
    R.u[7] = 0.0f;
}

// Per-launch setpoint preparation (commands are fixed across the K ticks).
__device__ __forceinline__ void setup_level(const Cols &C, int64_t r, int level, int overlay_active,
                                            const swarmstep_quad_params &P, Row &R)
{
    if (!R.has_prev) {
        // first sample: no D term (control.py:175-177) <=> prev := w
#pragma unroll
        for (int i = 0; i < 3; i++) R.prev[i] = R.w[i];
    }
    R.w_sp[0] = R.w_sp[1] = R.w_sp[2] = R.f_sp = 0.0f;
    if (level == SWARMSTEP_LEVEL_POS) {
        float s, c;
        sincosf(R.u[6], &s, &c);
        R.u[6] = c;
        R.u[7] = s;
        if (overlay_active) {
#pragma unroll
            for (int i = 0; i < 3; i++) R.u[3 + i] += __ldg(C.col(SWARMSTEP_COL_OVERLAY + i) + r);
        }
    } else if (level == SWARMSTEP_LEVEL_RATE) {
        R.w_sp[0] = R.u[0]; R.w_sp[1] = R.u[1]; R.w_sp[2] = R.u[2]; R.f_sp = R.u[3];
    } else {
        // MOTOR: the PID still runs on the stale setpoints (core.py:109-110,
        // 184-186); the integrated wrench comes from the rotor model
#pragma unroll
        for (int i = 0; i < 3; i++) R.w_sp[i] = __ldg(C.col(SWARMSTEP_COL_SP + i) + r);
        R.f_sp = __ldg(C.col(SWARMSTEP_COL_SP + 3) + r);
        float mt[3], mf;
        ssb::motor_wrench(R.u, P, mf, mt);
        R.u[0] = mf; R.u[1] = mt[0]; R.u[2] = mt[1]; R.u[3] = mt[2];
    }
}

// K ticks of one agent at a fixed command level (the body of QuadGroup.step,
// core.py:166-202, repeated), state updated in place.  Returns the tick at
// which the row faulted (its state registers are then garbage), or -1.
// With pid_only_at >= 0 the loop stops after the controller part of that tick
// (used to rebuild a faulted row's state, see the kernel).
template <int LEVEL, bool COMP, bool RERUN>
__device__ __forceinline__ int run_ticks(const Cols &C, int64_t r, int overlay_active,
                                         const swarmstep_quad_params &P, const ssb::Derived &D,
                                         float dt, int K, int pid_only_at, Row &R)
{
#pragma unroll kTickUnroll
    for (int k = 0; k < K; k++) {
        if (LEVEL == SWARMSTEP_LEVEL_POS) {
            float p_err[3];
#pragma unroll
            for (int i = 0; i < 3; i++) p_err[i] = (R.u[i] - R.p_hi[i]) - R.p_lo[i];
            ssb::outer_row(p_err, R.v, R.q, R.u + 3, R.u[6], R.u[7], P, R.w_sp, R.f_sp);
            if (k == 0 && overlay_active) {
                // the overlay lasts one tick (core.py:199-201)
#pragma unroll
                for (int i = 0; i < 3; i++) R.u[3 + i] = __ldg(C.col(SWARMSTEP_COL_CMD + 3 + i) + r);
            }
        }
        float tau[3], f_c = R.f_sp;
        ssb::pid_row(R.w, R.w_sp, P, D, dt, R.integ, R.prev, tau);
        if (RERUN && k == pid_only_at) return -1;
        if (LEVEL == SWARMSTEP_LEVEL_MOTOR) {
            f_c = R.u[0]; tau[0] = R.u[1]; tau[1] = R.u[2]; tau[2] = R.u[3];
        } else {
            ssb::mix_row(f_c, tau, P);
        }
        if (!ssb::rk4_inplace<COMP>(R.p_hi, R.p_lo, R.v, R.q, R.w, f_c, tau, P, D, dt)) return k;
    }
    return -1;
}

template <bool COMP, bool RERUN>
__device__ __forceinline__ int run_level(const Cols &C, int64_t r, int level, int overlay_active,
                                         const swarmstep_quad_params &P, const ssb::Derived &D,
                                         float dt, int K, int pid_only_at, Row &R)
{
    // level-specialised tick loops: no per-tick level branches
    if (level == SWARMSTEP_LEVEL_POS)
        return run_ticks<SWARMSTEP_LEVEL_POS, COMP, RERUN>(C, r, overlay_active, P, D, dt, K, pid_only_at, R);
    if (level == SWARMSTEP_LEVEL_RATE)
        return run_ticks<SWARMSTEP_LEVEL_RATE, COMP, RERUN>(C, r, 0, P, D, dt, K, pid_only_at, R);
    return run_ticks<SWARMSTEP_LEVEL_MOTOR, COMP, RERUN>(C, r, 0, P, D, dt, K, pid_only_at, R);
}

template <bool COMP>
__global__ void __launch_bounds__(kBlock, SSB_STEP_MINB)
quad_step_kernel(float *__restrict__ cols, uint8_t *__restrict__ flags, int64_t n, int64_t stride,
                 uint32_t *__restrict__ counters, uint64_t *__restrict__ fault_log,
                 int64_t fault_cap, int overlay_active, uint32_t tick_base, const int64_t *tick_dev,
                 const swarmstep_quad_params P, float dt, int K)
{
    const int64_t r = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    if (r >= n) return;
    const Cols C{cols, stride};
    // every state load is issued before the flag test: one memory round trip
    // per row (dead rows are rare; their loads are discarded)
    const uint8_t fl = flags[r];
    Row R;
    load_state<COMP>(C, r, R);
    if (!(fl & SWARMSTEP_FLAG_ALIVE)) return;  // dead rows are frozen (quad.py:395-437)
    const int level = (fl & SWARMSTEP_LEVEL_MASK) >> SWARMSTEP_LEVEL_SHIFT;
    R.has_prev = (fl & SWARMSTEP_FLAG_HAS_PREV) != 0;
    setup_level(C, r, level, overlay_active, P, R);
    const ssb::Derived D = ssb::derive(P, 1.0f / dt);

    const int fault_k = run_level<COMP, false>(C, r, level, overlay_active, P, D, dt, K, -1, R);
    bool alive = true;
    if (fault_k >= 0) {
        // Fault at tick fault_k: the row keeps its pre-tick values, dies and is
        // reported with its tick (quad.py:425-436).  The state was updated in
        // place, so rebuild it by re-running ticks [0, fault_k) from the
        // launch's inputs -- bit-identical by determinism -- plus the
        // controller part of tick fault_k (the reference updates the PID state
        // before rk4_step faults the row).
        alive = false;
        load_state<COMP>(C, r, R);
        R.has_prev = (fl & SWARMSTEP_FLAG_HAS_PREV) != 0;
        setup_level(C, r, level, overlay_active, P, R);
        run_level<COMP, true>(C, r, level, overlay_active, P, D, dt, fault_k + 1, fault_k, R);
        const uint32_t slot = atomicAdd(&counters[0], 1u);
        const uint32_t tick = (tick_dev ? (uint32_t)*tick_dev : 0u) + tick_base + (uint32_t)fault_k;
        if ((int64_t)slot < fault_cap)
            fault_log[slot] = ((uint64_t)(tick & 0xFFFFFFu) << 40) | (uint64_t)r;
    }

    // ---- store ----
#pragma unroll
    for (int i = 0; i < 3; i++) {
        __stcs(C.col(SWARMSTEP_COL_POS + i) + r, R.p_hi[i]);
        __stcs(C.col(SWARMSTEP_COL_VEL + i) + r, R.v[i]);
        __stcs(C.col(SWARMSTEP_COL_OMEGA + i) + r, R.w[i]);
        __stcs(C.col(SWARMSTEP_COL_INTEGRAL + i) + r, R.integ[i]);
        __stcs(C.col(SWARMSTEP_COL_PREV + i) + r, R.prev[i]);
        if (COMP) __stcs(C.col(SWARMSTEP_COL_POS_LO + i) + r, R.p_lo[i]);
    }
#pragma unroll
    for (int i = 0; i < 4; i++) __stcs(C.col(SWARMSTEP_COL_QUAT + i) + r, R.q[i]);
    if (level != SWARMSTEP_LEVEL_MOTOR) {
        // the last tick's setpoints become the stale setpoints a later MOTOR
        // command runs the PID on (core.py:178-182)
#pragma unroll
        for (int i = 0; i < 3; i++) __stcs(C.col(SWARMSTEP_COL_SP + i) + r, R.w_sp[i]);
        __stcs(C.col(SWARMSTEP_COL_SP + 3) + r, R.f_sp);
    }
    // has_prev |= alive (control.py:181): every row reaching here was alive
    const uint8_t nfl = (uint8_t)((fl & SWARMSTEP_LEVEL_MASK) | (alive ? SWARMSTEP_FLAG_ALIVE : 0u) |
                                  SWARMSTEP_FLAG_HAS_PREV);
    if (nfl != fl) flags[r] = nfl;
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
    for (int c = 0; c < 7; c++) cols[(int64_t)(SWARMSTEP_COL_CMD + c) * stride + r] = values[i * 7 + c];
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
        cols[(int64_t)(SWARMSTEP_COL_CMD + c) * stride + r] = c < nv ? values[(int64_t)c * ld + i] : 0.0f;
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

__global__ void retarget_kernel(float *cols, uint8_t *flags, int64_t n, int64_t stride, int compensated,
                                double px, double py, double pz, double radius, uint32_t *counters)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const uint8_t fl = flags[r];
    if (!(fl & SWARMSTEP_FLAG_ALIVE)) return;
    double p[3];
    for (int i = 0; i < 3; i++) {
        p[i] = (double)cols[(int64_t)(SWARMSTEP_COL_POS + i) * stride + r];
        if (compensated) p[i] += (double)cols[(int64_t)(SWARMSTEP_COL_POS_LO + i) * stride + r];
    }
    const double dx = p[0] - px, dy = p[1] - py, dz = p[2] - pz;
    const double d = sqrt(dx * dx + dy * dy + dz * dz);
    if (!(d < radius)) return;
    const double w = cols[(int64_t)(SWARMSTEP_COL_QUAT + 0) * stride + r];
    const double x = cols[(int64_t)(SWARMSTEP_COL_QUAT + 1) * stride + r];
    const double y = cols[(int64_t)(SWARMSTEP_COL_QUAT + 2) * stride + r];
    const double z = cols[(int64_t)(SWARMSTEP_COL_QUAT + 3) * stride + r];
    const double yaw = atan2(2.0 * (w * z + x * y), 1.0 - 2.0 * (y * y + z * z));  // quat.py:139-143
    flags[r] = (uint8_t)(fl & ~SWARMSTEP_LEVEL_MASK);  // POS level
    const float vals[7] = {(float)px, (float)py, (float)pz, 0.0f, 0.0f, 0.0f, (float)yaw};
    for (int c = 0; c < 7; c++) cols[(int64_t)(SWARMSTEP_COL_CMD + c) * stride + r] = vals[c];
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
            double p = cols[(int64_t)(SWARMSTEP_COL_POS + i) * stride + r];
            if (compensated) p += (double)cols[(int64_t)(SWARMSTEP_COL_POS_LO + i) * stride + r];
            pos[r * 3 + i] = p;
        }
        if (vel) vel[r * 3 + i] = cols[(int64_t)(SWARMSTEP_COL_VEL + i) * stride + r];
        if (omega) omega[r * 3 + i] = cols[(int64_t)(SWARMSTEP_COL_OMEGA + i) * stride + r];
    }
    if (quat)
        for (int i = 0; i < 4; i++) quat[r * 4 + i] = cols[(int64_t)(SWARMSTEP_COL_QUAT + i) * stride + r];
    if (alive) alive[r] = (flags[r] & SWARMSTEP_FLAG_ALIVE) ? 1 : 0;
}

__global__ void unpack_f64_kernel(float *cols, uint8_t *flags, int64_t n, int64_t stride, int compensated,
                                  const double *pos, const double *vel, const double *quat,
                                  const double *omega, const uint8_t *alive)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    for (int i = 0; i < 3; i++) {
        if (pos) {
            const double p = pos[r * 3 + i];
            const float hi = (float)p;
            cols[(int64_t)(SWARMSTEP_COL_POS + i) * stride + r] = hi;
            cols[(int64_t)(SWARMSTEP_COL_POS_LO + i) * stride + r] = compensated ? (float)(p - (double)hi) : 0.0f;
        }
        if (vel) cols[(int64_t)(SWARMSTEP_COL_VEL + i) * stride + r] = (float)vel[r * 3 + i];
        if (omega) cols[(int64_t)(SWARMSTEP_COL_OMEGA + i) * stride + r] = (float)omega[r * 3 + i];
    }
    if (quat)
        for (int i = 0; i < 4; i++) cols[(int64_t)(SWARMSTEP_COL_QUAT + i) * stride + r] = (float)quat[r * 4 + i];
    if (alive) {
        const uint8_t fl = flags[r];
        flags[r] = (uint8_t)((fl & SWARMSTEP_LEVEL_MASK) | (alive[r] ? SWARMSTEP_FLAG_ALIVE : 0u));
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

int swarmstep_preload(void)
{
    // force-load every kernel of this translation unit (lazy module loading
    // must not happen inside a CUDA graph capture)
    cudaFuncAttributes a;
    const void *fns[] = {(const void *)quad_step_kernel<true>, (const void *)quad_step_kernel<false>,
                         (const void *)apply_commands_kernel, (const void *)set_setpoints_kernel,
                         (const void *)mark_dead_kernel, (const void *)retarget_kernel,
                         (const void *)pack_f64_kernel, (const void *)unpack_f64_kernel};
    for (const void *f : fns)
        if (cudaFuncGetAttributes(&a, f) != cudaSuccess) return cuda_status("cudaFuncGetAttributes");
    return swarmstep_feed_preload();
}

int swarmstep_quad_step(const swarmstep_group_view *g, const swarmstep_quad_params *p, float dt,
                        int k_substeps, int overlay_active, uint32_t tick_base, const int64_t *tick_dev,
                        void *stream)
{
    int st = check_view(g);
    if (st) return st;
    if (!p) return set_err(SWARMSTEP_EINVAL, "null params");
    if (!(dt > 0.0f)) return set_err(SWARMSTEP_EINVAL, "dt must be positive");
    if (k_substeps < 1) return set_err(SWARMSTEP_EINVAL, "k_substeps must be >= 1");
    if (!g->counters) return set_err(SWARMSTEP_EINVAL, "null counters");
    if (g->n == 0) return SWARMSTEP_OK;
    auto kern = g->compensated ? quad_step_kernel<true> : quad_step_kernel<false>;
    kern<<<grid_for(g->n, kBlock), kBlock, 0, (cudaStream_t)stream>>>(
        g->cols, g->flags, g->n, g->stride, g->counters, g->fault_log, g->fault_log ? g->fault_cap : 0,
        overlay_active, tick_base, tick_dev, *p, dt, k_substeps);
    return cuda_status("quad_step_kernel");
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
