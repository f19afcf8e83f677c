// feed.cu -- device-resident setpoint feed.
//
// The reference's in-loop circle strategy builds one AgentCommand Python
// object per alive agent per tick (client.py:55-73 circle_swarm_strategy ->
// control.py:297-315 circle_reference -> core.py:117-135 apply_command),
// which the survey measured at 80% of a 5k-agent tick.  Here the same
// setpoints are written straight into the command columns by one kernel that
// reads the simulation tick from device memory, so a whole run of ticks --
// feed + fused step per tick -- can be captured in one CUDA graph.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "circle.cuh"
#include "common.cuh"

namespace {

// circle_reference for row r with phase phase0 + r*dphase (circle.cuh)
__global__ void circle_kernel(float *cols, uint8_t *flags, int64_t n, int64_t stride, const int64_t *tick_dev,
                              int64_t tick_offset, double dt, double radius, double omega, double z,
                              double phase0, double dphase)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const uint8_t fl = flags[r];
    if (!(fl & SWARMSTEP_FLAG_ALIVE)) return;       // the strategy skips dead agents (client.py:66-67)
    float vals[7];
    ssb::circle_values(*tick_dev + tick_offset, dt, radius, omega, z, phase0 + dphase * (double)r, vals);
#pragma unroll
    for (int i = 0; i < 7; i++) cols[ssb::at(SWARMSTEP_COL_CMD + i, r)] = vals[i];
    const uint8_t nfl = (uint8_t)(fl & ~SWARMSTEP_LEVEL_MASK);  // POS level
    if (nfl != fl) flags[r] = nfl;
}

__global__ void tick_add_kernel(int64_t *tick_dev, int64_t delta) { *tick_dev += delta; }

}  // namespace

extern "C" {

int swarmstep_quad_circle_setpoints(const swarmstep_group_view *g, const int64_t *tick_dev, int64_t tick_offset,
                                    double dt, double radius, double omega, double z, double phase0,
                                    double dphase, void *stream)
{
    if (!g || !g->cols || !g->flags || !tick_dev) return ssb::set_err(SWARMSTEP_EINVAL, "null argument");
    if (!(radius > 0.0)) return ssb::set_err(SWARMSTEP_EINVAL, "circle radius must be positive");  // control.py:305-306
    if (!(dt > 0.0)) return ssb::set_err(SWARMSTEP_EINVAL, "dt must be positive");
    if (g->n == 0) return SWARMSTEP_OK;
    circle_kernel<<<(unsigned)((g->n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        g->cols, g->flags, g->n, g->stride, tick_dev, tick_offset, dt, radius, omega, z, phase0, dphase);
    return ssb::cuda_status("circle_kernel");
}

int swarmstep_feed_preload(void)
{
    cudaFuncAttributes a;
    if (cudaFuncGetAttributes(&a, (const void *)circle_kernel) != cudaSuccess ||
        cudaFuncGetAttributes(&a, (const void *)tick_add_kernel) != cudaSuccess)
        return ssb::cuda_status("cudaFuncGetAttributes");
    return SWARMSTEP_OK;
}

int swarmstep_tick_add(int64_t *tick_dev, int64_t delta, void *stream)
{
    if (!tick_dev) return ssb::set_err(SWARMSTEP_EINVAL, "null tick");
    tick_add_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(tick_dev, delta);
    return ssb::cuda_status("tick_add_kernel");
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Unicycle group: the reference's second homogeneous type,
// core.py:208-289.  Exact-arc kinematic integration, evaluated in the
// cancellation-free form  sin th1 - sin th0 = 2 cos(th0 + w dt/2) sin(w dt/2)
// (and likewise for cos), which equals the reference's expression in R but
// keeps float32 accurate when w dt is small.
// ---------------------------------------------------------------------------
namespace {

__global__ void unicycle_kernel(float *cols, const uint8_t *flags, int64_t n, float v_max, float w_max, float dt,
                                int K, int overlay_active)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    if (!(flags[r] & SWARMSTEP_FLAG_ALIVE)) return;     // dead rows are untouched (core.py:241-246)
    float *c = cols + ssb::tile_base(r);
    auto col = [&](int k) -> float & { return c[k * SWARMSTEP_TILE]; };
    float qw = col(SWARMSTEP_COL_QUAT + 0), qx = col(SWARMSTEP_COL_QUAT + 1);
    float qy = col(SWARMSTEP_COL_QUAT + 2), qz = col(SWARMSTEP_COL_QUAT + 3);
    float th = atan2f(2.0f * (qw * qz + qx * qy), 1.0f - 2.0f * (qy * qy + qz * qz));   // quat.py:139-143
    double px = ssb::pos_f64(cols, r, 0, true);
    double py = ssb::pos_f64(cols, r, 1, true);
    float v_cmd = col(SWARMSTEP_COL_CMD + 0);
    const float w_cmd = col(SWARMSTEP_COL_CMD + 1);
    if (overlay_active) {
        // project the influence field onto the heading (core.py:277-283)
        v_cmd += col(SWARMSTEP_COL_OVERLAY + 0) * cosf(th) + col(SWARMSTEP_COL_OVERLAY + 1) * sinf(th);
    }
    // np.clip semantics (NaN passes through)
    auto clip = [](float x, float lo, float hi) { return x < lo ? lo : (x > hi ? hi : x); };
    const float w = clip(w_cmd, -w_max, w_max);
    float v = 0.0f, th1 = th;
    for (int k = 0; k < K; k++) {
        const float vk = (k == 0) ? v_cmd : col(SWARMSTEP_COL_CMD + 0);   // overlay lasts one tick
        v = clip(vk, -v_max, v_max);
        th1 = th + w * dt;
        float dx, dy;
        if (fabsf(w) <= 1e-9f) {
            dx = v * cosf(th) * dt;
            dy = v * sinf(th) * dt;
        } else {
            const float hs = sinf(0.5f * w * dt) * (2.0f / w);
            const float thm = th + 0.5f * w * dt;
            dx = v * hs * cosf(thm);
            dy = v * hs * sinf(thm);
        }
        px += (double)dx;
        py += (double)dy;
        // the reference re-derives the heading from the stored quaternion each tick
        th = atan2f(sinf(th1), cosf(th1));
    }
    const float hx = (float)px, hy = (float)py;
    col(SWARMSTEP_COL_POS + 0) = hx;
    col(SWARMSTEP_COL_POS + 1) = hy;
    // packed low parts (common.cuh): new x, y fields, z's kept
    const uint32_t low = __float_as_uint(col(SWARMSTEP_COL_POS_LO));
    col(SWARMSTEP_COL_POS_LO) = __uint_as_float(ssb::pos_lo_field((float)(px - (double)hx), 0, hx) |
                                                ssb::pos_lo_field((float)(py - (double)hy), 1, hy) |
                                                (low & (0x3FFu << 20)));
    float s, co;
    sincosf(0.5f * th1, &s, &co);                     // yaw_quat (quat.py:129-136)
    col(SWARMSTEP_COL_QUAT + 0) = co;
    col(SWARMSTEP_COL_QUAT + 1) = 0.0f;
    col(SWARMSTEP_COL_QUAT + 2) = 0.0f;
    col(SWARMSTEP_COL_QUAT + 3) = s;
    col(SWARMSTEP_COL_VEL + 0) = v * cosf(th1);
    col(SWARMSTEP_COL_VEL + 1) = v * sinf(th1);
    col(SWARMSTEP_COL_VEL + 2) = 0.0f;
    col(SWARMSTEP_COL_OMEGA + 2) = w;
}

}  // namespace

extern "C" int swarmstep_unicycle_step(const swarmstep_group_view *g, float v_max, float omega_max, float dt,
                                       int k_substeps, int launch_flags, void *stream)
{
    if (!g || !g->cols || !g->flags) return ssb::set_err(SWARMSTEP_EINVAL, "null argument");
    if (!(dt > 0.0f)) return ssb::set_err(SWARMSTEP_EINVAL, "dt must be positive");        // core.py:230-231
    if (k_substeps < 1) return ssb::set_err(SWARMSTEP_EINVAL, "k_substeps must be >= 1");
    if (g->n == 0) return SWARMSTEP_OK;
    unicycle_kernel<<<(unsigned)((g->n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
        g->cols, g->flags, g->n, v_max, omega_max, dt, k_substeps, launch_flags & SWARMSTEP_STEP_OVERLAY);
    return ssb::cuda_status("unicycle_kernel");
}
