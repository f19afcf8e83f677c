/*
 * swarmstep_b200.h -- C ABI of the B200 quadrotor-group library
 * (paper_2308_12698_b200/libswarmstep_b200.so).
 *
 * The reference (swarmstep, /root/reference/pkg/src/swarmstep) has no FFI:
 * its World duck-types homogeneous groups (core.py:308-318, 455-475) and the
 * quadrotor group's hot path is QuadGroup.step (core.py:166-202).  These
 * entry points are what that group protocol needs underneath; the Python
 * host class paper_2308_12698_b200.group.B200QuadGroup binds them with
 * ctypes and implements the reference's group protocol on top.
 *
 * Conventions
 *  - Plain pointers and sizes only.  Device memory is borrowed (the caller
 *    owns it); nothing here allocates except the library's own error string.
 *  - Every call returns an int status: SWARMSTEP_OK (0) or a negative code;
 *    swarmstep_last_error() returns the thread-local message.  Nothing throws
 *    across the ABI.
 *  - `stream` is a cudaStream_t passed as void*; every launch is async on it.
 *    Calls on distinct streams over distinct groups are thread-safe.
 *  - State is a tiled structure of arrays ("AoSoA") of float32: one column
 *    per scalar component, agents grouped in tiles of SWARMSTEP_TILE = 128;
 *    a tile stores its SWARMSTEP_NCOL columns contiguously (17,408 bytes),
 *    so element (column c, row r) is
 *        cols[(r / 128) * (NCOL * 128) + c * 128 + r % 128].
 *    A warp's access to one component is one 128-byte line, every column
 *    offset inside a tile is a compile-time constant, and a tile's inputs
 *    (or outputs) are one contiguous block for a single TMA bulk copy.
 *    `stride` is the row capacity (>= n, multiple of 128); rows in
 *    [n, stride) must have flags == 0 (dead padding).
 */
#ifndef SWARMSTEP_B200_H
#define SWARMSTEP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SWARMSTEP_ABI_VERSION 3

enum {
    SWARMSTEP_OK = 0,
    SWARMSTEP_EINVAL = -1,   /* bad argument (maps to ValidationError) */
    SWARMSTEP_ECUDA = -2,    /* CUDA launch / runtime error            */
    SWARMSTEP_ENODEV = -3    /* no usable sm_100 device                */
};

/* per-row flag byte (the reference's alive / has_prev / cmd_level columns:
 * state.py:57-65, control.py:100-104, core.py:98-104) */
#define SWARMSTEP_FLAG_ALIVE     0x01u
#define SWARMSTEP_FLAG_HAS_PREV  0x02u
#define SWARMSTEP_LEVEL_SHIFT    2
#define SWARMSTEP_LEVEL_MASK     0x0Cu
enum { SWARMSTEP_LEVEL_POS = 0, SWARMSTEP_LEVEL_RATE = 1, SWARMSTEP_LEVEL_MOTOR = 2 }; /* core.py:73 */

/* Per-type constants, float32 (QuadParams quad.py:39-69, PidGains
 * control.py:40-53, OuterGains control.py:56-68).  G / G_inv are the 4x4
 * allocation matrix and its inverse (quad.py:106-122), row-major. */
typedef struct swarmstep_quad_params {
    float m, inv_m, g;
    float inv_ixx, inv_iyy, inv_izz;
    float ixx, iyy, izz;
    float k_t, omega_max, f_max, fc_max;      /* fc_max = 4 * f_max (control.py:253) */
    float G[16];
    float G_inv[16];
    float kp[3], ki[3], kd[3], i_limit[3];
    float kp_pos[3], kv[3], k_att[3];
    float omega_sp_max, a_cmd_min;
    float _pad[2];
} swarmstep_quad_params;

/* Physical constants and controller gains in float64, for hosts that do not
 * pack swarmstep_quad_params themselves: QuadParams (quad.py:39-69),
 * PidGains (control.py:40-53) and OuterGains (control.py:56-68). */
typedef struct swarmstep_quad_physics {
    double m, ixx, iyy, izz, g, k_t, k_q, arm_length, arm_angle, omega_max;
} swarmstep_quad_physics;
typedef struct swarmstep_quad_gains {
    double kp[3], ki[3], kd[3], i_limit[3];
    double kp_pos[3], kv[3], k_att[3];
    double omega_sp_max, a_cmd_min;
} swarmstep_quad_gains;

/* Column offsets inside a tile (each block is k consecutive columns).  The
 * order puts everything the step kernel reads first (cols [0, 27)) and keeps
 * the columns it writes in two runs ([0, 20) and [27, 31)).
 * COL_POS_LO is ONE 32-bit word per row holding the compensated-position
 * low parts of x, y, z: bits [10 i, 10 i + 10) = signed q_i, and
 * lo_i = q_i * ulp(hi_i) / 512 (ulp of the float32 position word hi_i; the
 * unit is floored at 2^-126, the smallest normal float; ssb::pos_lo_* in
 * csrc/common.cuh).
 * |lo| <= ulp(hi)/2 always holds, so |q| <= 256: position carries 33
 * significant bits in 4 bytes instead of 12. */
#define SWARMSTEP_TILE 128
enum {
    SWARMSTEP_COL_POS = 0,      /* px py pz          (state.py:57)          */
    SWARMSTEP_COL_VEL = 3,      /* vx vy vz                                 */
    SWARMSTEP_COL_QUAT = 6,     /* qw qx qy qz (scalar-first Hamilton)      */
    SWARMSTEP_COL_OMEGA = 10,   /* wx wy wz (body rates)                    */
    SWARMSTEP_COL_POS_LO = 13,  /* packed compensated-position low parts    */
    SWARMSTEP_COL_INTEGRAL = 14,/* RatePidState.integral (control.py:103)   */
    SWARMSTEP_COL_PREV = 17,    /* RatePidState.prev_omega                  */
    SWARMSTEP_COL_CMD = 20,     /* QuadGroup.cmd_values[0..6] (core.py:99)  */
    SWARMSTEP_COL_SP = 27,      /* QuadGroup.omega_sp xyz, f_c_sp (core.py:109-110) */
    SWARMSTEP_COL_OVERLAY = 31, /* QuadGroup.v_overlay (core.py:106)        */
    SWARMSTEP_NCOL = 34
};

/* A borrowed view of one group's device columns. */
typedef struct swarmstep_group_view {
    int64_t n;              /* live rows                                    */
    int64_t stride;         /* row capacity (>= n, multiple of 128)         */
    float *cols;            /* [stride/128][SWARMSTEP_NCOL][128] float32    */
    uint8_t *flags;         /* [stride], 2-byte aligned                     */
    uint32_t *counters;     /* device [4]: 0 faults logged (monotonic), 1 retarget count, 2 viewer count */
    uint64_t *fault_log;    /* device [fault_cap]: (tick << 40) | row       */
    int64_t fault_cap;
    int32_t compensated;    /* 1: position = hi + lo (COL_POS_LO in use)    */
    int32_t _pad;
} swarmstep_group_view;

/* Library / device info.  Returns SWARMSTEP_ABI_VERSION. */
int swarmstep_abi_version(void);
/* Message of the calling thread's last non-zero status: the text of the
 * exception the reference would raise (errors.py ValidationError /
 * InvalidStateError; bindings map the status code back to that class). */
const char *swarmstep_last_error(void);
/* Loads every kernel of the library on the current device (no side effects);
 * call before capturing launches into a CUDA graph.  Infrastructure, no
 * reference counterpart (likewise memcpy_async, stream_sync, device_info and
 * the *_workspace_bytes queries below). */
int swarmstep_preload(void);

/* Packs the kernel's float32 per-type constants: G and its exact inverse
 * (G^-1 = G^T diag(1/|row|^2), the rows of the X-geometry G being orthogonal;
 * quad.py:106-122), f_max = k_t omega_max^2, fc_max = 4 f_max (control.py:253),
 * 1/m, 1/I and the gains.  Host-only (no device needed).  Errors as
 * QuadParams: non-positive / non-finite constants or a singular geometry ->
 * SWARMSTEP_EINVAL (quad.py:56-60). */
int swarmstep_quad_params_init(swarmstep_quad_params *p, const swarmstep_quad_physics *phys,
                               const swarmstep_quad_gains *gains);

/* Host-side plumbing for thin bindings: an async copy of `bytes` on `stream`
 * (cudaMemcpyDefault: any direction, pinned host or device pointers), and a
 * stream synchronisation that also reports any error the stream's work
 * raised (SWARMSTEP_ECUDA + message). */
int swarmstep_memcpy_async(void *dst, const void *src, uint64_t bytes, void *stream);
int swarmstep_stream_sync(void *stream);
/* Fills sm count and compute capability of the current device. */
int swarmstep_device_info(int *sm_count, int *cc_major, int *cc_minor);

/* One launch = k_substeps successive QuadGroup.step(dt) calls
 * (core.py:166-202) with commands held fixed: setpoint selection by level,
 * position_outer_loop (control.py:222-294), rate_pid_step (control.py:136-187),
 * mix_to_motors (quad.py:143-168), raw-motor override (core.py:189-197) and
 * rk4_step (quad.py:350-437) including fault revert + kill.  The overlay
 * column block is added to v_sp on substep 0 only with SWARMSTEP_STEP_OVERLAY
 * (core.py:172-175, 199-201); the caller clears it afterwards.  Without
 * SWARMSTEP_STEP_MOTOR no row may be at MOTOR level (the stale-setpoint
 * columns are then not read).  K = 1 launches run the direct kernel (HBM-bound
 * regime), K >= 2 the paired FFMA2 kernel (FP32-bound); FORCE_* select one.
 * Faulted rows are appended to fault_log as ((tick_base + substep) mod 2^24)
 * << 40 | row and counted in counters[0], which only ever grows: a row can
 * fault at most once (dead rows never revive), so fault_cap >= n never
 * overflows and no per-launch reset is needed.
 * Replaces: QuadGroup.step (core.py:166).  Errors: dt <= 0 or k < 1 ->
 * SWARMSTEP_EINVAL (quad.py:359-360, control.py:154-155). */
/* launch_flags for swarmstep_quad_step */
#define SWARMSTEP_STEP_OVERLAY       0x1  /* add the overlay block to v_sp on tick 0      */
#define SWARMSTEP_STEP_MOTOR         0x2  /* some row may be at MOTOR level               */
#define SWARMSTEP_STEP_FORCE_DIRECT  0x4  /* tuning: force the direct-load kernel         */
#define SWARMSTEP_STEP_FORCE_TMA     0x8  /* tuning: force the TMA-staged kernel          */
#define SWARMSTEP_STEP_FORCE_PAIR    0x10 /* tuning: force the paired FFMA2 kernel        */
int swarmstep_quad_step(const swarmstep_group_view *g, const swarmstep_quad_params *p,
                        float dt, int k_substeps, int launch_flags, uint32_t tick_base,
                        const int64_t *tick_dev, void *stream);

/* swarmstep_quad_step (tick_dev = NULL) for launches issued back to back on
 * one stream: the launch may start while the previous overlapped launch of the
 * same group is still finishing (programmatic dependent launch), each 128-row
 * tile waiting only for ITS tile of the previous launch.  tile_epoch: one
 * uint32 per tile (stride / 128), zeroed once, owned by the group; the launch
 * waits until tile_epoch[t] >= wait_epoch (0: no wait -- the first overlapped
 * launch) and stores set_epoch (non-zero, after wait_epoch in wrapping order)
 * when tile t is done.  Kernels other than these step launches keep full
 * stream ordering, so commands, setpoints or reads enqueued in between need
 * nothing special.  Not for CUDA-graph capture (the epochs are per launch) and
 * not with SWARMSTEP_STEP_FORCE_TMA.  Same results as swarmstep_quad_step.
 * A tile that waits ~18 s for its epoch traps (a broken chain fails loudly
 * instead of hanging): keep overlapped launches to K <= 4096 ticks, and never
 * pass wait_epoch = 0 after an overlapped launch on the same stream. */
int swarmstep_quad_step_overlapped(const swarmstep_group_view *g, const swarmstep_quad_params *p,
                                   float dt, int k_substeps, int launch_flags, uint32_t tick_base,
                                   uint32_t *tile_epoch, uint32_t wait_epoch, uint32_t set_epoch,
                                   void *stream);

/* The synchronous World tick in one call: swarmstep_quad_step(..., tick_dev =
 * NULL, ...), then the four counters copied to counters_host (pinned host
 * memory) and the stream synchronised.  counters_host[0] is the fault-log
 * count after the launch (QuadGroup.step returns the ids, core.py:166-202). */
int swarmstep_quad_step_collect(const swarmstep_group_view *g, const swarmstep_quad_params *p,
                                float dt, int k_substeps, int launch_flags, uint32_t tick_base,
                                uint32_t *counters_host, void *stream);

/* swarmstep_quad_step with the device circle strategy evaluated per tick
 * inside the kernel (circle_swarm_strategy client.py:55-73 -> circle_reference
 * control.py:297-315, as swarmstep_quad_circle_setpoints computes it): tick k
 * of the launch puts every alive row at POS level with the circle setpoint of
 * t = (*tick_dev + tick_base + k) * feed->dt and phase phase0 + dphase * row,
 * so K ticks of a time-varying reference fuse into one launch, bit-identical
 * to K x (swarmstep_quad_circle_setpoints + a 1-tick step).  The command
 * columns are left holding the last tick's setpoints.  No overlay.
 * launch_flags: SWARMSTEP_STEP_FORCE_DIRECT / _FORCE_PAIR as for
 * swarmstep_quad_step (default: the paired FFMA2 kernel from K >= 2). */
typedef struct swarmstep_circle_feed {
    double dt, radius, omega, z, phase0, dphase;
} swarmstep_circle_feed;
int swarmstep_quad_step_circle(const swarmstep_group_view *g, const swarmstep_quad_params *p, float dt,
                               int k_substeps, int launch_flags, uint32_t tick_base, const int64_t *tick_dev,
                               const swarmstep_circle_feed *feed, void *stream);
/* swarmstep_quad_step_circle whose back-to-back launches overlap, with the
 * tile_epoch / wait_epoch / set_epoch chain of swarmstep_quad_step_overlapped
 * (the two share one chain per group). */
int swarmstep_quad_step_circle_overlapped(const swarmstep_group_view *g, const swarmstep_quad_params *p, float dt,
                                          int k_substeps, int launch_flags, uint32_t tick_base,
                                          const int64_t *tick_dev, const swarmstep_circle_feed *feed,
                                          uint32_t *tile_epoch, uint32_t wait_epoch, uint32_t set_epoch,
                                          void *stream);

/* swarmstep_quad_step with the opt-in first-order rotor lag of the north star
 * (absent in the reference; tau_m = 0 is swarmstep_quad_step
 * itself).  Each rotor thrust f_i follows its commanded thrust u_i (the
 * mixer's clamped motor thrust, or k_t clip(rpm)^2 for MOTOR rows), held over
 * the tick: f(t + s) = u + (f(t) - u) exp(-s / tau_m); the rigid body
 * integrates (wrench held, as QuadGroup.step) the wrench of the tick-mean
 * thrust u + (f(t) - u)(tau_m/dt)(1 - exp(-dt/tau_m)): the thrust impulse is
 * exact and tau_m -> 0 recovers the instantaneous mixer.  motor: device float32, tiled like
 * the state -- 4 columns x 128 rows per tile, stride rows, 16-byte aligned;
 * rotor i of row r at (r / 128) * 512 + i * 128 + r % 128 (newtons).  Dead
 * and faulted rows keep their thrusts.  Errors: tau_m <= 0 or non-finite,
 * dt <= 0, k < 1 -> SWARMSTEP_EINVAL.  No reference interface: this extends
 * QuadGroup.step (core.py:166) behind the same group protocol. */
int swarmstep_quad_step_lag(const swarmstep_group_view *g, const swarmstep_quad_params *p,
                            float *motor, float tau_m, float dt, int k_substeps, int launch_flags,
                            uint32_t tick_base, const int64_t *tick_dev, void *stream);

/* Latest-wins command scatter (QuadGroup.apply_command, core.py:117-135).
 * rows[i] (int64), levels[i] (uint8, SWARMSTEP_LEVEL_*), values[i*7..]
 * (float32; RATE/MOTOR entries carry 4 values and zeros) are device arrays;
 * rows must be unique.  Dead rows are skipped on device as well. */
int swarmstep_quad_apply_commands(const swarmstep_group_view *g, const int64_t *rows,
                                  const uint8_t *levels, const float *values,
                                  int64_t count, void *stream);

/* Bulk device setpoints: every row in [row0, row0+count) gets `level` and
 * values from the plain column block `values` ([7][ld] float32, device), alive
 * rows only.  Replaces one QuadGroup.apply_command (core.py:117-135) per agent
 * for whole swarms: the device-resident setpoint feed. */
int swarmstep_quad_set_setpoints(const swarmstep_group_view *g, int64_t row0, int64_t count,
                                 int level, const float *values, int64_t ld, void *stream);

/* mark_dead (core.py:151-158): rows[i] unique device int64; was_alive[i]
 * (uint8, device) receives 1 where the row was alive before the call. */
int swarmstep_quad_mark_dead(const swarmstep_group_view *g, const int64_t *rows,
                             uint8_t *was_alive, int64_t count, void *stream);

/* retarget_waypoint (core.py:141-149): alive rows with |p - point| < radius
 * switch to POS level with p_sp = point, v_sp = 0, yaw_sp = quat_yaw(q)
 * (quat.py:139-143).  counters[1] += number of rows retargeted. */
int swarmstep_quad_retarget_waypoint(const swarmstep_group_view *g, const double *point3,
                                     double radius, void *stream);

/* Viewer ATTRACT / REPEL influence (World._apply_viewer_input, core.py:445-453)
 * on the device: for alive rows with 1e-12 < d = |point - p| < radius the
 * overlay columns get += float32(gain * (1 - d/radius) / d * (point - p)),
 * evaluated in float64 in viewer_velocity_offsets' order (wire.py:320-340);
 * gain = +strength (attract) or -strength (repel).  counters[2] += rows whose
 * offset is non-zero, the reference's `offsets.any()` gate for
 * add_velocity_overlay.  The caller zeroes the overlay columns first when no
 * overlay is pending.  radius <= 0 is a no-op (wire.py:331). */
int swarmstep_quad_viewer_overlay(const swarmstep_group_view *g, const double *point3,
                                  double radius, double gain, void *stream);

/* Device-side snapshot packing (batch_snapshot, state.py:193-204): writes
 * float64 row-major pos (n,3), vel (n,3), quat (n,4), omega (n,3) and
 * alive (n,) u8 / level (n,) u8 into the device buffers given (any may be
 * NULL).  Position is hi + lo when compensated. */
int swarmstep_quad_pack_f64(const swarmstep_group_view *g, double *pos, double *vel,
                            double *quat, double *omega, uint8_t *alive, void *stream);

/* Inverse of the above (the state a group is built from: batch_create,
 * state.py:143-190): loads float64 row-major host-layout columns (device
 * pointers) into the float32 SoA columns, splitting position into hi + lo
 * when compensated.  Flags: alive from `alive` (u8); has_prev and level
 * left unchanged (a new group's flags start at 0: no previous sample). */
int swarmstep_quad_unpack_f64(const swarmstep_group_view *g, const double *pos,
                              const double *vel, const double *quat, const double *omega,
                              const uint8_t *alive, void *stream);

/* ---- the reference's function-level API (SURVEY 8(b) kernel-level) -------
 * One thread per row on the reference's own row-major layout: float32 (n,3)
 * pos / vel / omega / tau, (n,4) quat, (n,) f_c, u8 alive / flags; all
 * device pointers.  pos_lo (nullable): float32 low words of the positions
 * (float64 host positions split hi + lo), carried like the group's columns. */

/* dynamics_deriv (quad.py:320-335): derivative of every alive row; dead rows
 * (alive[r] == 0; alive may be NULL = all alive) get exactly zero. */
int swarmstep_op_deriv(int64_t n, const float *pos, const float *vel, const float *quat, const float *omega,
                       const uint8_t *alive, const float *f_c, const float *tau, const swarmstep_quad_params *p,
                       float *dpos, float *dvel, float *dquat, float *domega, void *stream);

/* rk4_step (quad.py:350-437): one step in place for alive rows; a row whose
 * result is non-finite (or has a zero quaternion norm) keeps its pre-step
 * state, gets alive = 0 and fault = 1.  dt <= 0 -> SWARMSTEP_EINVAL. */
int swarmstep_op_rk4(int64_t n, float *pos, float *pos_lo, float *vel, float *quat, float *omega, uint8_t *alive,
                     const float *f_c, const float *tau, const swarmstep_quad_params *p, float dt, uint8_t *fault,
                     void *stream);

/* mix_to_motors (quad.py:143-168): motors (n,4) clamped to [0, f_max],
 * realized (n,4) = (f_c, tau) the clamped motors produce (the request itself
 * for unsaturated rows), saturated (n,). */
int swarmstep_op_mix(int64_t n, const float *f_c, const float *tau, const swarmstep_quad_params *p, float *motors,
                     float *realized, uint8_t *saturated, void *stream);

/* rotor_thrust_torque (quad.py:130-140), elementwise over `count` speeds. */
int swarmstep_op_rotor(int64_t count, const float *rpm, float k_t, float k_q, float omega_max, float *thrust,
                       float *torque, uint8_t *saturated, void *stream);

/* rate_pid_step (control.py:136-187): updates integral / prev_omega /
 * has_prev in place, writes tau (n,3) and f_c (n,); dead rows: frozen state,
 * zero output.  dt <= 0 -> SWARMSTEP_EINVAL. */
int swarmstep_op_pid(int64_t n, const float *omega, const float *omega_sp, const float *f_c_sp,
                     const swarmstep_quad_params *p, float dt, float *integral, float *prev_omega, uint8_t *has_prev,
                     const uint8_t *alive, float *tau_out, float *f_c_out, void *stream);

/* position_outer_loop (control.py:222-294): omega_sp (n,3), f_c_sp (n,),
 * low (n,) free-fall floor flag; dead rows get zeros.  Non-finite inputs are
 * the caller's to reject (the reference raises InvalidStateError). */
int swarmstep_op_outer(int64_t n, const float *pos, const float *pos_lo, const float *vel, const float *quat,
                       const uint8_t *alive, const float *p_sp, const float *v_sp, const float *yaw_sp,
                       const swarmstep_quad_params *p, float *omega_sp, float *f_c_sp, uint8_t *low, void *stream);

/* ---- neighbour-coupled swarm controller (config 5) --------- */

/* Packs the alive rows' positions as float4 (x, y, z, 0) -- NaN for dead rows
 * and for padding rows [n, n_out) -- into out_xyzw (device, n_out float4):
 * the per-rank contribution to the NCCL all-gather (the alive-only gather of
 * collision.py:66-80, by rank). */
int swarmstep_pack_positions(const swarmstep_group_view *g, float *out_xyzw, int64_t n_out,
                             void *stream);

/* Device workspace needed by swarmstep_neighbor_overlay for n_all agents. */
int swarmstep_neighbor_workspace_bytes(int64_t n_all, uint64_t *bytes);

/* Separation overlay for the local rows from all gathered positions:
 *   v_i += sum_{j != i, alive, |p_i - p_j| < r_sense} k_sep (1 - d/r_sense) (p_i - p_j)/d
 * (wire.py:320-340 repel field per neighbour, strict < as collision.py:166).
 * Local row r is gathered row self_offset + r.  Linear spatial hash (cell >=
 * r_sense), counting sort by bucket, 27-cell scan in 9 contiguous x-rows;
 * writes (or adds, accumulate != 0) the overlay column block.  Sums in 64-bit
 * fixed point: bit-deterministic.  |k_sep| < 2^30. */
int swarmstep_neighbor_overlay(const swarmstep_group_view *g, const float *all_xyzw, int64_t n_all,
                               int64_t self_offset, float r_sense, float k_sep, float cell,
                               int accumulate, void *workspace, uint64_t ws_bytes,
                               const uint32_t *slot_epoch, void *stream);
/* all_xyzw = NULL: a single rank reads its own rows from the columns (n_all
 * == n, self_offset 0) -- no pack pass, same bits as packing first.
 * slot_epoch: NULL (all_xyzw holds n_all float4), or the device epoch counter
 * of the P2P exchange below (all_xyzw is its double buffer; the kernels read
 * slot (*slot_epoch & 1), n_all float4 each). */

/* The position all-gather fused into the pack kernel, over peer memory
 * (NVLink P2P stores into every rank's symmetric buffer) -- the NCCL-free
 * exchange of config 5.  peer_bufs: device array [world] of the ranks'
 * double buffers (2 * world * n_pad float4 each); this rank's rows land at
 * slot (E & 1), offset rank * n_pad, in every buffer, E = *epoch + 1.
 * peer_signals: device array [world] of the ranks' signal pads (>= world
 * uint32, zero-initialised); the last block release-stores E into
 * peer_signals[q][rank] after a system fence.  arrive: this rank's device
 * block counter (zero-initialised, left at zero).  swarmstep_p2p_wait then
 * spins (acquire) until every writer's signal reached E and sets *epoch = E
 * (it traps after 10 s without a peer instead of hanging).  Replaces:
 * swarmstep_pack_positions + ncclAllGather (parallel.py NeighborSeparation). */
int swarmstep_p2p_pack_push(const swarmstep_group_view *g, void *const *peer_bufs, int world, int rank,
                            int64_t n_pad, uint32_t *const *peer_signals, const uint32_t *epoch,
                            uint32_t *arrive, void *stream);
int swarmstep_p2p_wait(const uint32_t *local_signals, int world, uint32_t *epoch, void *stream);

/* Single-process form of the fused exchange (one host process driving several
 * shards: MultiDeviceQuadGroup, the drop-in for the single-process World,
 * core.py:308-505).  Packs this shard's rows as float4 (NaN for dead / padding
 * rows) straight into EVERY shard's gathered buffer: bufs is a device array
 * [world] of float4 buffers, rows land at offset + rank * n_pad.  No signals:
 * the caller orders each reader after every writer with CUDA events.  Buffers
 * on other devices need swarmstep_enable_peer_access(reader_dev, writer_dev)
 * first (NVLink peer stores). */
int swarmstep_pack_scatter(const swarmstep_group_view *g, void *const *bufs, int world, int rank, int64_t n_pad,
                           int64_t offset, void *stream);

/* cudaDeviceEnablePeerAccess(peer) from `device` (idempotent; OK for device
 * == peer).  SWARMSTEP_ENODEV when the pair has no peer access. */
int swarmstep_enable_peer_access(int device, int peer);

/* ---- device-resident setpoint feed ---------------------- */

/* circle_swarm_strategy (client.py:55-73) + circle_reference (control.py:
 * 297-315) on the device: every alive row r gets POS level and
 *   th = omega t + phase0 + r dphase,  t = (*tick_dev + tick_offset) dt,
 *   p_sp = (R cos th, R sin th, z), v_sp = (-R omega sin th, R omega cos th, 0),
 *   yaw_sp = th + copysign(pi/2, omega)   (angles reduced mod 2 pi).
 * The reference layout uses phase0 = 0, dphase = 2 pi / n (client.py:43-52).
 * Reading the tick from device memory lets a run of ticks be one CUDA graph. */
int swarmstep_quad_circle_setpoints(const swarmstep_group_view *g, const int64_t *tick_dev,
                                    int64_t tick_offset, double dt, double radius, double omega,
                                    double z, double phase0, double dphase, void *stream);

/* *tick_dev += delta (one thread; graph-capturable tick counter: the device
 * copy of SimClock.tick, state.py:24-40). */
int swarmstep_tick_add(int64_t *tick_dev, int64_t delta, void *stream);

/* ---- device snapshot packing ----------------------------- */

/* Swarm-wide reductions over one group (World.alive_counts core.py:370,
 * cli.py:161; the occupied extent of collision.py:124-128), one launch:
 * out12 (device double[12]) = alive count, sum of alive positions (x, y, z),
 * sum of |v|^2, max |v|^2, alive bounding box min (x, y, z), max (x, y, z)
 * (+inf / -inf when no row is alive).  Warp-shuffle + shared-memory block
 * reduction, last-block fold of the block partials in block order:
 * deterministic.  workspace: >= swarmstep_swarm_stats_workspace_bytes()
 * bytes, 16-byte aligned, ZEROED once at allocation (its ticket word is left
 * at zero by every launch); one workspace per concurrent stream. */
int swarmstep_swarm_stats_workspace_bytes(uint64_t *bytes);
int swarmstep_quad_swarm_stats(const swarmstep_group_view *g, double *out12, void *workspace,
                               uint64_t ws_bytes, void *stream);

/* One group's SnapshotMsg section body (wire.py:162-178, PROTOCOL.md
 * "Snapshot (0x01)"): u64*n agent_ids | u8*n alive | f32*3n pos | f32*3n vel |
 * f32*4n quat (canonical, w >= 0) | f32*3n omega, little-endian, into `out`
 * (device, 8-byte aligned, 61*n bytes).  agent_ids: device uint64[n].
 * Bytes equal encode_snapshot of the group's float64 host mirror. */
int swarmstep_quad_pack_wire(const swarmstep_group_view *g, const uint64_t *agent_ids, uint8_t *out,
                             void *stream);

/* ---- GPU collision / neighbour detection ----------------- */

/* Gathers a group's rows as float64 (x, y, z, r) into xyzr[offset + row]
 * (r = NaN for dead rows, which the detector skips; _gather_alive,
 * collision.py:66-80); position is hi + lo. */
int swarmstep_pack_collision(const swarmstep_group_view *g, double radius, double *xyzr, int64_t offset,
                             void *stream);

/* Device workspace for swarmstep_collision_pairs over m gathered agents. */
int swarmstep_collision_workspace_bytes(int64_t m, uint64_t *bytes);

/* detect() (collision.py:110-176) over m gathered agents: grid cells of size
 * `cell`, candidate pairs = same-cell pairs (i < j) + the half-space cell
 * offsets given (int[3 * n_off], device; collision.py:86-95), narrow phase in
 * float64 with the reference's operation order.  Colliding pairs
 * (d2 < (r_i + r_j)^2) go to coll[2k], coll[2k+1] and neighbour pairs
 * (d2 < r_sense^2) to near[...] as gathered indices (i, j); counts_dev[0],
 * counts_dev[1] receive the pair counts and counts_dev[2] is non-zero if a
 * cell coordinate left (-2^20, 2^20).  Two calls: fill == 0 sorts, counts
 * the pairs per agent and scans the counts (nothing stored); fill == 1, with
 * the same inputs and the workspace left as the fill == 0 call left it,
 * stores the pairs (the first *_cap of each kind) at their scanned offsets --
 * no atomics, deterministic order. */
int swarmstep_collision_pairs(const double *xyzr, int64_t m, double cell, const int *offsets_dev, int n_off,
                              double r_sense, uint32_t *coll, uint64_t coll_cap, uint32_t *near,
                              uint64_t near_cap, uint64_t *counts_dev, void *workspace, uint64_t ws_bytes,
                              int fill, void *stream);

/* ---- unicycle group -------------------------------------- */

/* k_substeps ticks of unicycle_step (core.py:221-246) for every alive row:
 * (v, w) = clip(cmd cols 0, 1) (+ overlay projected on the heading on tick 0
 * with SWARMSTEP_STEP_OVERLAY, core.py:277-283); exact-arc xy update, yaw
 * quaternion, vel = v (cos th1, sin th1, 0), omega_z = w.  Layout as the quad
 * group (tiled SoA, COL_CMD + 0 / + 1 hold v / w). */
int swarmstep_unicycle_step(const swarmstep_group_view *g, float v_max, float omega_max, float dt,
                            int k_substeps, int launch_flags, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SWARMSTEP_B200_H */
