/*
 * c_host_demo.c -- the B200 hot path driven from plain C through the C ABI
 * (include/swarmstep_b200.h): no Python, no torch.  What a non-Python host of
 * the reference's group step does:
 *
 *   params_init -> cudaMalloc the tiled columns -> unpack the float64 state
 *   -> bulk POS setpoints -> K fused ticks per launch -> pack float64 back.
 *
 *   ./c_host_demo N K LAUNCHES [OUT]   prints one JSON line with a position
 *   checksum; OUT (optional) receives the final float64 positions (n x 3)
 *
 * tests/test_gpu_c_host.py runs the same workload through B200QuadGroup and
 * requires identical bits.
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "swarmstep_b200.h"

#define CHECK(call)                                                                  \
    do {                                                                             \
        int rc_ = (call);                                                            \
        if (rc_ != 0) {                                                              \
            fprintf(stderr, "%s failed (%d): %s\n", #call, rc_, swarmstep_last_error()); \
            return 1;                                                                \
        }                                                                            \
    } while (0)
#define CUDA(call)                                                                   \
    do {                                                                             \
        cudaError_t e_ = (call);                                                     \
        if (e_ != cudaSuccess) {                                                     \
            fprintf(stderr, "%s: %s\n", #call, cudaGetErrorString(e_));              \
            return 1;                                                                \
        }                                                                            \
    } while (0)

int main(int argc, char **argv)
{
    const int64_t n = argc > 1 ? atoll(argv[1]) : 1000;
    const int k = argc > 2 ? atoi(argv[2]) : 10;
    const int launches = argc > 3 ? atoi(argv[3]) : 10;
    const float dt = 1e-3f;

    /* per-type constants: the reference defaults (quad.py:47-65, control.py:63-80) */
    swarmstep_quad_physics phys = {1.0, 0.01, 0.01, 0.02, 9.81, 1e-8, 1e-10, 0.2, M_PI / 4.0, 40000.0};
    swarmstep_quad_gains gains = {{0.25, 0.25, 0.1}, {0.05, 0.05, 0.02}, {0.002, 0.002, 0.001}, {0.2, 0.2, 0.2},
                                  {16, 16, 16}, {8, 8, 8}, {12, 12, 3}, 20.0, 0.5};
    swarmstep_quad_params p;
    CHECK(swarmstep_quad_params_init(&p, &phys, &gains));

    /* host state: a grid at 10 m, hovering (layout_poses "grid", spacing 3 m) */
    const int64_t side = (int64_t)ceil(sqrt((double)n));
    double *pos = calloc((size_t)n * 3, sizeof(double)), *vel = calloc((size_t)n * 3, sizeof(double));
    double *quat = calloc((size_t)n * 4, sizeof(double)), *omega = calloc((size_t)n * 3, sizeof(double));
    uint8_t *alive = malloc((size_t)n);
    float *sp = malloc(sizeof(float) * 7 * (size_t)n);      /* [7][n] column block */
    for (int64_t r = 0; r < n; r++) {
        pos[3 * r] = 3.0 * (double)(r % side);
        pos[3 * r + 1] = 3.0 * (double)(r / side);
        pos[3 * r + 2] = 10.0;
        quat[4 * r] = 1.0;
        alive[r] = 1;
        /* setpoint: 0.5 m up and 0.25 m east of the start, yaw 0.1 rad */
        sp[0 * n + r] = (float)(pos[3 * r] + 0.25);
        sp[1 * n + r] = (float)pos[3 * r + 1];
        sp[2 * n + r] = (float)(pos[3 * r + 2] + 0.5);
        sp[3 * n + r] = sp[4 * n + r] = sp[5 * n + r] = 0.0f;
        sp[6 * n + r] = 0.1f;
    }

    /* device columns: tiled SoA, capacity rounded up to whole 128-row tiles */
    const int64_t stride = (n + SWARMSTEP_TILE - 1) / SWARMSTEP_TILE * SWARMSTEP_TILE;
    swarmstep_group_view g;
    memset(&g, 0, sizeof(g));
    g.n = n;
    g.stride = stride;
    g.fault_cap = n;
    g.compensated = 1;
    CUDA(cudaMalloc((void **)&g.cols, sizeof(float) * SWARMSTEP_NCOL * (size_t)stride));
    CUDA(cudaMemset(g.cols, 0, sizeof(float) * SWARMSTEP_NCOL * (size_t)stride));
    CUDA(cudaMalloc((void **)&g.flags, (size_t)stride));
    CUDA(cudaMemset(g.flags, 0, (size_t)stride));
    CUDA(cudaMalloc((void **)&g.counters, 4 * sizeof(uint32_t)));
    CUDA(cudaMemset(g.counters, 0, 4 * sizeof(uint32_t)));
    CUDA(cudaMalloc((void **)&g.fault_log, sizeof(uint64_t) * (size_t)n));
    cudaStream_t s;
    CUDA(cudaStreamCreate(&s));

    double *d_pos, *d_vel, *d_quat, *d_omega;
    uint8_t *d_alive;
    float *d_sp;
    CUDA(cudaMalloc((void **)&d_pos, sizeof(double) * 3 * (size_t)n));
    CUDA(cudaMalloc((void **)&d_vel, sizeof(double) * 3 * (size_t)n));
    CUDA(cudaMalloc((void **)&d_quat, sizeof(double) * 4 * (size_t)n));
    CUDA(cudaMalloc((void **)&d_omega, sizeof(double) * 3 * (size_t)n));
    CUDA(cudaMalloc((void **)&d_alive, (size_t)n));
    CUDA(cudaMalloc((void **)&d_sp, sizeof(float) * 7 * (size_t)n));
    CUDA(cudaMemcpy(d_pos, pos, sizeof(double) * 3 * (size_t)n, cudaMemcpyHostToDevice));
    CUDA(cudaMemcpy(d_vel, vel, sizeof(double) * 3 * (size_t)n, cudaMemcpyHostToDevice));
    CUDA(cudaMemcpy(d_quat, quat, sizeof(double) * 4 * (size_t)n, cudaMemcpyHostToDevice));
    CUDA(cudaMemcpy(d_omega, omega, sizeof(double) * 3 * (size_t)n, cudaMemcpyHostToDevice));
    CUDA(cudaMemcpy(d_alive, alive, (size_t)n, cudaMemcpyHostToDevice));
    CUDA(cudaMemcpy(d_sp, sp, sizeof(float) * 7 * (size_t)n, cudaMemcpyHostToDevice));

    CHECK(swarmstep_quad_unpack_f64(&g, d_pos, d_vel, d_quat, d_omega, d_alive, s));
    CHECK(swarmstep_quad_set_setpoints(&g, 0, n, 0 /* POS */, d_sp, n, s));
    /* argv[5] = 1: back-to-back launches overlap tile by tile (one zeroed
       epoch word per tile; launch l waits for epoch l, publishes l + 1) */
    const int overlap = argc > 5 ? atoi(argv[5]) : 0;
    uint32_t *d_epoch = NULL;
    if (overlap) {
        CUDA(cudaMalloc((void **)&d_epoch, sizeof(uint32_t) * (size_t)(stride / SWARMSTEP_TILE)));
        CUDA(cudaMemset(d_epoch, 0, sizeof(uint32_t) * (size_t)(stride / SWARMSTEP_TILE)));
    }
    for (int l = 0; l < launches; l++) {
        if (overlap)
            CHECK(swarmstep_quad_step_overlapped(&g, &p, dt, k, 0, (uint32_t)(l * k), d_epoch, (uint32_t)l,
                                                 (uint32_t)(l + 1), s));
        else
            CHECK(swarmstep_quad_step(&g, &p, dt, k, 0, (uint32_t)(l * k), NULL, s));
    }
    CHECK(swarmstep_quad_pack_f64(&g, d_pos, d_vel, d_quat, d_omega, d_alive, s));
    CHECK(swarmstep_stream_sync(s));
    CUDA(cudaMemcpy(pos, d_pos, sizeof(double) * 3 * (size_t)n, cudaMemcpyDeviceToHost));
    CUDA(cudaMemcpy(alive, d_alive, (size_t)n, cudaMemcpyDeviceToHost));
    uint32_t faults = 0;
    CUDA(cudaMemcpy(&faults, g.counters, sizeof(uint32_t), cudaMemcpyDeviceToHost));

    if (argc > 4) {
        FILE *f = fopen(argv[4], "wb");
        if (!f || fwrite(pos, sizeof(double), 3 * (size_t)n, f) != 3 * (size_t)n) {
            fprintf(stderr, "cannot write %s\n", argv[4]);
            return 1;
        }
        fclose(f);
    }
    double sum = 0.0;
    int64_t n_alive = 0;
    for (int64_t r = 0; r < n; r++) {
        sum += pos[3 * r] + 2.0 * pos[3 * r + 1] + 3.0 * pos[3 * r + 2];
        n_alive += alive[r];
    }
    printf("{\"n\": %lld, \"k\": %d, \"launches\": %d, \"pos_checksum\": %.17g, \"pos0\": [%.17g, %.17g, %.17g], "
           "\"alive\": %lld, \"faults\": %u, \"abi\": %d}\n",
           (long long)n, k, launches, sum, pos[0], pos[1], pos[2], (long long)n_alive, faults,
           swarmstep_abi_version());
    return 0;
}
