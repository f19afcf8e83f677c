// neighbors.cu -- neighbour-coupled swarm controller support (config 5).
//
// The reference has no swarm-level controller; the one built
// here follows the survey's definition: a separation velocity overlay
//     v_i += sum_{j != i, alive, d_ij < r} k (1 - d_ij / r) (p_i - p_j) / d_ij
// i.e. the viewer "repel" influence field of wire.py:320-340 applied per
// neighbour, with the strict "<" neighbour test of collision.py:166 and the
// zero-distance guard of wire.py:335.  It feeds the existing one-tick overlay
// input of the group (core.py:137-139, 172-175).
//
// Pipeline per tick (one process per GPU): pack the local shard's positions
// (float4, NaN for dead rows) -> NCCL all-gather across ranks (host side,
// torch.distributed) -> spatial hash of every gathered agent -> radix sort
// (CUB) -> bucket ranges -> per local agent, scan the 27 neighbouring cells.
// Summation order is fixed (cell order, then agent index), so results are
// bit-deterministic.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"

namespace {

int nb_err(int code, const char *msg) { return ssb::set_err(code, msg); }
int nb_cuda(const char *where) { return ssb::cuda_status(where); }

__device__ __forceinline__ uint32_t cell_hash(int ix, int iy, int iz, uint32_t mask)
{
    return (((uint32_t)ix * 73856093u) ^ ((uint32_t)iy * 19349663u) ^ ((uint32_t)iz * 83492791u)) & mask;
}

__device__ __forceinline__ int cell_of(float x, float inv_cell)
{
    return (int)floorf(x * inv_cell);
}

uint64_t next_pow2(uint64_t x)
{
    uint64_t p = 1;
    while (p < x) p <<= 1;
    return p;
}

struct Workspace {
    uint32_t *keys, *vals, *keys_sorted, *vals_sorted, *cell_start, *cell_end;
    void *cub_tmp;
    size_t cub_bytes;
    uint32_t mask;
    int key_bits;
};

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// Lays the workspace out in one caller-provided buffer; returns its size.
size_t layout(int64_t n_all, char *base, Workspace *w)
{
    const uint64_t m = next_pow2((uint64_t)(2 * (n_all > 0 ? n_all : 1)));
    size_t cub_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, cub_bytes, (uint32_t *)nullptr, (uint32_t *)nullptr,
                                    (uint32_t *)nullptr, (uint32_t *)nullptr, (int)n_all);
    size_t off = 0;
    const size_t nb = align256(sizeof(uint32_t) * (size_t)n_all), mb = align256(sizeof(uint32_t) * m);
    if (w) {
        w->keys = (uint32_t *)(base + off);
        w->vals = (uint32_t *)(base + off + nb);
        w->keys_sorted = (uint32_t *)(base + off + 2 * nb);
        w->vals_sorted = (uint32_t *)(base + off + 3 * nb);
        w->cell_start = (uint32_t *)(base + off + 4 * nb);
        w->cell_end = (uint32_t *)(base + off + 4 * nb + mb);
        w->cub_tmp = base + off + 4 * nb + 2 * mb;
        w->cub_bytes = cub_bytes;
        w->mask = (uint32_t)(m - 1);
        int bits = 0;
        while ((1ull << bits) <= m) bits++;   // keys in [0, m], m = sentinel
        w->key_bits = bits;
    }
    return 4 * nb + 2 * mb + align256(cub_bytes);
}

__global__ void pack_positions_kernel(const float *cols, const uint8_t *flags, int64_t n, int64_t stride,
                                      int compensated, int64_t n_out, float4 *out)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_out) return;
    float4 p = make_float4(__int_as_float(0x7fc00000), __int_as_float(0x7fc00000), __int_as_float(0x7fc00000), 0.0f);
    if (r < n && (flags[r] & SWARMSTEP_FLAG_ALIVE)) {
        float x = cols[ssb::at(SWARMSTEP_COL_POS + 0, r)];
        float y = cols[ssb::at(SWARMSTEP_COL_POS + 1, r)];
        float z = cols[ssb::at(SWARMSTEP_COL_POS + 2, r)];
        if (compensated) {
            x += cols[ssb::at(SWARMSTEP_COL_POS_LO + 0, r)];
            y += cols[ssb::at(SWARMSTEP_COL_POS_LO + 1, r)];
            z += cols[ssb::at(SWARMSTEP_COL_POS_LO + 2, r)];
        }
        p = make_float4(x, y, z, 0.0f);
    }
    out[r] = p;
}

__global__ void hash_kernel(const float4 *pos, int64_t n_all, float inv_cell, uint32_t mask,
                            uint32_t *keys, uint32_t *vals)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_all) return;
    const float4 p = pos[i];
    // dead / padding rows (NaN) sort past every bucket
    keys[i] = isnan(p.x) ? mask + 1 : cell_hash(cell_of(p.x, inv_cell), cell_of(p.y, inv_cell),
                                                 cell_of(p.z, inv_cell), mask);
    vals[i] = (uint32_t)i;
}

__global__ void bucket_ranges_kernel(const uint32_t *keys_sorted, int64_t n_all, uint32_t mask,
                                     uint32_t *cell_start, uint32_t *cell_end)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_all) return;
    const uint32_t k = keys_sorted[i];
    if (k > mask) return;
    if (i == 0 || keys_sorted[i - 1] != k) cell_start[k] = (uint32_t)i;
    if (i == n_all - 1 || keys_sorted[i + 1] != k) cell_end[k] = (uint32_t)(i + 1);
}

__global__ void query_kernel(const float4 *pos, const uint32_t *vals_sorted, const uint32_t *cell_start,
                             const uint32_t *cell_end, uint32_t mask, float inv_cell, float r_sense,
                             float k_sep, int64_t n_local, int64_t self_offset, int64_t stride,
                             const uint8_t *flags, float *cols, int accumulate)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_local) return;
    float ax = 0.0f, ay = 0.0f, az = 0.0f;
    const int64_t self = self_offset + r;
    if (flags[r] & SWARMSTEP_FLAG_ALIVE) {
        const float4 p = pos[self];
        const int cx = cell_of(p.x, inv_cell), cy = cell_of(p.y, inv_cell), cz = cell_of(p.z, inv_cell);
        uint32_t seen[27];
        int nseen = 0;
        const float inv_r = 1.0f / r_sense;
        for (int dz = -1; dz <= 1; dz++)
            for (int dy = -1; dy <= 1; dy++)
                for (int dx = -1; dx <= 1; dx++) {
                    const uint32_t b = cell_hash(cx + dx, cy + dy, cz + dz, mask);
                    bool dup = false;
                    for (int s = 0; s < nseen; s++) dup = dup || (seen[s] == b);
                    if (dup) continue;          // two neighbour cells share a bucket
                    seen[nseen++] = b;
                    const uint32_t e = cell_end[b];
                    for (uint32_t j = cell_start[b]; j < e; j++) {
                        const uint32_t idx = vals_sorted[j];
                        if ((int64_t)idx == self) continue;
                        const float4 q = pos[idx];
                        const float ddx = p.x - q.x, ddy = p.y - q.y, ddz = p.z - q.z;
                        const float d2 = fmaf(ddx, ddx, fmaf(ddy, ddy, ddz * ddz));
                        if (!(d2 < r_sense * r_sense) || !(d2 > 1e-24f)) continue;  // strict <, d > 1e-12
                        const float d = sqrtf(d2);
                        const float s = k_sep * (1.0f - d * inv_r) / d;
                        ax = fmaf(s, ddx, ax);
                        ay = fmaf(s, ddy, ay);
                        az = fmaf(s, ddz, az);
                    }
                }
    }
    float *ox = cols + ssb::at(SWARMSTEP_COL_OVERLAY + 0, r);
    float *oy = cols + ssb::at(SWARMSTEP_COL_OVERLAY + 1, r);
    float *oz = cols + ssb::at(SWARMSTEP_COL_OVERLAY + 2, r);
    if (accumulate) {
        *ox += ax; *oy += ay; *oz += az;
    } else {
        *ox = ax; *oy = ay; *oz = az;
    }
}

unsigned grid_n(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

}  // namespace

extern "C" {

int swarmstep_pack_positions(const swarmstep_group_view *g, float *out_xyzw, int64_t n_out, void *stream)
{
    if (!g || !g->cols || !g->flags || !out_xyzw) return nb_err(SWARMSTEP_EINVAL, "null argument");
    if (n_out < g->n) return nb_err(SWARMSTEP_EINVAL, "n_out < n");
    if (n_out == 0) return SWARMSTEP_OK;
    pack_positions_kernel<<<grid_n(n_out, 256), 256, 0, (cudaStream_t)stream>>>(
        g->cols, g->flags, g->n, g->stride, g->compensated, n_out, (float4 *)out_xyzw);
    return nb_cuda("pack_positions_kernel");
}

int swarmstep_neighbor_workspace_bytes(int64_t n_all, uint64_t *bytes)
{
    if (n_all < 0 || n_all > 0x7fffffffLL || !bytes) return nb_err(SWARMSTEP_EINVAL, "bad n_all");
    *bytes = (uint64_t)layout(n_all, nullptr, nullptr);
    return SWARMSTEP_OK;
}

int swarmstep_neighbor_overlay(const swarmstep_group_view *g, const float *all_xyzw, int64_t n_all,
                               int64_t self_offset, float r_sense, float k_sep, float cell, int accumulate,
                               void *workspace, uint64_t ws_bytes, void *stream)
{
    if (!g || !g->cols || !g->flags || !all_xyzw || !workspace) return nb_err(SWARMSTEP_EINVAL, "null argument");
    if (!(r_sense > 0.0f) || !(cell >= r_sense)) return nb_err(SWARMSTEP_EINVAL, "need r_sense > 0 and cell >= r_sense");
    if (self_offset < 0 || self_offset + g->n > n_all) return nb_err(SWARMSTEP_EINVAL, "local shard outside n_all");
    if (ws_bytes < (uint64_t)layout(n_all, nullptr, nullptr)) return nb_err(SWARMSTEP_EINVAL, "workspace too small");
    if (n_all == 0 || g->n == 0) return SWARMSTEP_OK;
    cudaStream_t s = (cudaStream_t)stream;
    Workspace w;
    layout(n_all, (char *)workspace, &w);
    const float inv_cell = 1.0f / cell;
    const float4 *pos = (const float4 *)all_xyzw;
    hash_kernel<<<grid_n(n_all, 256), 256, 0, s>>>(pos, n_all, inv_cell, w.mask, w.keys, w.vals);
    size_t cb = w.cub_bytes;
    if (cub::DeviceRadixSort::SortPairs(w.cub_tmp, cb, w.keys, w.keys_sorted, w.vals, w.vals_sorted,
                                        (int)n_all, 0, w.key_bits, s) != cudaSuccess)
        return nb_cuda("cub::DeviceRadixSort");
    cudaMemsetAsync(w.cell_start, 0, sizeof(uint32_t) * ((size_t)w.mask + 1), s);
    cudaMemsetAsync(w.cell_end, 0, sizeof(uint32_t) * ((size_t)w.mask + 1), s);
    bucket_ranges_kernel<<<grid_n(n_all, 256), 256, 0, s>>>(w.keys_sorted, n_all, w.mask, w.cell_start, w.cell_end);
    query_kernel<<<grid_n(g->n, 128), 128, 0, s>>>(pos, w.vals_sorted, w.cell_start, w.cell_end, w.mask, inv_cell,
                                                 r_sense, k_sep, g->n, self_offset, g->stride, g->flags, g->cols,
                                                 accumulate);
    return nb_cuda("neighbor overlay");
}

}  // extern "C"
