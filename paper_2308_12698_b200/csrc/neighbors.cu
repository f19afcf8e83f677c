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
// (float4, NaN for dead rows) -> all-gather across ranks (NCCL, or fused into
// the pack kernel over peer memory, exchange.cu) -> counting sort by spatial
// hash bucket: one kernel hashes every gathered agent and takes its rank in
// its bucket with an atomic counter, a CUB exclusive scan of the counts gives
// every bucket's start, one kernel scatters the positions into bucket order
// -> one thread per local agent, in bucket order, scans the 9 x-rows of its 27
// neighbouring cells.  The atomic ranks make the order inside a bucket vary
// run to run, so the overlay is summed in 64-bit fixed point (2^-32 m/s
// resolution): integer adds commute, and results are bit-deterministic.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <cub/device/device_scan.cuh>

#include "common.cuh"

namespace {

int nb_err(int code, const char *msg) { return ssb::set_err(code, msg); }
int nb_cuda(const char *where) { return ssb::cuda_status(where); }

// Linear cell hash h = ix + HB*iy + HC*iz (mod m, m a power of two >= 64).
// Being linear, the buckets of a cell's neighbours follow from its own bucket
// (h + dx + HB*dy + HC*dz), x-neighbours are CONSECUTIVE buckets (so the three
// cells of an x-row are one contiguous range of the sorted order), and with
// HB = 3, HC = 9 (mod 32) the 27 neighbours of any cell land in 27 distinct
// buckets for every m >= 32 (dx + 3dy + 9dz is injective on {-1,0,1}^3 with
// span 26 < 32), so no bucket is ever scanned twice.
constexpr uint32_t kHB = 0x8DA6B343u, kHC = 0xD8163849u;

__device__ __forceinline__ uint32_t cell_hash(int ix, int iy, int iz, uint32_t mask)
{
    return ((uint32_t)ix + (uint32_t)iy * kHB + (uint32_t)iz * kHC) & mask;
}

__device__ __forceinline__ int cell_of(float x, float inv_cell)
{
    return (int)floorf(x * inv_cell);
}

uint64_t next_pow2(uint64_t x)
{
    uint64_t p = 64;
    while (p < x) p <<= 1;
    return p;
}

struct Workspace {
    uint32_t *keys, *ranks, *keys_sorted, *vals_sorted;
    uint32_t *count;        // m + 1 bucket counts (bucket m: dead / padding rows)
    uint32_t *cell_start;   // m + 1 exclusive-scan starts: bucket k is [start[k], start[k+1])
    float4 *pos_sorted;     // alive positions in bucket order, .w = original index bits
    void *cub_tmp;
    size_t cub_bytes;
    uint32_t mask;
};

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// Lays the workspace out in one caller-provided buffer; returns its size.
size_t layout(int64_t n_all, char *base, Workspace *w)
{
    const uint64_t m = next_pow2((uint64_t)(2 * (n_all > 0 ? n_all : 1)));
    size_t cub_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, cub_bytes, (uint32_t *)nullptr, (uint32_t *)nullptr, (int)(m + 1));
    const size_t nb = align256(sizeof(uint32_t) * (size_t)n_all), mb = align256(sizeof(uint32_t) * (m + 1));
    const size_t pb = align256(sizeof(float4) * (size_t)n_all);
    if (w) {
        w->keys = (uint32_t *)base;
        w->ranks = (uint32_t *)(base + nb);
        w->keys_sorted = (uint32_t *)(base + 2 * nb);
        w->vals_sorted = (uint32_t *)(base + 3 * nb);
        w->count = (uint32_t *)(base + 4 * nb);
        w->cell_start = (uint32_t *)(base + 4 * nb + mb);
        w->pos_sorted = (float4 *)(base + 4 * nb + 2 * mb);
        w->cub_tmp = base + 4 * nb + 2 * mb + pb;
        w->cub_bytes = cub_bytes;
        w->mask = (uint32_t)(m - 1);
    }
    return 4 * nb + 2 * mb + pb + align256(cub_bytes);
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
            x += ssb::pos_lo(cols, r, 0);
            y += ssb::pos_lo(cols, r, 1);
            z += ssb::pos_lo(cols, r, 2);
        }
        p = make_float4(x, y, z, 0.0f);
    }
    out[r] = p;
}

// The gathered positions: one buffer, or (P2P exchange) slot (*slot_epoch & 1)
// of a double buffer, chosen on the device so graph replays follow the epoch.
__device__ __forceinline__ const float4 *gathered(const float4 *base, const uint32_t *slot_epoch, int64_t n_all)
{
    return slot_epoch ? base + (int64_t)(*slot_epoch & 1u) * n_all : base;
}

// Where the pipeline reads the swarm's positions: the gathered float4 buffer,
// or -- a single rank, no exchange -- the group's own columns directly (the
// pack kernel's arithmetic: hi + lo, NaN for dead rows), saving the pack pass.
struct PosSrc {
    const float4 *base;          // gathered buffer, or null: read the columns
    const uint32_t *slot_epoch;
    const float *cols;
    const uint8_t *flags;
    int compensated;
    __device__ __forceinline__ float4 get(int64_t i, int64_t n_all) const
    {
        if (base) return gathered(base, slot_epoch, n_all)[i];
        const float nan = __int_as_float(0x7fc00000);
        float4 p = make_float4(nan, nan, nan, 0.0f);
        if (flags[i] & SWARMSTEP_FLAG_ALIVE) {
            float x = cols[ssb::at(SWARMSTEP_COL_POS + 0, i)];
            float y = cols[ssb::at(SWARMSTEP_COL_POS + 1, i)];
            float z = cols[ssb::at(SWARMSTEP_COL_POS + 2, i)];
            if (compensated) {
                x += ssb::pos_lo(cols, i, 0);
                y += ssb::pos_lo(cols, i, 1);
                z += ssb::pos_lo(cols, i, 2);
            }
            p = make_float4(x, y, z, 0.0f);
        }
        return p;
    }
};

// bucket of every gathered agent (dead / padding rows: bucket m, past every
// real bucket) and its rank inside the bucket
__global__ void hash_count_kernel(const PosSrc src, int64_t n_all, float inv_cell, uint32_t mask, uint32_t *keys,
                                  uint32_t *ranks, uint32_t *count)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_all) return;
    const float4 p = src.get(i, n_all);
    const uint32_t k = isnan(p.x) ? mask + 1 : cell_hash(cell_of(p.x, inv_cell), cell_of(p.y, inv_cell),
                                                          cell_of(p.z, inv_cell), mask);
    keys[i] = k;
    ranks[i] = atomicAdd(&count[k], 1u);
}

// counting-sort scatter: the agent goes to start[bucket] + rank, its position
// (index in .w) with it
__global__ void scatter_kernel(const PosSrc src, int64_t n_all, uint32_t mask, const uint32_t *keys,
                               const uint32_t *ranks, const uint32_t *cell_start, uint32_t *keys_sorted,
                               uint32_t *vals_sorted, float4 *pos_sorted)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_all) return;
    const uint32_t k = keys[i];
    const uint32_t slot = cell_start[k] + ranks[i];
    keys_sorted[slot] = k;
    vals_sorted[slot] = (uint32_t)i;
    if (k <= mask) {
        float4 p = src.get(i, n_all);
        p.w = __uint_as_float((uint32_t)i);
        pos_sorted[slot] = p;
    }
}

// overlay sums in 64-bit fixed point, 2^32 units per m/s: order-independent
constexpr float kFix = 4294967296.0f;

__device__ __forceinline__ void sep_accumulate(const float4 &p, const float4 &q, bool take, float r2, float inv_r,
                                               float k_sep, long long &ax, long long &ay, long long &az)
{
    const float ddx = p.x - q.x, ddy = p.y - q.y, ddz = p.z - q.z;
    const float d2 = fmaf(ddx, ddx, fmaf(ddy, ddy, ddz * ddz));
    if (!take || !(d2 < r2) || !(d2 > 1e-24f)) return;   // strict <, d > 1e-12
    const float d = sqrtf(d2);
    const float s = k_sep * (1.0f - d * inv_r) / d;
    // |s dd| <= |k_sep| < 2^30 (checked by the caller): exact scaling, one rounding
    ax += __float2ll_rn(s * ddx * kFix);
    ay += __float2ll_rn(s * ddy * kFix);
    az += __float2ll_rn(s * ddz * kFix);
}

// One thread per agent in BUCKET order (neighbouring threads are neighbouring
// cells, so their candidate ranges overlap and hit L1).  An agent's 27
// neighbour cells are 9 x-rows, each one contiguous range of pos_sorted
// (split in two only where the row wraps the table end); each range is read
// four candidates at a time with independent loads.  Fixed-point sums: the
// result does not depend on the order the candidates are visited in.
__global__ void __launch_bounds__(128) query_kernel(const float4 *pos_sorted, const uint32_t *keys_sorted,
                                                    const uint32_t *vals_sorted, const uint32_t *cell_start,
                                                    uint32_t mask, float r_sense, float k_sep, int64_t n_all,
                                                    int64_t n_local, int64_t self_offset, const uint8_t *flags,
                                                    float *cols, int accumulate)
{
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n_all) return;
    const int64_t r = (int64_t)vals_sorted[j] - self_offset;
    if (r < 0 || r >= n_local) return;                       // another rank's agent
    const uint32_t h = keys_sorted[j];
    long long ax = 0, ay = 0, az = 0;
    if (h <= mask && (flags[r] & SWARMSTEP_FLAG_ALIVE)) {
        const float4 p = pos_sorted[j];
        const float r2 = r_sense * r_sense, inv_r = 1.0f / r_sense;
        const uint32_t end_all = cell_start[mask + 1];
#pragma unroll 1
        for (int row = 0; row < 9; row++) {
            const int dy = row % 3 - 1, dz = row / 3 - 1;
            const uint32_t hc = h + (uint32_t)dy * kHB + (uint32_t)dz * kHC;
            const uint32_t lo = (hc - 1u) & mask, hi = (hc + 1u) & mask;
            uint32_t s0 = cell_start[lo], e0, s1 = 0, e1 = 0;
            if (lo <= hi) {
                e0 = cell_start[hi + 1];
            } else {                                         // row wraps the table end
                e0 = end_all;
                e1 = cell_start[hi + 1];
            }
#pragma unroll 1
            for (int seg = 0; seg < 2; seg++) {
                const uint32_t s = seg ? s1 : s0, e = seg ? e1 : e0;
#pragma unroll 1
                for (uint32_t c = s; c < e; c += 4) {
                    float4 q[4];
#pragma unroll
                    for (int u = 0; u < 4; u++)
                        q[u] = c + u < e ? pos_sorted[c + u] : p;
#pragma unroll
                    for (int u = 0; u < 4; u++)
                        sep_accumulate(p, q[u], c + u < e && (int64_t)(c + u) != j, r2, inv_r, k_sep, ax, ay, az);
                }
            }
        }
    }
    float *ox = cols + ssb::at(SWARMSTEP_COL_OVERLAY + 0, r);
    float *oy = cols + ssb::at(SWARMSTEP_COL_OVERLAY + 1, r);
    float *oz = cols + ssb::at(SWARMSTEP_COL_OVERLAY + 2, r);
    const float fx = (float)((double)ax / kFix), fy = (float)((double)ay / kFix), fz = (float)((double)az / kFix);
    if (accumulate) {
        *ox += fx; *oy += fy; *oz += fz;
    } else {
        *ox = fx; *oy = fy; *oz = fz;
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
    // m = next_pow2(2 n_all) + 1 bucket counts are scanned with an int count
    if (n_all < 0 || n_all > (1LL << 29) || !bytes) return nb_err(SWARMSTEP_EINVAL, "bad n_all (0 .. 2^29)");
    *bytes = (uint64_t)layout(n_all, nullptr, nullptr);
    return SWARMSTEP_OK;
}

int swarmstep_neighbor_overlay(const swarmstep_group_view *g, const float *all_xyzw, int64_t n_all,
                               int64_t self_offset, float r_sense, float k_sep, float cell, int accumulate,
                               void *workspace, uint64_t ws_bytes, const uint32_t *slot_epoch, void *stream)
{
    if (!g || !g->cols || !g->flags || !workspace) return nb_err(SWARMSTEP_EINVAL, "null argument");
    if (!all_xyzw && (n_all != g->n || self_offset != 0 || slot_epoch))
        return nb_err(SWARMSTEP_EINVAL, "all_xyzw = NULL reads the group's own rows: needs n_all == n, offset 0");
    if (!(r_sense > 0.0f) || !(cell >= r_sense)) return nb_err(SWARMSTEP_EINVAL, "need r_sense > 0 and cell >= r_sense");
    if (self_offset < 0 || self_offset + g->n > n_all) return nb_err(SWARMSTEP_EINVAL, "local shard outside n_all");
    if (n_all > (1LL << 29)) return nb_err(SWARMSTEP_EINVAL, "n_all above 2^29");
    if (ws_bytes < (uint64_t)layout(n_all, nullptr, nullptr)) return nb_err(SWARMSTEP_EINVAL, "workspace too small");
    if (n_all == 0 || g->n == 0) return SWARMSTEP_OK;
    cudaStream_t s = (cudaStream_t)stream;
    Workspace w;
    layout(n_all, (char *)workspace, &w);
    const float inv_cell = 1.0f / cell;
    const PosSrc src{(const float4 *)all_xyzw, slot_epoch, g->cols, g->flags, g->compensated};
    if (!(fabsf(k_sep) < 1073741824.0f)) return nb_err(SWARMSTEP_EINVAL, "need |k_sep| < 2^30 (fixed-point sums)");
    cudaMemsetAsync(w.count, 0, sizeof(uint32_t) * ((size_t)w.mask + 2), s);
    hash_count_kernel<<<grid_n(n_all, 256), 256, 0, s>>>(src, n_all, inv_cell, w.mask, w.keys, w.ranks, w.count);
    size_t cb = w.cub_bytes;
    if (cub::DeviceScan::ExclusiveSum(w.cub_tmp, cb, w.count, w.cell_start, (int)(w.mask + 2), s) != cudaSuccess)
        return nb_cuda("cub::DeviceScan");
    scatter_kernel<<<grid_n(n_all, 256), 256, 0, s>>>(src, n_all, w.mask, w.keys, w.ranks, w.cell_start,
                                                      w.keys_sorted, w.vals_sorted, w.pos_sorted);
    query_kernel<<<grid_n(n_all, 128), 128, 0, s>>>(w.pos_sorted, w.keys_sorted, w.vals_sorted, w.cell_start,
                                                   w.mask, r_sense, k_sep, n_all, g->n, self_offset, g->flags,
                                                   g->cols, accumulate);
    return nb_cuda("neighbor overlay");
}

}  // extern "C"
