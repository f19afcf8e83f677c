// collision.cu -- GPU sphere-collision and neighbour detection.
//
// Restates collision.py:110-176 (detect) on the device with the same
// arithmetic, so results are identical to the reference on the same float64
// positions:
//   * broad phase: grid cells floor(p / cell) (collision.py:59-63), agents
//     sorted by an exact 63-bit cell key (CUB radix sort, stable), candidate
//     pairs = same-cell pairs with i < j plus the reference's half-space cell
//     offsets (collision.py:86-95, computed on the host and passed in), each
//     neighbour cell found by binary search -- every unordered pair once;
//   * narrow phase in float64: d2 = (dx^2 + dy^2) + dz^2; collide iff
//     d2 < (r_a + r_b)^2, neighbours iff d2 < r_sense^2 (strict, collision.py:
//     157-166).
// Pairs are appended through atomic counters (count pass, then fill pass);
// the host sorts them exactly as the reference does.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"

namespace {

constexpr int64_t kBias = 1LL << 20;   // cell coordinates must lie in (-2^20, 2^20)

__device__ __forceinline__ uint64_t pack_key(int64_t cx, int64_t cy, int64_t cz)
{
    return ((uint64_t)(cx + kBias) << 42) | ((uint64_t)(cy + kBias) << 21) | (uint64_t)(cz + kBias);
}

__global__ void pack_collision_kernel(const float *cols, const uint8_t *flags, int64_t n, int compensated,
                                      double radius, double *xyzr, int64_t offset)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    double *o = xyzr + 4 * (offset + r);
    for (int i = 0; i < 3; i++) {
        double p = (double)cols[ssb::at(SWARMSTEP_COL_POS + i, r)];
        if (compensated) p += (double)cols[ssb::at(SWARMSTEP_COL_POS_LO + i, r)];
        o[i] = p;
    }
    o[3] = (flags[r] & SWARMSTEP_FLAG_ALIVE) ? radius : __longlong_as_double(0x7ff8000000000000LL);  // NaN = dead
}

__global__ void cell_key_kernel(const double *xyzr, int64_t m, double cell, uint64_t *keys, uint32_t *vals,
                                uint32_t *range_err)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const double *p = xyzr + 4 * i;
    uint64_t key = ~0ull;   // dead rows sort last
    if (!isnan(p[3])) {
        const double cx = floor(p[0] / cell), cy = floor(p[1] / cell), cz = floor(p[2] / cell);
        const double lim = (double)(kBias - 8);
        if (fabs(cx) >= lim || fabs(cy) >= lim || fabs(cz) >= lim)
            atomicOr(range_err, 1u);
        else
            key = pack_key((int64_t)cx, (int64_t)cy, (int64_t)cz);
    }
    keys[i] = key;
    vals[i] = (uint32_t)i;
}

__device__ __forceinline__ int64_t lower_bound(const uint64_t *a, int64_t n, uint64_t k)
{
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (a[mid] < k) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// One thread per gathered agent i (alive): same-cell partners j > i and the
// half-space neighbour cells.  fill == 0: count only.
__global__ void pair_kernel(const double *xyzr, const uint64_t *keys_sorted, const uint32_t *vals_sorted,
                            int64_t m, double cell, const int *offsets, int n_off, double r_sense,
                            unsigned long long *counters, uint32_t *coll, uint32_t *near,
                            unsigned long long coll_cap, unsigned long long near_cap, int fill)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const double *pi = xyzr + 4 * i;
    if (isnan(pi[3])) return;
    const int64_t cx = (int64_t)floor(pi[0] / cell), cy = (int64_t)floor(pi[1] / cell), cz = (int64_t)floor(pi[2] / cell);
    const double rs2 = r_sense * r_sense;
    for (int o = -1; o < n_off; o++) {
        const int ox = o < 0 ? 0 : offsets[3 * o], oy = o < 0 ? 0 : offsets[3 * o + 1], oz = o < 0 ? 0 : offsets[3 * o + 2];
        const uint64_t k = pack_key(cx + ox, cy + oy, cz + oz);
        int64_t j0 = lower_bound(keys_sorted, m, k);
        for (int64_t s = j0; s < m && keys_sorted[s] == k; s++) {
            const int64_t j = vals_sorted[s];
            if (o < 0 && j <= i) continue;              // same cell: each pair once (collision.py:139-143)
            const double *pj = xyzr + 4 * j;
            const double dx = pi[0] - pj[0], dy = pi[1] - pj[1], dz = pi[2] - pj[2];
            const double d2 = (dx * dx + dy * dy) + dz * dz;
            const double rsum = pi[3] + pj[3];
            if (d2 < rsum * rsum) {
                const unsigned long long slot = atomicAdd(&counters[0], 1ull);
                if (fill && slot < coll_cap) { coll[2 * slot] = (uint32_t)i; coll[2 * slot + 1] = (uint32_t)j; }
            }
            if (d2 < rs2) {
                const unsigned long long slot = atomicAdd(&counters[1], 1ull);
                if (fill && slot < near_cap) { near[2 * slot] = (uint32_t)i; near[2 * slot + 1] = (uint32_t)j; }
            }
        }
    }
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

size_t sort_tmp_bytes(int64_t m)
{
    size_t b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, b, (uint64_t *)nullptr, (uint64_t *)nullptr, (uint32_t *)nullptr,
                                    (uint32_t *)nullptr, (int)m);
    return b;
}

}  // namespace

extern "C" {

int swarmstep_pack_collision(const swarmstep_group_view *g, double radius, double *xyzr, int64_t offset, void *stream)
{
    if (!g || !g->cols || !g->flags || !xyzr) return ssb::set_err(SWARMSTEP_EINVAL, "null argument");
    if (g->n == 0) return SWARMSTEP_OK;
    pack_collision_kernel<<<(unsigned)((g->n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        g->cols, g->flags, g->n, g->compensated, radius, xyzr, offset);
    return ssb::cuda_status("pack_collision_kernel");
}

int swarmstep_collision_workspace_bytes(int64_t m, uint64_t *bytes)
{
    if (m < 0 || m > 0x7fffffffLL || !bytes) return ssb::set_err(SWARMSTEP_EINVAL, "bad m");
    *bytes = 2 * align256(8 * (size_t)m) + 2 * align256(4 * (size_t)m) + align256(sort_tmp_bytes(m)) + 256;
    return SWARMSTEP_OK;
}

int swarmstep_collision_pairs(const double *xyzr, int64_t m, double cell, const int *offsets_dev, int n_off,
                              double r_sense, uint32_t *coll, uint64_t coll_cap, uint32_t *near,
                              uint64_t near_cap, uint64_t *counts_dev, void *workspace, uint64_t ws_bytes,
                              int fill, void *stream)
{
    if (!xyzr || !counts_dev || !workspace || (n_off > 0 && !offsets_dev)) return ssb::set_err(SWARMSTEP_EINVAL, "null argument");
    if (!(cell > 0.0) || !(r_sense > 0.0)) return ssb::set_err(SWARMSTEP_EINVAL, "cell and r_sense must be positive");
    uint64_t need = 0;
    swarmstep_collision_workspace_bytes(m, &need);
    if (ws_bytes < need) return ssb::set_err(SWARMSTEP_EINVAL, "workspace too small");
    cudaStream_t s = (cudaStream_t)stream;
    cudaMemsetAsync(counts_dev, 0, 3 * sizeof(uint64_t), s);
    if (m == 0) return ssb::cuda_status("collision (empty)");
    char *base = (char *)workspace;
    uint64_t *keys = (uint64_t *)base;
    uint64_t *keys_sorted = (uint64_t *)(base + align256(8 * (size_t)m));
    uint32_t *vals = (uint32_t *)(base + 2 * align256(8 * (size_t)m));
    uint32_t *vals_sorted = (uint32_t *)(base + 2 * align256(8 * (size_t)m) + align256(4 * (size_t)m));
    void *tmp = base + 2 * align256(8 * (size_t)m) + 2 * align256(4 * (size_t)m);
    size_t tb = sort_tmp_bytes(m);
    const unsigned grid = (unsigned)((m + 255) / 256);
    cell_key_kernel<<<grid, 256, 0, s>>>(xyzr, m, cell, keys, vals, (uint32_t *)(counts_dev + 2));
    if (cub::DeviceRadixSort::SortPairs(tmp, tb, keys, keys_sorted, vals, vals_sorted, (int)m, 0, 64, s) != cudaSuccess)
        return ssb::cuda_status("cub::DeviceRadixSort");
    pair_kernel<<<grid, 256, 0, s>>>(xyzr, keys_sorted, vals_sorted, m, cell, offsets_dev, n_off, r_sense,
                                     (unsigned long long *)counts_dev, coll, near, (unsigned long long)coll_cap,
                                     (unsigned long long)near_cap, fill);
    return ssb::cuda_status("pair_kernel");
}

}  // extern "C"
