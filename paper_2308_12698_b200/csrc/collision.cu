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
// Pairs are counted per sorted position (count pass), exclusive-scanned, and
// written at their offsets (fill pass): no atomics, deterministic order; the
// host sorts them exactly as the reference does.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

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
        if (compensated) p += (double)ssb::pos_lo(cols, r, i);
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

// One thread per SORTED position t (agent i = vals_sorted[t]; neighbouring
// threads sit in the same / adjacent cells, so their searches and candidate
// reads share cache lines): same-cell partners j > i plus the half-space
// neighbour cells.  FILL == false: per-thread pair counts; FILL == true: the
// pairs, written at this thread's exclusive-scan offsets -- no atomics, and
// the output order is deterministic.
template <bool FILL>
__global__ void __launch_bounds__(256) pair_kernel(const double *xyzr, const uint64_t *keys_sorted,
                                                   const uint32_t *vals_sorted, int64_t m, double cell,
                                                   const int *offsets, int n_off, double r_sense,
                                                   uint64_t *cnt_coll, uint64_t *cnt_near, uint32_t *coll,
                                                   uint32_t *near, uint64_t coll_cap, uint64_t near_cap)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m) return;
    uint64_t nc = 0, nn = 0, oc = 0, on = 0;
    if (FILL) {
        oc = cnt_coll[t];
        on = cnt_near[t];
    }
    const uint64_t kself = keys_sorted[t];
    if (kself != ~0ull) {
        const int64_t i = vals_sorted[t];
        const double *pi = xyzr + 4 * i;
        const double px = pi[0], py = pi[1], pz = pi[2], ri = pi[3];
        const int64_t cx = (int64_t)floor(px / cell), cy = (int64_t)floor(py / cell), cz = (int64_t)floor(pz / cell);
        const double rs2 = r_sense * r_sense;
        for (int o = -1; o < n_off; o++) {
            const int ox = o < 0 ? 0 : offsets[3 * o], oy = o < 0 ? 0 : offsets[3 * o + 1], oz = o < 0 ? 0 : offsets[3 * o + 2];
            const uint64_t k = pack_key(cx + ox, cy + oy, cz + oz);
            for (int64_t s = lower_bound(keys_sorted, m, k); s < m && keys_sorted[s] == k; s++) {
                const int64_t j = vals_sorted[s];
                if (o < 0 && j <= i) continue;              // same cell: each pair once (collision.py:139-143)
                const double *pj = xyzr + 4 * j;
                const double dx = px - pj[0], dy = py - pj[1], dz = pz - pj[2];
                const double d2 = (dx * dx + dy * dy) + dz * dz;
                const double rsum = ri + pj[3];
                if (d2 < rsum * rsum) {
                    if (FILL && oc + nc < coll_cap) { coll[2 * (oc + nc)] = (uint32_t)i; coll[2 * (oc + nc) + 1] = (uint32_t)j; }
                    nc++;
                }
                if (d2 < rs2) {
                    if (FILL && on + nn < near_cap) { near[2 * (on + nn)] = (uint32_t)i; near[2 * (on + nn) + 1] = (uint32_t)j; }
                    nn++;
                }
            }
        }
    }
    if (!FILL) {
        cnt_coll[t] = nc;
        cnt_near[t] = nn;
    }
}

// totals after the exclusive scans: counts[k] = offset[m-1] + count[m-1]
__global__ void totals_kernel(const uint64_t *cnt_coll, const uint64_t *cnt_near, const uint64_t *off_coll,
                              const uint64_t *off_near, int64_t m, uint64_t *counts)
{
    counts[0] = off_coll[m - 1] + cnt_coll[m - 1];
    counts[1] = off_near[m - 1] + cnt_near[m - 1];
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

size_t sort_tmp_bytes(int64_t m)
{
    size_t b = 0, c = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, b, (uint64_t *)nullptr, (uint64_t *)nullptr, (uint32_t *)nullptr,
                                    (uint32_t *)nullptr, (int)m);
    cub::DeviceScan::ExclusiveSum(nullptr, c, (uint64_t *)nullptr, (uint64_t *)nullptr, (int)m);
    return b > c ? b : c;
}

// workspace layout (one buffer): keys, keys_sorted (u64), vals, vals_sorted
// (u32), per-position pair counts and their exclusive-scan offsets (u64 x 4),
// CUB temporary storage
struct Ws {
    uint64_t *keys, *keys_sorted;
    uint32_t *vals, *vals_sorted;
    uint64_t *cnt_coll, *cnt_near, *off_coll, *off_near;
    void *tmp;
    size_t tmp_bytes;
};

size_t ws_layout(int64_t m, char *base, Ws *w)
{
    const size_t b8 = align256(8 * (size_t)m), b4 = align256(4 * (size_t)m), bt = align256(sort_tmp_bytes(m));
    if (w) {
        w->keys = (uint64_t *)base;
        w->keys_sorted = (uint64_t *)(base + b8);
        w->vals = (uint32_t *)(base + 2 * b8);
        w->vals_sorted = (uint32_t *)(base + 2 * b8 + b4);
        w->cnt_coll = (uint64_t *)(base + 2 * b8 + 2 * b4);
        w->cnt_near = (uint64_t *)(base + 3 * b8 + 2 * b4);
        w->off_coll = (uint64_t *)(base + 4 * b8 + 2 * b4);
        w->off_near = (uint64_t *)(base + 5 * b8 + 2 * b4);
        w->tmp = base + 6 * b8 + 2 * b4;
        w->tmp_bytes = bt;
    }
    return 6 * b8 + 2 * b4 + bt + 256;
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
    *bytes = ws_layout(m, nullptr, nullptr);
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
    if (m == 0) {
        cudaMemsetAsync(counts_dev, 0, 3 * sizeof(uint64_t), s);
        return ssb::cuda_status("collision (empty)");
    }
    Ws w;
    ws_layout(m, (char *)workspace, &w);
    const unsigned grid = (unsigned)((m + 255) / 256);
    if (fill) {
        // the count pass of the same inputs left keys, order and offsets in the workspace
        pair_kernel<true><<<grid, 256, 0, s>>>(xyzr, w.keys_sorted, w.vals_sorted, m, cell, offsets_dev, n_off,
                                               r_sense, w.off_coll, w.off_near, coll, near, coll_cap, near_cap);
        return ssb::cuda_status("pair_kernel<fill>");
    }
    cudaMemsetAsync(counts_dev, 0, 3 * sizeof(uint64_t), s);
    cell_key_kernel<<<grid, 256, 0, s>>>(xyzr, m, cell, w.keys, w.vals, (uint32_t *)(counts_dev + 2));
    size_t tb = w.tmp_bytes;
    if (cub::DeviceRadixSort::SortPairs(w.tmp, tb, w.keys, w.keys_sorted, w.vals, w.vals_sorted, (int)m, 0, 64, s) !=
        cudaSuccess)
        return ssb::cuda_status("cub::DeviceRadixSort");
    pair_kernel<false><<<grid, 256, 0, s>>>(xyzr, w.keys_sorted, w.vals_sorted, m, cell, offsets_dev, n_off, r_sense,
                                            w.cnt_coll, w.cnt_near, nullptr, nullptr, 0, 0);
    tb = w.tmp_bytes;
    if (cub::DeviceScan::ExclusiveSum(w.tmp, tb, w.cnt_coll, w.off_coll, (int)m, s) != cudaSuccess ||
        (tb = w.tmp_bytes, cub::DeviceScan::ExclusiveSum(w.tmp, tb, w.cnt_near, w.off_near, (int)m, s)) != cudaSuccess)
        return ssb::cuda_status("cub::DeviceScan");
    totals_kernel<<<1, 1, 0, s>>>(w.cnt_coll, w.cnt_near, w.off_coll, w.off_near, m, counts_dev);
    return ssb::cuda_status("pair_kernel<count>");
}

}  // extern "C"
