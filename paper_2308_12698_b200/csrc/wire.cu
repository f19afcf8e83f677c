// wire.cu -- device-side snapshot packing.
//
// Builds one group's section body of the binary SnapshotMsg (wire.py:162-178,
// PROTOCOL.md "Snapshot (0x01)") directly from the device columns:
//   u64*n agent_ids | u8*n alive | f32*3n pos | f32*3n vel | f32*4n quat | f32*3n omega
// little-endian, each column contiguous, quaternions canonicalised to w >= 0
// (quat.py:52-59, including the "+ 0.0" that turns -0 into +0).  Positions are
// rounded to float32 from the exact double hi + lo, i.e. exactly what
// encode_snapshot produces from the group's float64 host mirror.  The host
// then needs one device->host copy of 61 bytes per agent instead of packing
// 13 float64 columns in Python.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace {

__device__ __forceinline__ void put_f32(uint8_t *dst, bool aligned, float v)
{
    if (aligned) {
        *reinterpret_cast<float *>(dst) = v;
    } else {
        const uint32_t u = __float_as_uint(v);
        dst[0] = (uint8_t)u;
        dst[1] = (uint8_t)(u >> 8);
        dst[2] = (uint8_t)(u >> 16);
        dst[3] = (uint8_t)(u >> 24);
    }
}

__global__ void pack_wire_kernel(const float *cols, const uint8_t *flags, const uint64_t *ids, int64_t n,
                                 int compensated, uint8_t *out)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    reinterpret_cast<uint64_t *>(out)[r] = ids[r];      // 8-byte aligned: out is
    out[8 * n + r] = (flags[r] & SWARMSTEP_FLAG_ALIVE) ? 1 : 0;
    uint8_t *f = out + 9 * n;                           // float columns start here
    const bool aligned = ((9 * n) & 3) == 0;
    for (int i = 0; i < 3; i++) {
        double p = (double)cols[ssb::at(SWARMSTEP_COL_POS + i, r)];
        if (compensated) p += (double)ssb::pos_lo(cols, r, i);
        put_f32(f + 4 * (3 * r + i), aligned, (float)p);
        put_f32(f + 4 * (3 * n + 3 * r + i), aligned, cols[ssb::at(SWARMSTEP_COL_VEL + i, r)]);
        put_f32(f + 4 * (10 * n + 3 * r + i), aligned, cols[ssb::at(SWARMSTEP_COL_OMEGA + i, r)]);
    }
    const float sgn = cols[ssb::at(SWARMSTEP_COL_QUAT, r)] < 0.0f ? -1.0f : 1.0f;
    for (int i = 0; i < 4; i++)
        put_f32(f + 4 * (6 * n + 4 * r + i), aligned, cols[ssb::at(SWARMSTEP_COL_QUAT + i, r)] * sgn + 0.0f);
}

}  // namespace

extern "C" int swarmstep_quad_pack_wire(const swarmstep_group_view *g, const uint64_t *agent_ids, uint8_t *out,
                                        void *stream)
{
    if (!g || !g->cols || !g->flags || !agent_ids || !out) return ssb::set_err(SWARMSTEP_EINVAL, "null argument");
    if ((reinterpret_cast<uintptr_t>(out) & 7u) != 0) return ssb::set_err(SWARMSTEP_EINVAL, "out must be 8-byte aligned");
    if (g->n == 0) return SWARMSTEP_OK;
    pack_wire_kernel<<<(unsigned)((g->n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        g->cols, g->flags, agent_ids, g->n, g->compensated, out);
    return ssb::cuda_status("pack_wire_kernel");
}
