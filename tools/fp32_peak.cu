// fp32_peak.cu -- FP32 SIMT peak microbenchmark (tuning/measurement aid, not product).
//
// MEASURED_PEAKS.json carries HBM and tensor-core peaks only; the fused step at
// K >= 4 is bound by the FP32 SIMT pipes, so bench.py measures their peak here:
// 8 independent FFMA chains per thread, 256 threads x (#SM x 8) CTAs, both the
// register-operand and the immediate-operand FFMA forms, and packed FFMA2 (imm == 2);
// imm == 3 is packed FFMA2 with three vector-register operands (context, not a peak).
//   build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Xcompiler -fPIC -shared
//          -o tools/libfp32peak.so tools/fp32_peak.cu
#include <cuda_runtime.h>
#include <stdint.h>

template <bool IMM>
__global__ void __launch_bounds__(256) ffma_kernel(float *out, float a, float b, int iters)
{
    float x[8];
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int r = 0; r < 16; r++) {
#pragma unroll
            for (int i = 0; i < 8; i++) {
                if (IMM)
                    x[i] = fmaf(x[i], 0.9999f, 0.0001f);
                else
                    x[i] = fmaf(x[i], a, b);
            }
        }
    }
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < 8; i++) s += x[i];
    if (s == 12345.678f) out[0] = s;  // keep the chains alive
}

// packed f32x2 FMA (FFMA2, sm_100): 8 independent float2 chains per thread
__global__ void __launch_bounds__(256) ffma2_kernel(float *out, float a, float b, int iters)
{
    float2 x[8];
    const float2 av = make_float2(a, a), bv = make_float2(b, b);
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int r = 0; r < 16; r++) {
#pragma unroll
            for (int i = 0; i < 8; i++) x[i] = __ffma2_rn(x[i], av, bv);
        }
    }
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < 8; i++) s += x[i].x + x[i].y;
    if (s == 12345.678f) out[0] = s;
}

// packed FFMA2 with three distinct vector-register operand pairs: issues at
// ~2/3 of the rate above (register-file read bandwidth) -- the form of an
// FMA whose three operands are all per-agent values
__global__ void __launch_bounds__(256) ffma2_3reg_kernel(float *out, float a, float b, int iters)
{
    float2 x[8], y[8], z[8];
#pragma unroll
    for (int i = 0; i < 8; i++) {
        x[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
        y[i] = make_float2(a - threadIdx.x * 1e-9f * i, a * 0.99999f);
        z[i] = make_float2(b * (i + 1) + threadIdx.x * 1e-9f, b * 0.5f * (i + 1));
    }
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int r = 0; r < 16; r++) {
#pragma unroll
            for (int i = 0; i < 8; i++) x[i] = __ffma2_rn(x[i], y[i], z[i]);
        }
    }
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < 8; i++) s += x[i].x + x[i].y + y[i].y + z[i].y;
    if (s == 12345.678f) out[0] = s;
}

extern "C" int fp32_peak_tflops(int imm, double *tflops, double *ms)
{
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    float *out = nullptr;
    cudaMalloc(&out, sizeof(float));
    const int iters = 2048, blocks = sms * 8, threads = 256;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; rep++) {  // rep 0 warms up
        cudaEventRecord(e0);
        if (imm == 3)
            ffma2_3reg_kernel<<<blocks, threads>>>(out, 0.9999f, 0.0001f, iters);
        else if (imm == 2)
            ffma2_kernel<<<blocks, threads>>>(out, 0.9999f, 0.0001f, iters);
        else if (imm)
            ffma_kernel<true><<<blocks, threads>>>(out, 0.9999f, 0.0001f, iters);
        else
            ffma_kernel<false><<<blocks, threads>>>(out, 0.9999f, 0.0001f, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
    }
    float t = 0.0f;
    cudaEventElapsedTime(&t, e0, e1);
    const double ffma = (double)blocks * threads * iters * 16 * 8 * (imm >= 2 ? 2 : 1);
    *ms = t;
    *tflops = 2.0 * ffma / (t * 1e-3) / 1e12;
    cudaFree(out);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}
