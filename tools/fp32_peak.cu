// FP32 SIMT throughput microbenchmark (cross-check of the derived ALU peak in DESIGN.md §7):
// scalar FFMA and packed FFMA2 (sm_100a FP32x2), 8 independent chains per thread, 4 warps x 8
// CTAs per SM.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp32_peak tools/fp32_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__global__ void ffma_kernel(float* out, float a, float b) {
    float x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, b);
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 1234.5f) out[threadIdx.x] = s;
}

__global__ void ffma2_kernel(float* out, float a, float b) {
    float2 x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
    const float2 a2 = make_float2(a, a), b2 = make_float2(b, b);
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __ffma2_rn(x[i], a2, b2);
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i].x + x[i].y;
    if (s == 1234.5f) out[threadIdx.x] = s;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    cudaMalloc(&out, 4096);
    const int blocks = sms * 8, threads = 128;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int v = 0; v < 2; ++v) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (v == 0) ffma_kernel<<<blocks, threads>>>(out, 0.999f, 0.001f);
            else ffma2_kernel<<<blocks, threads>>>(out, 0.999f, 0.001f);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e0, e1);
            const double flops = 2.0 * 8 * ITERS * (double)blocks * threads * (v == 0 ? 1 : 2);
            if (rep == 1) printf("%s: %.1f TFLOP/s (%d SMs)\n", v == 0 ? "FFMA " : "FFMA2", flops / (ms * 1e-3) / 1e12, sms);
        }
    }
    return 0;
}
