// Shared-memory atomics vs plain RMW throughput on this GPU (decides the squeeze / OLA design).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_atom(float* out, int iters, int stride) {
    __shared__ float s[8192];
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) s[i] = 0;
    __syncthreads();
    float v = threadIdx.x * 1e-3f;
    int base = (threadIdx.x * stride) & 8191;
    for (int it = 0; it < iters; ++it) {
        atomicAdd(&s[(base + it * 37) & 8191], v);
    }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = s[5];
}
__global__ void k_rmw(float* out, int iters, int stride) {
    __shared__ float s[8192];
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) s[i] = 0;
    __syncthreads();
    float v = threadIdx.x * 1e-3f;
    int base = (threadIdx.x * stride) & 8191;
    for (int it = 0; it < iters; ++it) {
        float* p = &s[(base + it * 37) & 8191];
        *p = *p + v;
    }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = s[5];
}
int main() {
    float* out; cudaMalloc(&out, 148 * 64 * sizeof(float));
    int iters = 4096;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int stride : {1, 0, 33}) {
        for (int kind = 0; kind < 2; ++kind) {
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(a);
                if (kind == 0) k_atom<<<148 * 4, 256>>>(out, iters, stride);
                else k_rmw<<<148 * 4, 256>>>(out, iters, stride);
                cudaEventRecord(b); cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b);
                double lane_ops = 148.0 * 4 * 256 * iters;
                if (rep) printf("%s stride=%d: %.3f ms, %.2f lane-ops/clk/SM (at 1.965 GHz)\n", kind ? "rmw " : "atom", stride, ms,
                       lane_ops / (ms * 1e-3) / 148 / 1.965e9);
            }
        }
    }
    return 0;
}
