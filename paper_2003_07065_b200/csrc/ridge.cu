// Mode retrieval kernels (reading R22), sm_100a.
//
//  ridge_emission: E[m, l] = log(|T[m, l]| + eps), eps = 1e-12 max|T|  (fp64)
//  ridge_dp:       penalised dynamic programme over frames, one CTA, all in fp64:
//                  V_m[l] = E[m, l] + max_{l'} (V_{m-1}[l'] - lambda (l - l')^2)  (smallest l').
//                  Because the transition score has increasing differences in (l, l'), the
//                  smallest maximiser opt(l) is non-decreasing in l, so each frame is solved
//                  exactly by level-synchronous divide and conquer: level d fixes the points
//                  whose 1-based index has lowest set bit S/2^(d+1) (S = pow2 > B), searching
//                  only between the optima of their already-solved neighbours: O(B log B) per
//                  frame instead of O(B^2), same result.  Candidates are rounded as the oracle
//                  rounds them (no fused multiply-add).  Backpointers (int32) go to global
//                  memory; one thread traces the path back.  After each ridge the zone
//                  +-suppress bins is set to the floor emission log(eps).
//  zone_mask:      T outside (or inside) the zone |l - path[m]| <= half set to zero.
//  mode_full:      Eq. 15, H_t = 1: x_q[m] = (2 / (N_f g[c])) Re sum_{l in zone} w_l T[m, l].
#include <cuda_pipeline.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "sst_internal.h"

namespace sst {

// ------------------------------------------------------------------------------ emission ------
__global__ void absmax2_kernel(const float2* T, int64_t rows, int64_t cols, int64_t ldT, unsigned long long* out) {
    double m = 0.0;
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x)
        for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) {
            const float2 v = T[r * ldT + c];
            m = fmax(m, hypot((double)v.x, (double)v.y));
        }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    // non-negative doubles order as unsigned 64-bit integers: the max is exact and order-free
    if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

__global__ void emission_kernel(const float2* T, int64_t rows, int64_t cols, int64_t ldT,
                                const unsigned long long* amax, double* E, double* floor_out) {
    const double amax_d = __longlong_as_double((long long)*amax);
    const double eps = 1e-12 * amax_d;
    if (blockIdx.x == 0 && threadIdx.x == 0) *floor_out = log(eps);
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x)
        for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) {
            const float2 v = T[r * ldT + c];
            E[r * cols + c] = log(hypot((double)v.x, (double)v.y) + eps);
        }
}

cudaError_t launch_ridge_emission(const float2* T, int64_t rows, int64_t cols, int64_t ldT,
                                  unsigned long long* scratch, double* E, double* floor_out, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(scratch, 0, sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
    const int blocks = (int)(rows < 1184 ? rows : 1184);
    absmax2_kernel<<<blocks, 256, 0, s>>>(T, rows, cols, ldT, scratch);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    emission_kernel<<<blocks, 256, 0, s>>>(T, rows, cols, ldT, scratch, E, floor_out);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------ DP ------------
constexpr int kRidgeThreads = 1024;

// V[a] - lam (l - a)^2 rounded as the oracle rounds it (product, then difference): written with
// explicit _rn intrinsics so that the compiler cannot contract it into one fused multiply-add,
// whose single rounding could order near-tied candidates differently from the oracle's argmax
__device__ __forceinline__ double ridge_cand(const double* V, int l, int a, double lam) {
    const double dd = (double)(l - a);
    return __dsub_rn(V[a], __dmul_rn(lam, dd * dd));
}

// smallest maximiser of V[a] - lam (l - a)^2 over a in [a0, a1] by one thread
__device__ __forceinline__ void scan_thread(const double* V, int l, int a0, int a1, double lam, double& best, int& arg) {
    best = -INFINITY;
    arg = a0;
    for (int a = a0; a <= a1; ++a) {
        const double v = ridge_cand(V, l, a, lam);
        if (v > best) { best = v; arg = a; }
    }
}

// smallest maximiser of V[a] - lam (l - a)^2 over a in [a0, a1] by one warp (lanes split the
// range, then a warp argmax that keeps the smallest index on ties) -> opt[l]
__device__ __forceinline__ void warp_scan(const double* V, int l, int a0, int a1, double lam, int lane, int* opt) {
    double best = -INFINITY;
    int arg = a0;
    for (int a = a0 + lane; a <= a1; a += 32) {
        const double v = ridge_cand(V, l, a, lam);
        if (v > best) { best = v; arg = a; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
        if (ob > best || (ob == best && oa < arg)) { best = ob; arg = oa; }
    }
    if (lane == 0) opt[l] = arg;
}

constexpr int kRidgeLong = 64;     // a thread-per-point level's ranges of at least this length go to the warp

__global__ void __launch_bounds__(kRidgeThreads, 1)
ridge_dp_kernel(double* E, int64_t rows, int cols, double lam, int count, int suppress, const double* floor_in,
                int32_t* back, int32_t* paths) {
    extern __shared__ __align__(16) unsigned char sm[];
    double* V = reinterpret_cast<double*>(sm);            // [cols] previous frame (ping-pong with Vn)
    double* Vn = V + cols;                                 // [cols] current frame
    double* En = Vn + cols;                                // [cols] emission row of the frame, prefetched
    int* opt = reinterpret_cast<int*>(En + cols);          // [cols]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = kRidgeThreads / 32;
    int S = 1;
    while (S <= cols) S <<= 1;                             // S > cols: every p in [1, cols] has a level
    int levels = 0;
    while ((1 << levels) < S) ++levels;
    const double floor_e = *floor_in;

    for (int q = 0; q < count; ++q) {
        for (int l = tid; l < cols; l += kRidgeThreads) V[l] = E[l];
        if (rows > 1)
            for (int l = tid; l < cols; l += kRidgeThreads) __pipeline_memcpy_async(En + l, E + cols + l, sizeof(double));
        __pipeline_commit();
        __syncthreads();
        for (int64_t m = 1; m < rows; ++m) {
            int32_t* bk = back + m * cols;
            for (int d = 0; d < levels; ++d) {
                const int step = S >> (d + 1);                 // points p = step (2i + 1), p <= cols
                const int npts = (cols >= step) ? (((cols - step) >> (levels - d)) + 1) : 0;   // 2 step = 2^(levels-d)
                if (npts <= NW) {
                    // one warp per point: lanes split the candidate range, then a warp argmax
                    for (int i = warp; i < npts; i += NW) {
                        const int p = step * (2 * i + 1), l = p - 1;
                        const int a0 = (p - step >= 1) ? opt[p - step - 1] : 0;
                        const int a1 = (p + step <= cols) ? opt[p + step - 1] : cols - 1;
                        warp_scan(V, l, a0, a1, lam, lane, opt);
                    }
                } else {
                    // one thread per point; the points of a warp whose candidate range is long (the
                    // optimum jumps across it: two peaks of V, or lambda = 0 where the edge points
                    // span [0, argmax] and [argmax, B)) are then scanned by the whole warp, one after
                    // another, so no lane scans more than kRidgeLong candidates serially and no
                    // extra CTA barrier is needed
                    for (int i0 = tid - lane; i0 < npts; i0 += kRidgeThreads) {
                        const int i = i0 + lane;
                        const bool in = i < npts;
                        const int p = step * (2 * i + 1), l = p - 1;
                        int a0 = 0, a1 = -1;
                        if (in) {
                            a0 = (p - step >= 1) ? opt[p - step - 1] : 0;
                            a1 = (p + step <= cols) ? opt[p + step - 1] : cols - 1;
                        }
                        const bool lng = a1 - a0 >= kRidgeLong;
                        if (in && !lng) {
                            double best;
                            int arg;
                            scan_thread(V, l, a0, a1, lam, best, arg);
                            opt[l] = arg;
                        }
                        unsigned m = __ballot_sync(0xffffffffu, lng);
                        while (m) {
                            const int src = __ffs(m) - 1;
                            m &= m - 1;
                            warp_scan(V, __shfl_sync(0xffffffffu, l, src), __shfl_sync(0xffffffffu, a0, src),
                                      __shfl_sync(0xffffffffu, a1, src), lam, lane, opt);
                        }
                    }
                }
                __syncthreads();
            }
            __pipeline_wait_prior(0);                         // this frame's emissions (own copies)
            for (int l = tid; l < cols; l += kRidgeThreads) {
                const int a = opt[l];
                Vn[l] = __dadd_rn(En[l], ridge_cand(V, l, a, lam));
                bk[l] = a;
            }
            __syncthreads();
            { double* t = V; V = Vn; Vn = t; }                // ping-pong: the new row becomes V
            // prefetch the next frame's emission row (each thread copies the entries it reads)
            if (m + 1 < rows)
                for (int l = tid; l < cols; l += kRidgeThreads)
                    __pipeline_memcpy_async(En + l, E + (m + 1) * cols + l, sizeof(double));
            __pipeline_commit();
            __syncthreads();
        }
        // final argmax (smallest index), traceback, suppression
        if (warp == 0) {
            double best = -INFINITY;
            int arg = 0;
            for (int l = lane; l < cols; l += 32)
                if (V[l] > best) { best = V[l]; arg = l; }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
                if (ob > best || (ob == best && oa < arg)) { best = ob; arg = oa; }
            }
            if (lane == 0) {
                int32_t* path = paths + (int64_t)q * rows;
                int cur = arg;
                path[rows - 1] = cur;
                for (int64_t m = rows - 1; m > 0; --m) {
                    cur = back[m * cols + cur];
                    path[m - 1] = cur;
                }
            }
        }
        __syncthreads();
        if (q + 1 < count) {
            const int32_t* path = paths + (int64_t)q * rows;
            for (int64_t m = tid; m < rows; m += kRidgeThreads) {
                const int c = path[m];
                const int lo = max(0, c - suppress), hi = min(cols - 1, c + suppress);
                for (int l = lo; l <= hi; ++l) E[m * cols + l] = floor_e;
            }
            __threadfence_block();
            __syncthreads();
        }
    }
}

cudaError_t launch_ridge_dp(double* E, int64_t rows, int cols, double lam, int count, int suppress,
                            const double* floor_in, int32_t* back, int32_t* paths, cudaStream_t s) {
    const size_t smem = (size_t)cols * (3 * sizeof(double) + sizeof(int));
    cudaError_t e = cudaFuncSetAttribute(ridge_dp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    ridge_dp_kernel<<<1, kRidgeThreads, smem, s>>>(E, rows, cols, lam, count, suppress, floor_in, back, paths);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------ zone / Eq. 15 --
__global__ void zone_mask_kernel(float2* T, int64_t rows, int cols, int64_t ldT, const int32_t* path, int half,
                                 int keep_inside) {
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
        const int c = path[r];
        for (int l = threadIdx.x; l < cols; l += blockDim.x) {
            const bool in = abs(l - c) <= half;
            if (in != (bool)keep_inside) T[r * ldT + l] = make_float2(0.0f, 0.0f);
        }
    }
}

cudaError_t launch_zone_mask(float2* T, int64_t rows, int cols, int64_t ldT, const int32_t* path, int half,
                             int keep_inside, cudaStream_t s) {
    const int blocks = (int)(rows < 4736 ? rows : 4736);
    zone_mask_kernel<<<blocks, 256, 0, s>>>(T, rows, cols, ldT, path, half, keep_inside);
    return cudaGetLastError();
}

// one warp per frame, fixed-order fp64 reduction over the zone
__global__ void mode_full_kernel(const float2* T, int64_t rows, int cols, int64_t ldT, const int32_t* path, int half,
                                 int dc_bin, double scale, float* x) {
    const int lane = threadIdx.x & 31;
    const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t r = w; r < rows; r += nw) {
        const int c = path[r];
        const int lo = max(0, c - half), hi = min(cols - 1, c + half);
        double acc = 0.0;
        for (int l = lo + lane; l <= hi; l += 32) {
            const double v = (double)T[r * ldT + l].x;
            acc += (l == dc_bin) ? 0.5 * v : v;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) x[r] = (float)(scale * acc);
    }
}

cudaError_t launch_mode_full(const float2* T, int64_t rows, int cols, int64_t ldT, const int32_t* path, int half,
                             int dc_bin, double scale, float* x, cudaStream_t s) {
    const int64_t want = (rows + 7) / 8;
    const int blocks = (int)(want < 4736 ? want : 4736);
    mode_full_kernel<<<blocks, 256, 0, s>>>(T, rows, cols, ldT, path, half, dc_bin, scale, x);
    return cudaGetLastError();
}

}  // namespace sst
