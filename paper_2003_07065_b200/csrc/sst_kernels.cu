// sm_100a kernels of the fast downsampled SST (He & Cao, arXiv 2003.07065).
//
// This file: the dispatch over the per-N2 kernel modules (kern_inst.cu, compiled once per N2 and
// direction), the seam / finalize kernels of the inverse and the Renyi reduction.  The kernels
// themselves are in fwd_kernel.cuh (forward) and inv_kernel.cuh (inverse).
//
// Forward (one fused persistent kernel, rows a1-a7 of DESIGN.md §1):
//   Each CTA walks a contiguous chunk of frames in tiles of G frames.  The tile's input span
//   ((G-1) H + L samples) is copied HBM -> shared memory with one cp.async.bulk (TMA bulk copy)
//   completed on an mbarrier, double-buffered so tile t+1 streams in while tile t computes; the
//   window taps (g, alpha g') stay resident in shared memory.
//   Frame m: packed buffer z[n] = x[m H + tau] (g[tau+c] + i alpha g'[tau+c]), n = tau mod N_f
//   (circular placement == Eq. 9's phase factor e^{i 2 pi k M/N_f}).
//   N_f = 64 N2 four-step FFT: N2 threads per frame, each a 64-point register DFT of the decimated
//   row n2 = thread, twiddle W_N^{n2 k1}, one padded shared-memory exchange, then N2-point register
//   DFTs of columns.  Columns are assigned in conjugate pairs (k1, 64-k1) so that Z[k] and Z[N-k]
//   meet in one thread (N2 <= 32): the unpack S = (Z[k] + conj Z[N-k])/2,
//   S' = (Z[k] - conj Z[N-k])/(2 i alpha) is register-only.
//   Per source bin: mask |S| > gamma (Eq. 13), r = -Im(S'/S) N/(2 pi) (Eq. 36), target
//   l = z(k-k1) + floor(z r + 1/2) (Eq. 28, R17), shared-memory atomics into the frame's band
//   accumulator (Eq. 27/28), coalesced store of the band row.
//
// Inverse (rows a9-a11): two frames per complex IFFT (Hermitian packing), the z N_f-point band
//   IDFT of P:L222 split into z N_f-point sub-transforms by residue b = j mod z; work item =
//   (frame pair, b), one per group; outer phase e^{i 2 pi b tau/(z N)}; the CTA sums a pair's
//   items, windows by g[tau+c]/N_f and overlap-adds frame A (real part) and frame B (imaginary
//   part) into a shared-memory ring (Eq. 26).  Samples shared with the neighbouring CTA go to a
//   seam buffer combined by a second small kernel.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace sst {

// seam i (1..ctas-1) joins the right seam of CTA i-1 and the left seam of CTA i
__global__ void seam_kernel(const InvArgs a, int ctas) {
    const int64_t total = (int64_t)(ctas - 1) * a.seam_len;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = 1 + idx / a.seam_len;
        const int64_t t = idx % a.seam_len;
        const int64_t s = (a.frame_begin + i * a.frames_per_cta) * a.hop - a.c + t;
        if (s < 0 || s >= a.n) continue;
        const float val = a.seam[(i * 2 + 0) * a.seam_len + t] + a.seam[((i - 1) * 2 + 1) * a.seam_len + t];
        if (a.normalize) a.y[s - a.y_off] = val * inv_norm(s, a) * a.out_scale;
        else             a.y[s - a.y_off] += val;
    }
}

// y = (y + seam) / (C d[n]) on [y_off, y_off + y_len): the received rank seam (partial OLA sums of the
// neighbouring rank's frames, Eq. 26) is added in the same pass that normalises (seam == nullptr: none)
__global__ void finalize_kernel(float* y, int64_t y_off, int64_t y_len, InvArgs a, const float* seam,
                                int64_t seam_off, int64_t seam_len) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    // r = (s + c) mod hop, advanced incrementally (one 64-bit modulo per thread)
    int r = (int)(((y_off + i + a.c) % a.hop + a.hop) % a.hop);
    const int step = (int)(stride % a.hop);
    for (; i < y_len; i += stride) {
        const int64_t s = y_off + i;
        if (s >= 0 && s < a.n) {
            float v = y[i];
            if (seam && s >= seam_off && s < seam_off + seam_len) v += seam[s - seam_off];
            y[i] = v * inv_norm_r(s, r, a) * a.out_scale;
        }
        r += step;
        r -= (r >= a.hop) ? a.hop : 0;
    }
}

// ------------------------------------------------------------------------------- R23 ---------
constexpr int kRedecideSplit = 8;   // CTAs per queue region (latency hiding: the per-bin sums are long)
// Deferred fp64 re-decisions (reading R23): one warp per queued bin (frame within the launch, k, fp32
// target), the direct Eq. 8 sum over the frame's samples in global memory, the oracle's decision in
// fp64.  Targets mode: the fp64 target is written to a.lout.  Forward mode: a frame whose target
// changed is listed once (dirty_bits / dirty_list / a.gq_n[1]) for the list-mode repair launch.
__global__ void __launch_bounds__(256) redecide_kernel(const FwdArgs a, int mode, unsigned int* dirty_bits,
                                                      int* dirty_list) {
    // one CTA per queue region (the main launch's CTA b), 8 lanes per queued bin: lane u of the
    // octet takes taps j = u + 8 t of the direct Eq. 8 sum (a load instruction covers 4 bins x 8
    // consecutive samples), with the twiddle recurrence w <- w W^{8 k} from W^{k (u - c)}
    // (<= L/8 fp64 complex products, ~1e-14 relative); fixed 3-level xor reduction (deterministic)
    const unsigned reg = a.gq_cap / a.gq_ctas;
    const int b = blockIdx.x / kRedecideSplit;              // queue region (main launch's CTA)
    const int sub = blockIdx.x % kRedecideSplit;            // this CTA's share of the region
    const unsigned cnt = __ldg(a.gq_counts + b);
    const double gam64 = launch_gamma64(a);
    const int64_t v_lo = a.x_off > 0 ? a.x_off : 0;
    const int64_t v_hi = min(a.n, a.x_off + a.x_len);
    const int64_t K = a.nfft / 2 + 1;
    const unsigned msk = (unsigned)a.nfft - 1u;
    const int u = threadIdx.x & 7;
    const unsigned per = 32 * kRedecideSplit;                        // bins per pass over the region's CTAs
    const unsigned rounds = (cnt + per - 1) / per;
    for (unsigned r = 0; r < rounds; ++r) {
        const unsigned e = r * per + sub * 32 + (threadIdx.x >> 3);
        const bool ok = e < cnt;
        const int4 it = ok ? a.gq[(size_t)b * reg + e] : make_int4(0, 0, 0, 0);
        const int64_t s0 = (a.frame_begin + it.x) * a.hop - a.c;
        const int k = it.y;
        double2 w = __ldg(a.tw64 + (((unsigned)k * (unsigned)(u - a.c)) & msk));   // W^{k (u - c)}
        const double2 st = __ldg(a.tw64 + ((8u * (unsigned)k) & msk));             // W^{8 k}
        double sr = 0.0, si = 0.0, dr = 0.0, di = 0.0;
        if (ok) {
#pragma unroll 4
            for (int j = u; j < a.L; j += 8) {
                const int64_t sj = s0 + j;
                const double xv = (sj >= v_lo && sj < v_hi) ? (double)__ldg(a.x + (sj - a.x_off)) : 0.0;
                const double2 g = __ldg(a.taps64 + j);
                const double p = xv * g.x, q = xv * g.y;
                sr = fma(p, w.x, sr);
                si = fma(p, w.y, si);
                dr = fma(q, w.x, dr);
                di = fma(q, w.y, di);
                const double wr = fma(w.x, st.x, -w.y * st.y);
                w.y = fma(w.x, st.y, w.y * st.x);
                w.x = wr;
            }
        }
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) {
            sr += __shfl_xor_sync(0xffffffffu, sr, o);
            si += __shfl_xor_sync(0xffffffffu, si, o);
            dr += __shfl_xor_sync(0xffffffffu, dr, o);
            di += __shfl_xor_sync(0xffffffffu, di, o);
        }
        if (!ok || u != 0) continue;
        const int ln = decide_fp64(a, gam64, k, sr, si, dr, di);
        atomicAdd(a.r23_count, 1ull);
        if (ln != it.z) {
            atomicAdd(a.r23_count + 1, 1ull);
            if (mode == kModeTargets) {
                a.lout[(int64_t)it.x * K + k] = ln;
            } else {
                const unsigned bit = 1u << (it.x & 31);
                if (!(atomicOr(dirty_bits + (it.x >> 5), bit) & bit)) dirty_list[atomicAdd(a.gq_n, 1u)] = it.x;
            }
        }
    }
}

cudaError_t launch_redecide(const FwdArgs& a, int mode, unsigned int* dirty_bits, int* dirty_list, cudaStream_t s) {
    redecide_kernel<<<a.gq_ctas * kRedecideSplit, 256, 0, s>>>(a, mode, dirty_bits, dirty_list);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------- Renyi -------
__global__ void __launch_bounds__(256) renyi_partial_kernel(const float2* T, int64_t rows, int64_t cols,
                                                            int64_t ldT, double alpha, double* partial) {
    double s1 = 0.0, sa = 0.0;
    const bool cube = (alpha == 3.0);
    auto acc = [&](float2 v) {
        const double p = (double)v.x * v.x + (double)v.y * v.y;         // P = |T|^2
        s1 += p;
        sa += cube ? p * p * p : pow(p, alpha);
    };
    if (ldT == cols && (cols & 1) == 0 && (reinterpret_cast<uintptr_t>(T) & 15) == 0) {
        // dense plane: one flat grid-stride pass, two coefficients per 16-byte load
        const float4* T4 = reinterpret_cast<const float4*>(T);
        const int64_t n4 = rows * cols / 2;
        const int64_t stride = (int64_t)gridDim.x * blockDim.x;
        int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
        for (; i + 3 * stride < n4; i += 4 * stride) {                  // 4 loads in flight per thread
            float4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = __ldcs(T4 + i + u * stride);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                acc(make_float2(v[u].x, v[u].y));
                acc(make_float2(v[u].z, v[u].w));
            }
        }
        for (; i < n4; i += stride) {
            const float4 v = __ldcs(T4 + i);
            acc(make_float2(v.x, v.y));
            acc(make_float2(v.z, v.w));
        }
    } else {
        for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
            const float2* row = T + r * ldT;
            for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) acc(row[c]);
        }
    }
    __shared__ double r1[256], ra[256];
    r1[threadIdx.x] = s1;
    ra[threadIdx.x] = sa;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            r1[threadIdx.x] += r1[threadIdx.x + o];
            ra[threadIdx.x] += ra[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        partial[2 * blockIdx.x] = r1[0];
        partial[2 * blockIdx.x + 1] = ra[0];
    }
}

__global__ void renyi_final_kernel(const double* partial, int n, double alpha, double* out) {
    if (threadIdx.x != 0) return;
    double s1 = 0.0, sa = 0.0;
    for (int i = 0; i < n; ++i) {
        s1 += partial[2 * i];
        sa += partial[2 * i + 1];
    }
    out[0] = s1;
    out[1] = sa;
    out[2] = log2(sa / pow(s1, alpha)) / (1.0 - alpha);      // Eq. 32
}

cudaError_t launch_renyi(const float2* T, int64_t rows, int64_t cols, int64_t ldT, double alpha, double* partial,
                         double* out, cudaStream_t s) {
    renyi_partial_kernel<<<kRenyiBlocks, 256, 0, s>>>(T, rows, cols, ldT, alpha, partial);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    renyi_final_kernel<<<1, 32, 0, s>>>(partial, kRenyiBlocks, alpha, out);
    return cudaGetLastError();
}

cudaError_t launch_finalize(float* y, int64_t y_off, int64_t y_len, int64_t n, int32_t hop, int32_t c,
                            const float* inv_head, int32_t n_head, const float* inv_tail, int32_t n_tail,
                            const float* inv_per, float out_scale, cudaStream_t s, const float* seam,
                            int64_t seam_off, int64_t seam_len) {
    InvArgs a{};
    a.out_scale = out_scale;
    a.n = n; a.hop = hop; a.c = c;
    a.inv_head = inv_head; a.n_head = n_head; a.inv_tail = inv_tail; a.n_tail = n_tail; a.inv_per = inv_per;
    const int threads = 256;
    const int64_t want = (y_len + threads - 1) / threads;
    const int blocks = (int)(want < 2368 ? want : 2368);
    if (blocks <= 0) return cudaSuccess;
    finalize_kernel<<<blocks, threads, 0, s>>>(y, y_off, y_len, a, seam, seam_off, seam_len);
    return cudaGetLastError();
}


// ------------------------------------------------------------------------------- dispatch -----
#define SST_DECL_N2(n2)                                                                     \
    cudaError_t launch_fwd_n2_##n2(const FwdArgs& a, int mode, int grid, cudaStream_t s);    \
    int occ_fwd_n2_##n2(int L, int H, int device);                                          \
    cudaError_t launch_inv_n2_##n2(const InvArgs& a, int grid, cudaStream_t s);              \
    int occ_inv_n2_##n2(int hop, int L, int zoom, int device);                              \
    int occ_inv_nb_n2_##n2(int hop, int L, int zoom, int k1, int bins, int device);
SST_DECL_N2(2)
SST_DECL_N2(4)
SST_DECL_N2(8)
SST_DECL_N2(16)
SST_DECL_N2(32)
SST_DECL_N2(64)
SST_DECL_N2(128)
#undef SST_DECL_N2

#define SST_SWITCH_N2(nfft, CALL)                 \
    switch (nfft) {                               \
        case 128: return CALL(2);                 \
        case 256: return CALL(4);                 \
        case 512: return CALL(8);                 \
        case 1024: return CALL(16);               \
        case 2048: return CALL(32);               \
        case 4096: return CALL(64);               \
        case 8192: return CALL(128);              \
    }

cudaError_t launch_forward(const FwdArgs& a, int mode, int grid, cudaStream_t s) {
#define SST_CALL(n2) launch_fwd_n2_##n2(a, mode, grid, s)
    SST_SWITCH_N2(a.nfft, SST_CALL)
#undef SST_CALL
    return cudaErrorInvalidValue;
}

int forward_max_grid(int nfft, int L, int H, int device) {
#define SST_CALL(n2) occ_fwd_n2_##n2(L, H, device)
    SST_SWITCH_N2(nfft, SST_CALL)
#undef SST_CALL
    return -1;
}

cudaError_t launch_inverse(const InvArgs& a, int grid, cudaStream_t s) {
#define SST_CALL(n2) launch_inv_n2_##n2(a, grid, s)
    SST_SWITCH_N2(a.nfft, SST_CALL)
#undef SST_CALL
    return cudaErrorInvalidValue;
}

int inverse_max_grid(int nfft, int hop, int L, int zoom, int device) {
#define SST_CALL(n2) occ_inv_n2_##n2(hop, L, zoom, device)
    SST_SWITCH_N2(nfft, SST_CALL)
#undef SST_CALL
    return -1;
}

int inverse_nb_max_grid(int nfft, int hop, int L, int zoom, int k1, int bins, int device) {
#define SST_CALL(n2) occ_inv_nb_n2_##n2(hop, L, zoom, k1, bins, device)
    SST_SWITCH_N2(nfft, SST_CALL)
#undef SST_CALL
    return 0;
}
#undef SST_SWITCH_N2

cudaError_t launch_inverse_seams(const InvArgs& a, int ctas, cudaStream_t s) {
    if (ctas < 2 || a.seam_len <= 0) return cudaSuccess;
    const int64_t total = (int64_t)(ctas - 1) * a.seam_len;
    const int threads = 256;
    const int64_t want = (total + threads - 1) / threads;
    const int blocks = (int)(want < 4096 ? want : 4096);
    seam_kernel<<<blocks, threads, 0, s>>>(a, ctas);
    return cudaGetLastError();
}

}  // namespace sst
