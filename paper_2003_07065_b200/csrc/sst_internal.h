// Internal interface between the host API (sst_api.cu) and the kernels (sst_forward.cu,
// sst_inverse.cu).  Not part of the ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace sst {

constexpr int kCtaThreads = 128;        // threads per CTA for both kernels
constexpr int kMinLogN = 7;             // N_f = 64 * N2, N2 in [2, 64]
constexpr int kMaxLogN = 12;

enum FwdMode : int { kModeForward = 0, kModeStft = 1, kModeTargets = 2, kModeAbsmax = 3 };

struct FwdArgs {
    const float* x;          // points at global sample x_off
    int64_t x_off;
    int64_t n;               // N
    int64_t frame_begin, frame_end;
    int32_t hop, L, c, nfft;
    const float2* taps;      // [L] (g, alpha g')
    const float2* tw;        // [nfft] W_N^i = exp(-2 pi i i/N)
    int32_t k1, k2, bins, zoom;
    int32_t src_lo, src_hi;  // source bins reassigned: [src_lo, src_hi) (truncate flag)
    float gamma2x4;          // 4 gamma^2 (mask on P^2 + Q^2 = 4|S|^2), used if gamma_dev == null
    const float* absmax_dev; // relative mode: gamma = gamma_rel * (*absmax_dev)
    float gamma_rel;
    float r_scale;           // N_f / (2 pi alpha)
    float inv_alpha2;        // 1 / (2 alpha)
    // outputs
    float2* T; int64_t ldT;
    float2* S; float2* Sd;   // kModeStft
    int32_t* lout;           // kModeTargets
    float* absmax_out;       // kModeAbsmax (atomicMax on float bits)
};

struct InvArgs {
    const float2* T; int64_t ldT;
    int64_t n;
    int64_t frame_begin, frame_end;   // frames in this launch; T row 0 = frame_begin
    int32_t hop, L, c, nfft, zoom, k1, bins;
    const float2* taps;               // .x = g
    const float2* tw;                 // [nfft] W_N^i forward (conj used)
    const float2* twz;                // [zoom*nfft] exp(+2 pi i e/(z N))
    float inv_n;                      // 1 / N_f
    // output
    float* y; int64_t y_off, y_len;
    int normalize;                    // 1: write x_hat = sum / (C d) (y overwritten); 0: y += sum
    const float* inv_head; int32_t n_head;   // 1/(C d[n]) for n in [0, n_head)
    const float* inv_tail; int32_t n_tail;   // for n in [N - n_tail, N)
    const float* inv_per;             // [hop] for interior n: index (n + c) mod hop
    float* seam;                      // [ctas][2][seam_len] partial sums
    int32_t seam_len;                 // L - hop
    int64_t frames_per_cta;           // contiguous chunk per CTA (>= ceil(L/hop))
    int32_t ring;                     // ring buffer length (power of two)
};

// launchers (return cudaGetLastError())
cudaError_t launch_forward(const FwdArgs& a, int mode, int grid, cudaStream_t s);
int forward_smem_bytes(int nfft);
int forward_max_grid(int nfft, int device);

cudaError_t launch_inverse(const InvArgs& a, int grid, cudaStream_t s);
cudaError_t launch_inverse_seams(const InvArgs& a, int grid, cudaStream_t s);
cudaError_t launch_finalize(float* y, int64_t y_off, int64_t y_len, int64_t n, int32_t hop, int32_t c,
                            const float* inv_head, int32_t n_head, const float* inv_tail, int32_t n_tail,
                            const float* inv_per, cudaStream_t s);
int inverse_smem_bytes(int nfft, int hop, int L, int* ring_out);
int inverse_max_grid(int nfft, int hop, int L, int device);

// constant-memory table W_64^e (forward), uploaded once per device by the API
cudaError_t upload_w64(const float2* w64_host);

}  // namespace sst
