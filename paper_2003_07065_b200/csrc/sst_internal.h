// Internal interface between the host API (sst_api.cu) and the kernels (sst_kernels.cu).
// Not part of the ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

// SST_BOUNDS (debug build libsst_bounds.so, `python __graft_entry__.py build bounds`): device-side
// checks of every shared-memory and global index the kernels compute, and a spin limit on mbarrier
// waits (a lost TMA completion traps instead of hanging).  compute-sanitizer is closed on the GPU
// pool, so `SST_LIB=bounds pytest -m gpu` is the memory-safety run.
#ifdef SST_BOUNDS
#include <cstdio>
#define SST_CHECK(cond)                                                                            \
    do {                                                                                           \
        if (!(cond)) {                                                                             \
            printf("SST_BOUNDS: %s failed at %s:%d (block %d thread %d)\n", #cond, __FILE__, __LINE__, \
                   (int)blockIdx.x, (int)threadIdx.x);                                             \
            __trap();                                                                              \
        }                                                                                          \
    } while (0)
#else
#define SST_CHECK(cond) ((void)0)
#endif

namespace sst {

enum FwdMode : int { kModeForward = 0, kModeStft = 1, kModeTargets = 2, kModeAbsmax = 3 };

// Threads per CTA: 128, or 256 for N_f = 4096 (two-warp frames).  G = TPB / N2 frames
// (forward) or frame pairs (inverse) in flight per CTA, N_f = 64 N2.
// threads per CTA: 256 for N_f = 4096 (two-warp frames) and for the N_f = 2048 forward (8 frames
// per CTA, measured 3 % faster than 4); 128 otherwise.  G = TPB / N2 frames (forward) or frame
// pairs (inverse) in flight per CTA, N_f = 64 N2.
__host__ __device__ constexpr int tpb_of(int n2, bool fwd) { return (n2 == 64 || (fwd && n2 == 32)) ? 256 : 128; }
__host__ __device__ constexpr int groups_of(int n2, bool fwd) { return tpb_of(n2, fwd) / n2; }
// float2 per group buffer: the 64 x (N2 + 1) padded exchange, plus N2 float2 when several groups share
// a warp so consecutive groups start N2 float2 apart in the banks (conflict-free 64-bit half-warps)
__host__ __device__ constexpr int cap_of(int n2) { return 64 * (n2 + 1) + (n2 < 16 ? n2 : 0); }
__host__ __device__ constexpr int round_up(int v, int m) { return (v + m - 1) / m * m; }
__host__ __device__ constexpr int ceil_log2_c(int v) { return v <= 1 ? 0 : 1 + ceil_log2_c((v + 1) / 2); }

// forward dynamic shared memory: [G exchange buffers][taps L float2][2 input tiles][2 mbarriers]
constexpr int kFwdStaticSmem = 1024;   // the forward's static shared memory (reductions, counters), bound
struct FwdLayout {
    int taps_off, xb_off, mbar_off, xcap, total;
};
__host__ __device__ inline FwdLayout fwd_layout(int n2, int L, int H) {
    FwdLayout f{};
    const int G = groups_of(n2, true);
    f.taps_off = G * cap_of(n2) * 8;
    f.xb_off = f.taps_off + round_up(L * 8, 16);
    f.xcap = round_up((G - 1) * H + L + 8, 4);          // floats per input tile buffer
    f.mbar_off = f.xb_off + 2 * f.xcap * 4;
    f.total = f.mbar_off + 16;
    return f;
}

// inverse dynamic shared memory: [G exchange buffers][window g, L floats][OLA ring]
struct InvLayout {
    int g_off, ring_off, ring, pairs, total;
};
__host__ __device__ inline InvLayout inv_layout(int n2, int L, int H, int zoom) {
    InvLayout v{};
    const int G = groups_of(n2, false);
    v.pairs = G / zoom > 1 ? G / zoom : 1;
    v.g_off = G * cap_of(n2) * 8;
    v.ring_off = v.g_off + round_up(L * 4, 16);
    const int span = (2 * v.pairs - 1) * H + L;
    int r = 1;
    while (r < span) r <<= 1;
    v.ring = r;
    v.total = v.ring_off + r * 4;
    return v;
}

// narrow-band inverse (inv_nb_kernel.cuh): the z N_f-point band IDFT as 64 x J (J = z N2) with the
// sum over residues inside the second stage (warp shuffles) instead of a shared-memory round trip.
// Applies to full windows (L = N_f, c = N_f / 2) with
//   narrow band: N_f in {1024, 2048}, z in {1, 2, 4, 8}, band/mirror rows within 8 of the 64 (C2, C3);
//   full band:   N_f = 512, z in {4, 8}, k1 = 0 and B = z N_f / 2 (C5).
// T staging buffers of the narrow-band form: 2 (the copy of pair p + 1 is issued when pair p starts)
// or 1 (issued after pair p's last stage-1 read; half the shared footprint)
#ifndef SST_NB_TBUF
#define SST_NB_TBUF 1
#endif
// full band: 1 = the pair's T rows staged by TMA (one buffer, issued after the previous pair's inputs
// are read; C5 inverse 22.5 ms per 2^24 samples); 0 = loaded straight into registers (24.2 ms)
#ifndef SST_NB_FULL_TMA
#define SST_NB_FULL_TMA 1
#endif
__host__ __device__ inline int inv_nb_rows(int n2, int k1, int bins, int zoom) { return (k1 + bins / zoom + n2 - 1) / n2; }
__host__ __device__ inline bool inv_nb_full(int nfft, int zoom, int k1, int bins) {
    return nfft == 512 && (zoom == 4 || zoom == 8) && k1 == 0 && bins == zoom * nfft / 2;
}
__host__ __device__ inline bool inv_nb_applicable(int nfft, int L, int c, int hop, int zoom, int k1, int bins) {
    const int n2 = nfft / 64;
    if (L != nfft || c != nfft / 2 || hop < 1 || hop > L) return false;
    if (inv_nb_full(nfft, zoom, k1, bins)) return true;
    if (n2 != 16 && n2 != 32) return false;
    if (zoom != 1 && zoom != 2 && zoom != 4 && zoom != 8) return false;
    return inv_nb_rows(n2, k1, bins, zoom) <= 8;
}
// [chunk buffer: RPC rows (narrow: N2, full: 32) x (J + z) float2][OLA ring: ring = round_up(L + 3 hop,
// 64 z) slots (sample index mod ring), stored bank-skewed (inv_nb_kernel.cuh: up to ring / (2 z) + 32
// more floats)][narrow: T staging, SST_NB_TBUF buffers x 2 rows x round_up(B + 1, 2) float2 (entry B: a
// zero), 2 mbarriers]   (g_off = T staging offset)
__host__ __device__ inline InvLayout inv_nb_layout(int n2, int L, int H, int zoom, int bins) {
    InvLayout v{};
    const bool full = inv_nb_full(64 * n2, zoom, 0, bins);
    v.pairs = 1;
    v.ring_off = round_up((full ? 32 : n2) * (zoom * n2 + zoom) * 8, 16);
    v.ring = round_up(L + 3 * H, 64 * zoom);
    v.g_off = round_up(v.ring_off + (v.ring + (zoom > 1 ? v.ring / (2 * zoom) : 0) + 64) * 4, 16);
    v.total = full ? (SST_NB_FULL_TMA ? v.g_off + 2 * round_up(bins + 1, 2) * 8 + 16 : v.g_off)
                   : v.g_off + SST_NB_TBUF * 2 * round_up(bins + 1, 2) * 8 + 16;
    return v;
}

struct FwdArgs {
    const float* x;          // points at global sample x_off
    int64_t x_off, x_len;
    int64_t n;               // N
    int64_t frame_begin, frame_end;
    int32_t hop, L, c, nfft;
    const float2* taps;      // [L] (g, alpha g')
    const float2* tw;        // [nfft] tw[k1 * N2 + t] = W_N^{t k1}
    int32_t k1, k2, bins, zoom;
    int32_t src_lo, src_hi;  // source bins reassigned: [src_lo, src_hi) (truncate flag)
    float gamma2x4;          // 4 gamma^2 (mask on P^2 + Q^2 = 4|S|^2), used if absmax_dev == null
    const float* absmax_dev; // relative mode: gamma = gamma_rel * (*absmax_dev)
    float gamma_rel;
    float r_scale;           // N_f / (2 pi alpha)
    float zr_scale;          // z N_f / (2 pi alpha)
    double r_scale_d;        // same, fp64 (near-boundary re-decision)
    float inv_alpha2;        // 1 / (2 alpha)
    // R23 fp64 re-decision of bins the fp32 FFT cannot decide (decide.cuh)
    int redecide;            // 1: on (forward / targets); 0: off (stft / absmax, or SST_NO_REDECIDE)
    float cflag;             // 8 zr_scale 4 u sqrt(log2 N_f): margin of the fine position per unit ||z_m||
    float kflag;             // 8 * 2 u sqrt(log2 N_f): margin of |S| per unit ||z_m||
    double gamma_d;          // absolute gamma (fp64)
    double gamma_rel_d;      // relative mode: gamma = gamma_rel_d * (*absmax_dev)
    const double2* taps64;   // [L] (g, g') fp64
    const double2* tw64;     // [nfft] exp(-2 pi i e / N_f) fp64
    int32_t* lscratch;       // multi-pass: [frames][N_f/2 + 1] targets of the chunk
    unsigned long long* r23_count;   // [2]: bins re-decided, of which the fp64 target differed
    // R23 deferral: flagged bins are squeezed at their fp32 target and queued (frame within the
    // launch, k, fp32 target); redecide_kernel re-takes them in fp64 and lists the frames whose target
    // changed; a list-mode launch (flist) recomputes those rows with inline re-decision
    int4* gq;                        // queue (nullptr: inline re-decision only): CTA b owns entries
                                     // [b * (gq_cap / grid), ...), counted in gq_counts[b]
    unsigned int* gq_counts;         // [grid] entries each CTA queued
    unsigned int* gq_n;              // [1]: dirty frames (redecide_kernel)
    unsigned int gq_cap;
    int gq_ctas;                     // grid of the launch that filled the queue (redecide_kernel)
    const int* flist;                // list mode: frames (within the launch) to process, one per tile
    const unsigned int* flist_n;     // list mode: device count
    FwdLayout lay;
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
    const float* gwin;                // [L] g / N_f (narrow-band kernel)
    const float2* tw;                 // [nfft] tw[k1 * N2 + t] = W_N^{t k1} (conjugated here)
    const float2* phz;                // [z][64 + 2 N2] phase factors of exp(+2 pi i b tau/(z N)), see sst_api.cu
    float inv_n;                      // 1 / N_f
    InvLayout lay;
    // output
    float* y; int64_t y_off, y_len;
    int normalize;                    // 1: write x_hat = sum / (C d) (y overwritten); 0: y += sum
    float out_scale;                  // extra factor at normalisation (1; C for the plain STFT synthesis)
    const float* inv_head; int32_t n_head;   // 1/(C d[n]) for n in [0, n_head)
    const float* inv_tail; int32_t n_tail;   // for n in [N - n_tail, N)
    const float* inv_per;             // [hop] for interior n: index (n + c) mod hop
    float* seam;                      // [ctas][2][seam_len] partial sums
    int32_t seam_len;                 // L - hop
    int64_t frames_per_cta;           // contiguous chunk per CTA (>= ceil(L/hop))
    // zone of mode retrieval (R22) applied to the T loads: entry l of frame m is used only if
    // (|l - zone_path[m]| <= zone_half) == zone_keep; zone_path == nullptr: no zone.  zone_path[0]
    // is frame frame_begin.
    const int32_t* zone_path;
    int32_t zone_half, zone_keep;
    int32_t nb;                       // 1: narrow-band kernel (inv_nb_kernel.cuh; lay = inv_nb_layout)
};

// Frequency-domain filter-bank STFT for truncated narrow bands (filterbank.cu)
struct FbArgs {
    const float* x;
    int64_t x_off, x_len, n;
    int64_t frame_begin, frame_end;   // frames of the launch (global indices)
    int32_t hop, c;
    int32_t ns, lg_ns, P, lg_P;       // block segment length Ns, fold length P = Ns / H
    int32_t fb, kc;                   // frames per block, band bins per staging chunk
    int32_t ratio;                    // Ns / N_f
    int32_t kb0, kb;                  // source bins [kb0, kb0 + kb) (= [k1, k2), SST_SOURCE_TRUNCATE)
    const float2* gam;                // [Ns] Gamma[d] of g   (sum_j g[j] e^{2 pi i d j / Ns})
    const float2* gamd;               // [Ns] of g'
    const float2* ph;                 // [kb] e^{2 pi i k c / N_f} / Ns
    const float2* twns;               // [Ns / 2] e^{-2 pi i e / Ns}
    const float2* twp;                // [P / 2] e^{+2 pi i e / P}
    float2* S; float2* Sd;            // planes [frames of the launch][kb]
    float* eta;                       // [frames of the launch] ||x_b||_2 of the frame's block
    float cflag, kflag;               // R23 margins per unit eta (filter-bank error model)
    float alpha;
};
int fb_transform_smem(const FbArgs& a);
cudaError_t launch_fb_transform(const FbArgs& a, cudaStream_t s);
cudaError_t launch_fb_squeeze(const FbArgs& fb, const FwdArgs& a, int grid, cudaStream_t s);
int fb_squeeze_grid(int device);

// Large-N_f multi-pass path (multipass.cu), used for kMaxFusedNfft < N_f <= kMaxNfft
constexpr int kMaxFusedNfft = 8192;
constexpr int kMaxNfft = 65536;
constexpr int kMpBinChunk = 8192;      // band bins per squeeze pass (16 B each in shared memory)

struct MpInvArgs {
    const float2* T; int64_t ldT;     // row 0 = frame_begin
    int64_t n;
    int64_t frame_begin, frame_end;
    int32_t hop, L, c, nfft, zoom, k1, bins;
    const float2* taps;               // .x = g
    const float2* twN;                // [nfft] W_N^k
    float inv_n;                      // 1 / N_f
    float2* buf0; float2* buf1;       // [ceil(F/2) z][nfft] each
    float* wf;                        // [F][L] windowed frames
    float* y; int64_t y_off, y_len;   // y += (accumulate)
    int direct;                       // 1: direct band sum per frame (mp_direct_kernel) instead of FFTs
    const int32_t* zone_path;         // as InvArgs (row 0 = frame frame_begin)
    int32_t zone_half, zone_keep;
};

void mp_factor(int nfft, int* r1, int* m);
int mp_bins_chunk(int bins);
// frames [frame_begin, frame_end) of the forward in one batch (scratch for all of them)
cudaError_t launch_mp_forward(const FwdArgs& a, int mode, const float2* twN, float2* buf0, float2* buf1,
                              cudaStream_t s);
cudaError_t launch_mp_inverse_accumulate(const MpInvArgs& a, cudaStream_t s);

// launchers (return cudaGetLastError())
cudaError_t launch_forward(const FwdArgs& a, int mode, int grid, cudaStream_t s);
// R23 deferred re-decisions of the queue a.gq (forward: dirty frames -> dirty_bits / dirty_list /
// a.gq_n[1]; targets: the fp64 targets written to a.lout)
cudaError_t launch_redecide(const FwdArgs& a, int mode, unsigned int* dirty_bits, int* dirty_list, cudaStream_t s);
int forward_max_grid(int nfft, int L, int H, int device);

cudaError_t launch_inverse(const InvArgs& a, int grid, cudaStream_t s);
cudaError_t launch_inverse_seams(const InvArgs& a, int grid, cudaStream_t s);
cudaError_t launch_finalize(float* y, int64_t y_off, int64_t y_len, int64_t n, int32_t hop, int32_t c,
                            const float* inv_head, int32_t n_head, const float* inv_tail, int32_t n_tail,
                            const float* inv_per, float out_scale, cudaStream_t s, const float* seam = nullptr,
                            int64_t seam_off = 0, int64_t seam_len = 0);
int inverse_max_grid(int nfft, int hop, int L, int zoom, int device);
// resident CTAs of the narrow-band inverse (0: not applicable)
int inverse_nb_max_grid(int nfft, int hop, int L, int zoom, int k1, int bins, int device);

// Renyi sums over a complex64 plane: partial[2*blockIdx] = {sum |T|^2, sum |T|^(2 alpha)},
// then out = {sum, sum, entropy}; fixed reduction order
// mode retrieval (ridge.cu)
cudaError_t launch_ridge_emission(const float2* T, int64_t rows, int64_t cols, int64_t ldT,
                                  unsigned long long* scratch, double* E, double* floor_out, cudaStream_t s);
cudaError_t launch_ridge_dp(double* E, int64_t rows, int cols, double lam, int count, int suppress,
                            const double* floor_in, int32_t* back, int32_t* paths, cudaStream_t s);
cudaError_t launch_zone_mask(float2* T, int64_t rows, int cols, int64_t ldT, const int32_t* path, int half,
                             int keep_inside, cudaStream_t s);
cudaError_t launch_mode_full(const float2* T, int64_t rows, int cols, int64_t ldT, const int32_t* path, int half,
                             int dc_bin, double scale, float* x, cudaStream_t s);
constexpr int kRidgeMaxCols = 8000;    // DP rows of V, V', E, opt in shared memory (28 B per bin)

constexpr int kRenyiBlocks = 1184;
cudaError_t launch_renyi(const float2* T, int64_t rows, int64_t cols, int64_t ldT, double alpha, double* partial,
                         double* out, cudaStream_t s);


}  // namespace sst
