// Large-N_f path (8192 < N_f <= 65536; the paper's §5.2 uses N_f = 2^15).
//
// A frame's packed buffer (N_f complex64 = 256 KiB at 2^15) no longer fits one CTA's shared
// memory next to anything else, so the transform is a four-step FFT split over a thread-block
// cluster of 8 CTAs (mp_cluster_kernel):
//   N_f = R1 M.  Stage 1: for every column a in [0, M) a P = R1-point DFT of x[a + M i], times
//   W_N^{a k1}, kept at [k1][a] in the shared memory of the CTA owning column a.  Stage 2: every
//   CTA reads its rows k1 from all 8 CTAs through distributed shared memory, runs P = M-point
//   DFTs over a and writes k1 + R1 k2 (natural order) once.  Each CTA works on tiles of 16
//   adjacent columns / rows, so every global load and store moves 128-byte segments, and runs a
//   radix-4 Stockham (autosort) FFT over them in shared memory with twiddles rounded once from
//   fp64 (the plan's W_N table).  (The two-pass form through an HBM scratch, mp_pass_kernel, is
//   kept for A/B timing: SST_MP_TWO_PASS=1.)
// Forward: stage 1 gathers and packs the frame on the fly (a1: z[n] = u (g + i alpha g'), circular
// placement, as in the fused kernel), stage 2 writes the spectrum, and one CTA per frame then does
// a3-a7 with the fused path's own per-bin decision (decide.cuh) and an exact 64-bit fixed-point
// squeeze in shared memory (order-independent, so bitwise reproducible).
// Inverse: per frame pair and residue b the Hermitian-packed sub-spectrum G_b (the fused
// inverse's split of the z N_f IDFT) is gathered from T in stage 1, transformed by
// both stages (conjugate twiddles), combined over b with e^{i 2 pi b tau/(z N)}, windowed by
// g[tau + c]/N_f (a9), and overlap-added by a gather kernel (one thread per output sample,
// frames in ascending order: no atomics, deterministic) (a10, Eq. 26).  For narrow bands with a
// large z (B L small against z N_f log N_f, e.g. the §5.2 Fig. 16(e) shape, z = 20) the plan
// picks a direct band sum per frame instead (mp_direct_kernel), with the same windowing and OLA.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "decide.cuh"
#include "sst_internal.h"

namespace sst {

namespace {

constexpr int kTile = 16;          // columns (pass 1) or rows (pass 2) per CTA
constexpr int kTS = kTile + 1;     // padded smem row: conflict-free column and row access
constexpr int kPassThreads = 256;
constexpr int kBinThreads = 512;
constexpr int kLoadBuf = 0, kLoadFwd = 1, kLoadInv = 2;

struct MpPass {
    const float2* in;
    float2* out;
    int64_t count;                 // transforms in the batch
    int N, R1, M;                  // N = R1 M
    const float2* twN;             // [N] W_N^k = exp(-2 pi i k/N)
    // kLoadFwd: frame gather + pack
    const float* x;
    int64_t x_off, v_lo, v_hi, frame0;
    int hop, L, c;
    const float2* taps;
    // kLoadInv: Hermitian-packed residue sub-spectra from T
    const float2* T;
    int64_t ldT, nfr;
    int zoom, k1, bins;
    const int32_t* zone_path;       // mode retrieval zone (row 0 = first frame of the chunk), or null
    int zone_half, zone_keep;
};

__device__ __forceinline__ float2 c_mul(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

template <int DIR>
__device__ __forceinline__ float2 tw_at(const float2* twN, int64_t e) {
    const float2 w = __ldg(twN + e);
    return DIR < 0 ? w : make_float2(w.x, -w.y);
}

// element n (pass-1 index) of transform t
template <int LOAD>
__device__ __forceinline__ float2 load_elem(const MpPass& a, int64_t t, int n) {
    if constexpr (LOAD == kLoadBuf) {
        return a.in[t * a.N + n];
    } else if constexpr (LOAD == kLoadFwd) {
        const int tau = (n <= a.L - 1 - a.c) ? n : n - a.N;        // circular placement (Eq. 9)
        const int j = tau + a.c;
        if (j < 0) return make_float2(0.0f, 0.0f);
        const int64_t s = (a.frame0 + t) * a.hop - a.c + j;
        const float xv = (s >= a.v_lo && s < a.v_hi) ? __ldg(a.x + (s - a.x_off)) : 0.0f;
        const float2 w = __ldg(a.taps + j);
        return make_float2(w.x * xv, w.y * xv);
    } else {
        // transform t = (pair, b): G_b[q] = H_A[z q + b] + i H_B[z q + b]
        const int64_t pair = t / a.zoom;
        const int b = (int)(t - pair * a.zoom);
        const int64_t fA = 2 * pair;
        const bool vA = fA < a.nfr, vB = fA + 1 < a.nfr;
        const int q = n;
        const int nr = a.bins / a.zoom;
        const bool inb = (unsigned)(q - a.k1) < (unsigned)nr;
        const int lm = a.zoom * (a.N - a.k1 - q) - b;
        const bool inm = !inb && q > 0 && (unsigned)lm < (unsigned)a.bins;
        if (!(inb || inm)) return make_float2(0.0f, 0.0f);
        const int li = inb ? a.zoom * (q - a.k1) + b : lm;
        float2 ta = make_float2(0.0f, 0.0f), tb = make_float2(0.0f, 0.0f);
        auto zok = [&](int64_t f) {
            return !a.zone_path || ((abs(li - __ldg(a.zone_path + f)) <= a.zone_half) == (bool)a.zone_keep);
        };
        if (vA && zok(fA)) ta = __ldg(a.T + fA * a.ldT + li);
        if (vB && zok(fA + 1)) tb = __ldg(a.T + (fA + 1) * a.ldT + li);
        if (b == 0 && (q == 0 || q == a.N / 2)) { ta.y = 0.0f; tb.y = 0.0f; }   // DC / Nyquist real (R14)
        return inb ? make_float2(ta.x - tb.y, ta.y + tb.x) : make_float2(ta.x + tb.y, tb.x - ta.y);
    }
}

// P-point transforms of the 16 columns of x ([P][kTS], element i of column al at x[i kTS + al]),
// y the same-size scratch; every thread of the CTA (kPassThreads) calls it; returns the buffer
// holding the result (natural order).  Twiddles W_P^e = W_N^{e N/P} from the plan's table.
template <int P, int DIR, int NT = kPassThreads>
__device__ __forceinline__ float2* stockham16(float2* x, float2* y, int N, const float2* twN) {
    // Stockham (autosort) FFT over the 16 columns: radix-4 stages, then one radix-2 stage when
    // log2 P is odd.  Radix 4 at length n = P/s: for p < m = n/4, q < s, with A..D = x[q + s(p + j m)],
    //   y[q + s(4p + k)] = X_k W_n^{p k},  X = the 4-point DFT of (A, B, C, D)
    const int tstep = N / P;
    const int tid = threadIdx.x;
    int s = 1, ls = 0;
#pragma unroll 1
    for (; 4 * s <= P; s <<= 2, ls += 2) {
        const int m = P / (4 * s);
        for (int bf = tid; bf < kTile * P / 4; bf += NT) {
            const int al = bf & 15, rest = bf >> 4;
            const int q = rest & (s - 1), p = rest >> ls;
            const int i0 = (q + s * p) * kTS + al, im = s * m * kTS;
            const float2 A = x[i0], B = x[i0 + im], C = x[i0 + 2 * im], D = x[i0 + 3 * im];
            const float2 apc = make_float2(A.x + C.x, A.y + C.y), amc = make_float2(A.x - C.x, A.y - C.y);
            const float2 bpd = make_float2(B.x + D.x, B.y + D.y), bmd = make_float2(B.x - D.x, B.y - D.y);
            const float2 jb = DIR < 0 ? make_float2(bmd.y, -bmd.x) : make_float2(-bmd.y, bmd.x);   // -+i (B - D)
            const int64_t e = (int64_t)p * s * tstep;                       // W_n^p = W_N^{p s N/P}
            const int o0 = (q + 4 * s * p) * kTS + al, os = s * kTS;
            y[o0] = make_float2(apc.x + bpd.x, apc.y + bpd.y);
            y[o0 + os] = c_mul(make_float2(amc.x + jb.x, amc.y + jb.y), tw_at<DIR>(twN, e));
            y[o0 + 2 * os] = c_mul(make_float2(apc.x - bpd.x, apc.y - bpd.y), tw_at<DIR>(twN, 2 * e));
            y[o0 + 3 * os] = c_mul(make_float2(amc.x - jb.x, amc.y - jb.y), tw_at<DIR>(twN, 3 * e));
        }
        __syncthreads();
        float2* tmp = x; x = y; y = tmp;
    }
    if (s < P) {                                                        // last radix-2 stage (n = 2)
        for (int bf = tid; bf < kTile * P / 2; bf += NT) {
            const int al = bf & 15, q = bf >> 4;
            const float2 u = x[q * kTS + al], v = x[(q + s) * kTS + al];
            y[q * kTS + al] = make_float2(u.x + v.x, u.y + v.y);
            y[(q + s) * kTS + al] = make_float2(u.x - v.x, u.y - v.y);
        }
        __syncthreads();
        float2* tmp = x; x = y; y = tmp;
    }
    return x;
}

template <int P, int PASS, int LOAD, int DIR>
__global__ void __launch_bounds__(kPassThreads) mp_pass_kernel(const MpPass a) {
    extern __shared__ __align__(16) float2 mp_smem[];
    float2* s0 = mp_smem;
    float2* s1 = mp_smem + P * kTS;
    const int tiles = (PASS == 1 ? a.M : a.R1) / kTile;
    const int64_t t = blockIdx.x / tiles;
    const int tile = blockIdx.x - (int)(t * tiles);
    const int tid = threadIdx.x;
    if (PASS == 1) {
        for (int idx = tid; idx < P * kTile; idx += kPassThreads) {
            const int i = idx >> 4, al = idx & 15;
            s0[i * kTS + al] = load_elem<LOAD>(a, t, tile * kTile + al + a.M * i);
        }
    } else {
        for (int idx = tid; idx < P * kTile; idx += kPassThreads) {
            const int al = idx / P, i = idx - al * P;
            s0[i * kTS + al] = a.in[t * a.N + (int64_t)(tile * kTile + al) * a.M + i];
        }
    }
    __syncthreads();
    const float2* x = stockham16<P, DIR>(s0, s1, a.N, a.twN);
    for (int idx = tid; idx < P * kTile; idx += kPassThreads) {
        const int k = idx >> 4, al = idx & 15;
        const int a_ = tile * kTile + al;
        float2 v = x[k * kTS + al];
        if (PASS == 1) {
            if (a_ && k) v = c_mul(v, tw_at<DIR>(a.twN, ((int64_t)a_ * k) & (a.N - 1)));   // W_N^{a k1}
            a.out[t * a.N + a_ + (int64_t)a.M * k] = v;
        } else {
            a.out[t * a.N + a_ + (int64_t)a.R1 * k] = v;
        }
    }
}

template <int LOAD, int DIR>
cudaError_t run_pass(const MpPass& a, int pass, cudaStream_t s) {
    const int P = pass == 1 ? a.R1 : a.M;
    const int64_t blocks = a.count * ((pass == 1 ? a.M : a.R1) / kTile);
    if (blocks <= 0) return cudaSuccess;
    const int smem = 2 * P * kTS * (int)sizeof(float2);
#define SST_MP_CASE(PP)                                                                                 \
    case PP: {                                                                                          \
        auto kern = (pass == 1) ? mp_pass_kernel<PP, 1, LOAD, DIR> : mp_pass_kernel<PP, 2, kLoadBuf, DIR>; \
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);    \
        if (e != cudaSuccess) return e;                                                                 \
        kern<<<(unsigned)blocks, kPassThreads, smem, s>>>(a);                                           \
        break;                                                                                          \
    }
    switch (P) {
        SST_MP_CASE(64)
        SST_MP_CASE(128)
        SST_MP_CASE(256)
        default: return cudaErrorInvalidValue;
    }
#undef SST_MP_CASE
    return cudaGetLastError();
}

// f3a: both passes of the four-step FFT in one thread-block cluster of kClu CTAs per transform,
// the transpose between them through distributed shared memory.
// CTA `rank` owns the column tiles [rank CT, (rank + 1) CT) in stage 1 (R1-point DFTs of
// x[a + M i] times W_N^{a k1}, kept in its shared memory) and the row tiles [rank RT, (rank + 1) RT)
// in stage 2: it reads rows k1 of every column from the 8 CTAs' shared memory (DSMEM, 16-column
// segments), runs the M-point DFTs and writes Z[k1 + R1 k2] once.  The intermediate never reaches
// HBM or L2, so a transform costs one gather of its input and one write of its output (the
// two-pass path moves each frame through HBM/L2 twice more).  Buffers: stage 1 holds CT tiles of
// [R1][kTS] in each of two halves; stage 2's RT tiles of [M][kTS] fill the same half sizes
// (CT R1 = RT M = N / (16 kClu)): the gather lands in the free half, and after the cluster barrier
// that ends all remote reads the stage-1 half becomes stage 2's scratch.
constexpr int kClu = 8;
constexpr int kCluThreads = 512;

template <int R1, int M, int LOAD, int DIR>
__global__ void __cluster_dims__(kClu, 1, 1) __launch_bounds__(kCluThreads) mp_cluster_kernel(const MpPass a) {
    namespace cg = cooperative_groups;
    constexpr int CT = M / (kTile * kClu), RT = R1 / (kTile * kClu);
    constexpr int B1 = R1 * kTS, B2 = M * kTS;
    static_assert(CT >= 1 && RT >= 1 && CT * B1 == RT * B2, "cluster FFT tiling");
    extern __shared__ __align__(16) float2 mp_smem[];
    float2* const hA = mp_smem;
    float2* const hB = mp_smem + CT * B1;
    cg::cluster_group cl = cg::this_cluster();
    const int rank = (int)cl.block_rank();
    const int64_t t = blockIdx.x / kClu;
    const int tid = threadIdx.x;
    // stage 1: gather (and for the forward, pack) the columns, R1-point DFTs, twiddle
#pragma unroll 8
    for (int idx = tid; idx < CT * R1 * kTile; idx += kCluThreads) {
        const int ct = idx / (R1 * kTile), rem = idx - ct * (R1 * kTile);
        const int i = rem >> 4, al = rem & 15;
        hA[ct * B1 + i * kTS + al] = load_elem<LOAD>(a, t, (rank * CT + ct) * kTile + al + M * i);
    }
    __syncthreads();
    float2* res = hA;
#pragma unroll
    for (int ct = 0; ct < CT; ++ct) res = stockham16<R1, DIR, kCluThreads>(hA + ct * B1, hB + ct * B1, a.N, a.twN) - ct * B1;
    float2* const fre = res == hA ? hB : hA;
    for (int idx = tid; idx < CT * R1 * kTile; idx += kCluThreads) {
        const int ct = idx / (R1 * kTile), rem = idx - ct * (R1 * kTile);
        const int k = rem >> 4, al = rem & 15;
        const int a_ = (rank * CT + ct) * kTile + al;
        if (a_ && k) {
            float2& v = res[ct * B1 + k * kTS + al];
            v = c_mul(v, tw_at<DIR>(a.twN, ((int64_t)a_ * k) & (a.N - 1)));      // W_N^{a k1}
        }
    }
    cl.sync();                                            // stage-1 results visible cluster-wide
    // transpose through DSMEM: row tile r, rows k1 = (rank RT + r) 16 + k1l, all M columns
    constexpr int GATHER = RT * M * kTile;
#pragma unroll 4
    for (int idx = tid; idx < GATHER; idx += kCluThreads) {
        const int al = idx & 15, k1l = (idx >> 4) & 15, rest = idx >> 8;
        const int r = rest / (M / kTile), at = rest - r * (M / kTile);
        const int src = at / CT, ct = at - src * CT;
        const int k1 = (rank * RT + r) * kTile + k1l;
        const float2* rp = cl.map_shared_rank(res, src);
        fre[r * B2 + (at * kTile + al) * kTS + k1l] = rp[ct * B1 + k1 * kTS + al];
    }
    cl.sync();                                            // remote reads done: `res` is free
#pragma unroll
    for (int r = 0; r < RT; ++r) {
        const float2* x = stockham16<M, DIR, kCluThreads>(fre + r * B2, res + r * B2, a.N, a.twN);
        for (int idx = tid; idx < M * kTile; idx += kCluThreads) {
            const int k = idx >> 4, al = idx & 15;
            a.out[t * a.N + (rank * RT + r) * kTile + al + (int64_t)R1 * k] = x[k * kTS + al];
        }
    }
}

// The whole N-point transform of every item of the batch: pass 1 reads via LOAD, the result goes to
// `out` in natural order.  Cluster kernel for the shapes it tiles (all N_f the multi-pass path
// takes); the two-pass form through `tmp` otherwise or when SST_MP_TWO_PASS=1 (A/B timing).
template <int LOAD, int DIR>
cudaError_t run_fft(MpPass p, float2* tmp, float2* out, cudaStream_t s) {
    if (p.count <= 0) return cudaSuccess;
    static const bool two_pass = [] { const char* e = getenv("SST_MP_TWO_PASS"); return e && atoi(e) != 0; }();
    void (*kern)(const MpPass) = nullptr;
    if (!two_pass) {
        if (p.R1 == 128 && p.M == 128) kern = mp_cluster_kernel<128, 128, LOAD, DIR>;
        else if (p.R1 == 256 && p.M == 128) kern = mp_cluster_kernel<256, 128, LOAD, DIR>;
        else if (p.R1 == 256 && p.M == 256) kern = mp_cluster_kernel<256, 256, LOAD, DIR>;
    }
    cudaError_t e;
    if (kern && (int64_t)p.count * kClu < (int64_t)1 << 31) {
        const int smem = 2 * (p.N / (kTile * kClu)) * kTS * (int)sizeof(float2);
        if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)) != cudaSuccess) return e;
        p.out = out;
        kern<<<(unsigned)(p.count * kClu), kCluThreads, smem, s>>>(p);
        return cudaGetLastError();
    }
    p.out = tmp;
    if ((e = run_pass<LOAD, DIR>(p, 1, s)) != cudaSuccess) return e;
    p.in = tmp;
    p.out = out;
    return run_pass<kLoadBuf, DIR>(p, 2, s);
}

__device__ __forceinline__ float block_max(float v, float* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    float m = 0.0f;
    for (int w = 0; w < kBinThreads / 32; ++w) m = fmaxf(m, red[w]);
    return m;
}

__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    float m = 0.0f;
    for (int w = 0; w < kBinThreads / 32; ++w) m += red[w];
    return m;
}

// a3-a7 for one frame of the spectrum Z (natural order, N_f entries): one CTA per frame.
// Forward / targets: every bin is decided once (decide.cuh) into the frame's target row (a.lout in
// targets mode, the plan's scratch otherwise); bins flagged by R23 are then re-decided in fp64 from
// the direct Eq. 8 sum, one warp per bin, before the squeeze reads the row.
template <int MODE>
__global__ void __launch_bounds__(kBinThreads) mp_bins_kernel(const FwdArgs a, const float2* Zall, int ch) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    long long* acc = reinterpret_cast<long long*>(smem_raw);          // [ch][2] (re, im)
    __shared__ float red[kBinThreads / 32];
    const int64_t fi = blockIdx.x;                                     // frame within the launch
    const int N = a.nfft, K = N / 2 + 1;
    const float2* Z = Zall + fi * N;
    float gam4 = a.gamma2x4;
    if (a.absmax_dev) {
        const float gm = a.gamma_rel * __ldg(a.absmax_dev);
        gam4 = 4.0f * gm * gm;
    }
    // frame sample j = x[(frame_begin + fi) H - c + j], zero outside the record / slice
    const int64_t s0 = (a.frame_begin + fi) * a.hop - a.c;
    const int64_t v_lo = a.x_off > 0 ? a.x_off : 0;
    const int64_t v_hi = a.n < a.x_off + a.x_len ? a.n : a.x_off + a.x_len;
    auto xat = [&](int j) -> float {
        const int64_t sj = s0 + j;
        return (sj >= v_lo && sj < v_hi) ? __ldg(a.x + (sj - a.x_off)) : 0.0f;
    };
    if constexpr (MODE == kModeStft || MODE == kModeAbsmax) {
        float vmax = 0.0f;
        for (int k = threadIdx.x; k < K; k += kBinThreads) {
            float2 PQ, UV;
            float mag4;
            bool unsure;
            bin_target<false>(a, gam4, 0.0f, -1.0f, k, Z[k], Z[(N - k) & (N - 1)], PQ, UV, mag4, unsure);
            if constexpr (MODE == kModeStft) {
                a.S[fi * K + k] = make_float2(0.5f * PQ.x, 0.5f * PQ.y);
                a.Sd[fi * K + k] = make_float2(UV.x * a.inv_alpha2, -UV.y * a.inv_alpha2);
            } else {
                vmax = fmaxf(vmax, mag4);
            }
        }
        if constexpr (MODE == kModeAbsmax) {
            const float m = block_max(vmax, red);
            if (threadIdx.x == 0) atomicMax(reinterpret_cast<unsigned int*>(a.absmax_out), __float_as_uint(0.5f * sqrtf(m)));
        }
        return;
    } else {
        int32_t* lrow = (MODE == kModeTargets ? a.lout : a.lscratch) + fi * K;
        // R23 margins from ||z_m||^2 = sum_j x_j^2 (g_j^2 + alpha^2 g'_j^2)
        float e = 0.0f;
        for (int j = threadIdx.x; j < a.L; j += kBinThreads) {
            const float xv = xat(j);
            const float2 w = __ldg(a.taps + j);
            e = fmaf(xv * xv, fmaf(w.x, w.x, w.y * w.y), e);
        }
        const float nrm2 = block_sum(e, red);
        float cm, km;
        fwd_margins(a, gam4, nrm2, cm, km);
        for (int k = threadIdx.x; k < K; k += kBinThreads) {
            float2 PQ, UV;
            float mag4;
            bool unsure;
            const int l = bin_target<false>(a, gam4, cm, km, k, Z[k], Z[(N - k) & (N - 1)], PQ, UV, mag4, unsure);
            SST_CHECK(k < K);
            lrow[k] = unsure ? -4 : l;                                 // -4: pending fp64 decision
        }
        __syncthreads();
        {
            // pending bins, one at a time with the whole CTA: warp w sums part w of the taps in fp64
            // (stft_bin_fp64_part's fixed decomposition), the parts are added in warp order, so the
            // decision does not depend on scheduling.  A bin's sum is L / (32 NW) steps deep per
            // lane instead of L / 32 on one warp while the other warps wait at the next barrier.
            constexpr int NW = kBinThreads / 32;
            __shared__ int plist[kBinThreads];
            __shared__ int pcount;
            __shared__ double4 ppart[NW];
            const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
            const double gam64 = launch_gamma64(a);
            auto tap64 = [&](int j) { return __ldg(a.taps64 + j); };
            for (int c0 = 0; c0 < K; c0 += kBinThreads) {
                const int k = c0 + threadIdx.x;
                const bool pend = k < K && lrow[k] == -4;
                if (threadIdx.x == 0) pcount = 0;
                __syncthreads();
                if (pend) plist[atomicAdd(&pcount, 1)] = k;
                const int np = __syncthreads_count(pend);
                for (int i = 0; i < np; ++i) {
                    const int kk = plist[i];
                    const double4 pr = stft_bin_fp64_part(xat, tap64, a.tw64, N, a.L, a.c, kk, warp, NW);
                    if (lane == 0) ppart[warp] = pr;
                    __syncthreads();
                    if (threadIdx.x == 0) {
                        double sr = 0.0, si = 0.0, dr = 0.0, di = 0.0;
                        for (int w = 0; w < NW; ++w) {
                            sr += ppart[w].x;
                            si += ppart[w].y;
                            dr += ppart[w].z;
                            di += ppart[w].w;
                        }
                        lrow[kk] = decide_fp64(a, gam64, kk, sr, si, dr, di);
                        atomicAdd(a.r23_count, 1ull);
                    }
                    __syncthreads();
                }
            }
        }
        if constexpr (MODE == kModeForward) {
            __syncthreads();
            // a6: exact fixed-point sums.  v_max < 2^ex bounds the kept |Re S|, |Im S| of the frame;
            // each value is scaled by 2^(39 - ex) and rounded to an int64 (|X| < 2^39); at most
            // N_f/2 + 1 <= 2^15 + 1 terms per target keep every sum below 2^55, so the integer sums
            // are exact in any order and the band row is bitwise reproducible.
            auto S_of = [&](int k) {                                    // S = (Z[k] + conj Z[N-k]) / 2
                const float2 za = Z[k], zb = Z[(N - k) & (N - 1)];
                return make_float2(0.5f * (za.x + zb.x), 0.5f * (za.y - zb.y));
            };
            float vmax = 0.0f;
            for (int k = threadIdx.x; k < K; k += kBinThreads) {
                if (lrow[k] >= 0) {
                    const float2 S = S_of(k);
                    vmax = fmaxf(vmax, fmaxf(fabsf(S.x), fabsf(S.y)));
                }
            }
            const float m = block_max(vmax, red);
            const int ex = max(-87, (int)((__float_as_uint(m) >> 23) & 0xff) - 126);
            const float scale = __uint_as_float((unsigned)(127 + 39 - ex) << 23);
            const float iscale = __uint_as_float((unsigned)(127 - 39 + ex) << 23);
            float2* trow = a.T + fi * a.ldT;
            for (int l0 = 0; l0 < a.bins; l0 += ch) {
                const int lc = min(ch, a.bins - l0);
                for (int i = threadIdx.x; i < 2 * lc; i += kBinThreads) acc[i] = 0;
                __syncthreads();
                for (int k = threadIdx.x; k < K; k += kBinThreads) {
                    const int lr = lrow[k] - l0;
                    if (lr >= 0 && lr < lc) {                               // -1/-2 give lr < 0 for l0 = 0
                        SST_CHECK(2 * lr + 1 < 2 * ch);
                        const float2 S = S_of(k);
                        long long xr, xi;
                        asm volatile("cvt.rni.s64.f32 %0, %1;" : "=l"(xr) : "f"(S.x * scale));
                        asm volatile("cvt.rni.s64.f32 %0, %1;" : "=l"(xi) : "f"(S.y * scale));
                        atomicAdd(reinterpret_cast<unsigned long long*>(acc + 2 * lr), (unsigned long long)xr);
                        atomicAdd(reinterpret_cast<unsigned long long*>(acc + 2 * lr + 1), (unsigned long long)xi);
                    }
                }
                __syncthreads();
                for (int i = threadIdx.x; i < lc; i += kBinThreads)
                    trow[l0 + i] = make_float2(__ll2float_rn(acc[2 * i]) * iscale, __ll2float_rn(acc[2 * i + 1]) * iscale);
                __syncthreads();
            }
        }
    }
}

// a9 tail: combine the residues of each frame pair, window by g[tau + c]/N_f, write frames A, B
__global__ void __launch_bounds__(256) mp_combine_kernel(const MpInvArgs a, const float2* Y) {
    const int64_t pair = blockIdx.x;
    const int j = blockIdx.y * 256 + threadIdx.x;                      // tau + c
    if (j >= a.L) return;
    const int N = a.nfft, z = a.zoom;
    const int tau = j - a.c;
    const int p = tau >= 0 ? tau : tau + N;
    const int64_t zN = (int64_t)z * N;
    float2 v = make_float2(0.0f, 0.0f);
    for (int b = 0; b < z; ++b) {
        float2 yb = Y[(pair * z + b) * N + p];
        if (b) {
            int64_t e = ((int64_t)b * tau) % zN;
            if (e < 0) e += zN;
            double sn, cs;
            sincospi(2.0 * (double)e / (double)zN, &sn, &cs);         // e^{i 2 pi b tau/(z N)}
            yb = c_mul(yb, make_float2((float)cs, (float)sn));
        }
        v.x += yb.x;
        v.y += yb.y;
    }
    const float w = __ldg(&a.taps[j].x) * a.inv_n;
    const int64_t fA = 2 * pair;
    a.wf[fA * a.L + j] = w * v.x;
    if (fA + 1 < a.frame_end - a.frame_begin) a.wf[(fA + 1) * a.L + j] = w * v.y;
}

// a9 as a direct band sum (narrow bands, large z): per frame and tau,
//   r~[tau] = (2/N_f) Re sum_l w_l T[l] e(j_l tau),  j_l = z k1 + l,  e(x) = exp(2 pi i x/(z N_f)),
// which is the z N_f-point IDFT of the conjugate-mirrored band (Eq. 25, R14: w = 1/2 with
// the imaginary part dropped at j = 0 and j = z N_f/2), windowed by g[tau + c].  Blocked Horner in
// w = e(tau) over 32 bins, blocks joined by phasors e(32 lb tau) whose arguments are reduced
// exactly in integers (no accumulated phase error beyond one 32-term block).
__global__ void __launch_bounds__(256) mp_direct_kernel(const MpInvArgs a) {
    extern __shared__ __align__(16) float2 trow[];                     // [B]
    const int64_t f = blockIdx.x;
    const int B = a.bins;
    const int64_t zN = (int64_t)a.zoom * a.nfft;
    const int64_t j0 = (int64_t)a.zoom * a.k1;
    const int zc = a.zone_path ? __ldg(a.zone_path + f) : 0;
    for (int l = threadIdx.x; l < B; l += 256) {
        float2 t = a.T[f * a.ldT + l];
        if (a.zone_path && ((abs(l - zc) <= a.zone_half) != (bool)a.zone_keep)) t = make_float2(0.0f, 0.0f);
        if (j0 + l == 0 || 2 * (j0 + l) == zN) t = make_float2(0.5f * t.x, 0.0f);
        trow[l] = t;
    }
    __syncthreads();
    const int jj = blockIdx.y * 256 + threadIdx.x;                    // tau + c
    if (jj >= a.L) return;
    const int64_t tau = jj - a.c;
    const float izN = 1.0f / (float)zN;
    auto e_of = [&](int64_t r) {                                        // e(r), 0 <= r < z N (exact in fp32)
        float sn, cs;
        sincospif(2.0f * (float)r * izN, &sn, &cs);
        return make_float2(cs, sn);
    };
    auto red = [&](int64_t x) { int64_t r = x % zN; return r < 0 ? r + zN : r; };
    const float2 w = e_of(red(tau));
    const float2 wi = make_float2(-w.y, w.x);                           // i w: h w + t as two packed FMAs
    const int64_t step = red(32 * tau);
    int64_t rb = 0;                                                     // 32 lb tau mod z N
    float2 acc = make_float2(0.0f, 0.0f);
    for (int l0 = 0; l0 < B; l0 += 32) {
        const int n = min(32, B - l0);
        float2 h = trow[l0 + n - 1];
        if (n == 32) {
#pragma unroll
            for (int ll = 30; ll >= 0; --ll) {
                const float2 t = trow[l0 + ll];
                h = __ffma2_rn(make_float2(h.x, h.x), w, __ffma2_rn(make_float2(h.y, h.y), wi, t));
            }
        } else {
            for (int ll = n - 2; ll >= 0; --ll) {
                const float2 t = trow[l0 + ll];
                h = __ffma2_rn(make_float2(h.x, h.x), w, __ffma2_rn(make_float2(h.y, h.y), wi, t));
            }
        }
        const float2 ph = e_of(rb);
        acc.x = fmaf(h.x, ph.x, fmaf(-h.y, ph.y, acc.x));
        acc.y = fmaf(h.x, ph.y, fmaf(h.y, ph.x, acc.y));
        rb += step;
        rb -= (rb >= zN) ? zN : 0;
    }
    const float2 base = e_of(red(j0 * tau));
    const float re = acc.x * base.x - acc.y * base.y;
    a.wf[f * a.L + jj] = 2.0f * __ldg(&a.taps[jj].x) * a.inv_n * re;
}

// a10: y[s] += sum over the chunk's frames m covering s of wf[m][s - m H + c] (ascending m)
__global__ void __launch_bounds__(256) mp_ola_kernel(const MpInvArgs a, int64_t lo, int64_t hi) {
    const int64_t s = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= hi) return;
    const int64_t H = a.hop, fb = a.frame_begin;
    const int64_t num = s + a.c - a.L + 1;                              // m >= num / H
    int64_t m_lo = num <= 0 ? 0 : (num + H - 1) / H;
    if (m_lo < fb) m_lo = fb;
    int64_t m_hi = (s + a.c) / H;
    if (m_hi > a.frame_end - 1) m_hi = a.frame_end - 1;
    float acc = 0.0f;
    for (int64_t m = m_lo; m <= m_hi; ++m) acc += a.wf[(m - fb) * a.L + (s - m * H + a.c)];
    SST_CHECK(s - a.y_off >= 0 && s - a.y_off < a.y_len);
    a.y[s - a.y_off] += acc;
}

}  // namespace

void mp_factor(int nfft, int* r1, int* m) {
    int lg = 0;
    while ((1 << lg) < nfft) ++lg;
    *r1 = 1 << ((lg + 1) / 2);
    *m = nfft / *r1;
}

int mp_bins_chunk(int bins) { return bins < kMpBinChunk ? bins : kMpBinChunk; }

cudaError_t launch_mp_forward(const FwdArgs& f, int mode, const float2* twN, float2* buf0, float2* buf1,
                              cudaStream_t s) {
    MpPass p{};
    const int64_t nfr = f.frame_end - f.frame_begin;
    if (nfr <= 0) return cudaSuccess;
    p.count = nfr;
    p.N = f.nfft;
    mp_factor(f.nfft, &p.R1, &p.M);
    p.twN = twN;
    p.x = f.x;
    p.x_off = f.x_off;
    p.v_lo = f.x_off > 0 ? f.x_off : 0;
    p.v_hi = f.n < f.x_off + f.x_len ? f.n : f.x_off + f.x_len;
    p.frame0 = f.frame_begin;
    p.hop = f.hop;
    p.L = f.L;
    p.c = f.c;
    p.taps = f.taps;
    cudaError_t e;
    if ((e = run_fft<kLoadFwd, -1>(p, buf0, buf1, s)) != cudaSuccess) return e;
    const int ch = mp_bins_chunk(f.bins);
    switch (mode) {
        case kModeForward: {
            const size_t smem = (size_t)ch * 16;
            auto k = mp_bins_kernel<kModeForward>;
            if ((e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess) return e;
            k<<<(unsigned)nfr, kBinThreads, smem, s>>>(f, buf1, ch);
            break;
        }
        case kModeStft: mp_bins_kernel<kModeStft><<<(unsigned)nfr, kBinThreads, 0, s>>>(f, buf1, ch); break;
        case kModeTargets: mp_bins_kernel<kModeTargets><<<(unsigned)nfr, kBinThreads, 0, s>>>(f, buf1, ch); break;
        case kModeAbsmax: mp_bins_kernel<kModeAbsmax><<<(unsigned)nfr, kBinThreads, 0, s>>>(f, buf1, ch); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_mp_inverse_accumulate(const MpInvArgs& a, cudaStream_t s) {
    const int64_t nfr = a.frame_end - a.frame_begin;
    if (nfr <= 0) return cudaSuccess;
    cudaError_t e;
    if (a.direct) {
        mp_direct_kernel<<<dim3((unsigned)nfr, (unsigned)((a.L + 255) / 256)), 256, (size_t)a.bins * 8, s>>>(a);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    } else {
    const int64_t pairs = (nfr + 1) / 2;
    MpPass p{};
    p.count = pairs * a.zoom;
    p.N = a.nfft;
    mp_factor(a.nfft, &p.R1, &p.M);
    p.twN = a.twN;
    p.T = a.T;
    p.ldT = a.ldT;
    p.nfr = nfr;
    p.zoom = a.zoom;
    p.k1 = a.k1;
    p.bins = a.bins;
    p.zone_path = a.zone_path;
    p.zone_half = a.zone_half;
    p.zone_keep = a.zone_keep;
    if ((e = run_fft<kLoadInv, +1>(p, a.buf0, a.buf1, s)) != cudaSuccess) return e;
    mp_combine_kernel<<<dim3((unsigned)pairs, (unsigned)((a.L + 255) / 256)), 256, 0, s>>>(a, a.buf1);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    const int64_t lo = a.frame_begin * a.hop - a.c > 0 ? a.frame_begin * a.hop - a.c : 0;
    int64_t hi = (a.frame_end - 1) * a.hop - a.c + a.L;
    if (hi > a.n) hi = a.n;
    if (hi > lo) mp_ola_kernel<<<(unsigned)((hi - lo + 255) / 256), 256, 0, s>>>(a, lo, hi);
    return cudaGetLastError();
}

}  // namespace sst
