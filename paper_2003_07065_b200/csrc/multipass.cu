// Large-N_f path (8192 < N_f <= 65536; the paper's §5.2 uses N_f = 2^15).
//
// A frame's packed buffer (N_f complex64 = 256 KiB at 2^15) no longer fits one CTA's shared
// memory next to anything else, so the transform runs as a multi-pass four-step FFT through HBM
// (the scratch of a chunk of frames stays mostly L2-resident):
//   N_f = R1 M.  Pass 1: for every column a in [0, M) a P = R1-point DFT of x[a + M i], times
//   W_N^{a k1}, stored at [k1][a].  Pass 2: for every row k1 a P = M-point DFT over a, stored at
//   k1 + R1 k2 (natural order).  Each CTA owns 16 adjacent columns / rows, so every global load
//   and store moves 128-byte segments, and runs a radix-4 Stockham (autosort) FFT over them in
//   shared memory with twiddles rounded once from fp64 (the plan's W_N table).
// Forward: pass 1 gathers and packs the frame on the fly (a1: z[n] = u (g + i alpha g'), circular
// placement, as in the fused kernel), pass 2 writes the spectrum, and one CTA per frame then does
// a3-a7 with the fused path's own per-bin decision (decide.cuh) and an exact 64-bit fixed-point
// squeeze in shared memory (order-independent, so bitwise reproducible).
// Inverse: per frame pair and residue b the Hermitian-packed sub-spectrum G_b (the fused
// inverse's split of the z N_f IDFT) is gathered from T in pass 1, transformed by
// passes 1-2 (conjugate twiddles), combined over b with e^{i 2 pi b tau/(z N)}, windowed by
// g[tau + c]/N_f (a9), and overlap-added by a gather kernel (one thread per output sample,
// frames in ascending order: no atomics, deterministic) (a10, Eq. 26).  For narrow bands with a
// large z (B L small against z N_f log N_f, e.g. the §5.2 Fig. 16(e) shape, z = 20) the plan
// picks a direct band sum per frame instead (mp_direct_kernel), with the same windowing and OLA.
#include <cuda_runtime.h>
#include <stdint.h>

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
    // Stockham (autosort) FFT over the 16 columns: radix-4 stages, then one radix-2 stage when
    // log2 P is odd.  Radix 4 at length n = P/s: for p < m = n/4, q < s, with A..D = x[q + s(p + j m)],
    //   y[q + s(4p + k)] = X_k W_n^{p k},  X = the 4-point DFT of (A, B, C, D)
    float2* x = s0;
    float2* y = s1;
    const int tstep = a.N / P;
    int s = 1, ls = 0;
#pragma unroll 1
    for (; 4 * s <= P; s <<= 2, ls += 2) {
        const int m = P / (4 * s);
        for (int bf = tid; bf < kTile * P / 4; bf += kPassThreads) {
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
            y[o0 + os] = c_mul(make_float2(amc.x + jb.x, amc.y + jb.y), tw_at<DIR>(a.twN, e));
            y[o0 + 2 * os] = c_mul(make_float2(apc.x - bpd.x, apc.y - bpd.y), tw_at<DIR>(a.twN, 2 * e));
            y[o0 + 3 * os] = c_mul(make_float2(amc.x - jb.x, amc.y - jb.y), tw_at<DIR>(a.twN, 3 * e));
        }
        __syncthreads();
        float2* tmp = x; x = y; y = tmp;
    }
    if (s < P) {                                                        // last radix-2 stage (n = 2)
        for (int bf = tid; bf < kTile * P / 2; bf += kPassThreads) {
            const int al = bf & 15, q = bf >> 4;
            const float2 u = x[q * kTS + al], v = x[(q + s) * kTS + al];
            y[q * kTS + al] = make_float2(u.x + v.x, u.y + v.y);
            y[(q + s) * kTS + al] = make_float2(u.x - v.x, u.y - v.y);
        }
        __syncthreads();
        float2* tmp = x; x = y; y = tmp;
    }
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
            const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
            const double gam64 = launch_gamma64(a);
            for (int b0 = warp * 32; b0 < K; b0 += kBinThreads) {
                const int k0 = b0 + lane;
                unsigned ball = __ballot_sync(0xffffffffu, k0 < K && lrow[k0] == -4);
                while (ball) {
                    const int k = b0 + __ffs(ball) - 1;
                    ball &= ball - 1;
                    double sr, si, dr, di;
                    stft_bin_fp64(xat, a.taps64, a.tw64, N, a.L, a.c, k, sr, si, dr, di);
                    const int ln = decide_fp64(a, gam64, k, sr, si, dr, di);
                    __syncwarp();
                    if (lane == 0) {
                        lrow[k] = ln;
                        atomicAdd(a.r23_count, 1ull);
                    }
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
                h = make_float2(fmaf(h.x, w.x, fmaf(-h.y, w.y, t.x)), fmaf(h.x, w.y, fmaf(h.y, w.x, t.y)));
            }
        } else {
            for (int ll = n - 2; ll >= 0; --ll) {
                const float2 t = trow[l0 + ll];
                h = make_float2(fmaf(h.x, w.x, fmaf(-h.y, w.y, t.x)), fmaf(h.x, w.y, fmaf(h.y, w.x, t.y)));
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
    p.out = buf0;
    cudaError_t e = run_pass<kLoadFwd, -1>(p, 1, s);
    if (e != cudaSuccess) return e;
    p.in = buf0;
    p.out = buf1;
    if ((e = run_pass<kLoadBuf, -1>(p, 2, s)) != cudaSuccess) return e;
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
    p.out = a.buf0;
    e = run_pass<kLoadInv, +1>(p, 1, s);
    if (e != cudaSuccess) return e;
    p.in = a.buf0;
    p.out = a.buf1;
    if ((e = run_pass<kLoadBuf, +1>(p, 2, s)) != cudaSuccess) return e;
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
