// Frequency-domain filter-bank STFT for truncated narrow bands (§6:
// "converting the calculation of STFT to filter bank-based in the frequency domain").
//
// With SST_SOURCE_TRUNCATE (R12) only the source bins k in [k1, k2) are reassigned, so only their
// S and S' are needed.  Frames are processed in blocks: block b shares the segment
// x_b[n] = x[n0 + n], n in [0, Ns), n0 = (frame_begin + b Fb) H - c, which holds the Fb frames
// m' = 0..Fb-1 (frame m' reads x_b[m' H + j], j = 0..L-1; (Fb - 1) H + L <= Ns).  Eq. 8
// rewritten with X_b = DFT_Ns(x_b) and Ns = ratio N_f:
//   S[m', k] = sum_j x_b[m' H + j] g[j] e^{-2 pi i k (j - c) / N_f}
//            = e^{2 pi i k c / N_f} / Ns  sum_f X_b[f] Gamma[f - ratio k] e^{2 pi i f m' H / Ns},
//   Gamma[d] = sum_j g[j] e^{2 pi i d j / Ns}   (all Ns values: a window cut at +-4 sigma has
//                                               sidelobes decaying only like 1/d, so no truncation)
// and since e^{2 pi i f m' H / Ns} depends on f only through q = f mod P (P = Ns / H), folding the
// products onto q (Y_k[q] = sum_{r < H} X_b[q + r P] Gamma[q + r P - ratio k], a fixed order) turns each
// (k, window) into one P-point inverse DFT that yields S (or S') for all Fb frames of the block:
// S[., k] = phase_k / Ns * IDFT_P(Y_k)[m'].  Cost per frame ~ 2 K_b H Ns/(Ns - L) complex MACs for the
// folds against ~N_f log2 N_f / 2 butterflies for a per-frame FFT: the plan picks the filter bank only
// where that is smaller (narrow bands at small H).
// fb_transform: one CTA per block: the Ns-point FFT of x_b (in-place radix-2 in shared memory), then
// per (k, window) one warp builds Y_k and runs the P-point inverse FFT in its own buffer; results go
// through a staging tile to the S / S' planes [frame][K_b] (coalesced rows).
// fb_squeeze: one warp per frame: the per-bin decision of the fused path (decide.cuh, same fp32
// arithmetic, R17) on (2 S, 2 alpha S'), R23 flags with the filter bank's own error model, the exact
// fixed-point squeeze (32-bit limbs, bitwise reproducible) and the band row store.  Flagged bins are
// queued for redecide_kernel exactly as on the fused path; changed frames are re-squeezed in list mode
// with inline fp64 re-decision.
#include <cuda_runtime.h>
#include <stdint.h>

#include "decide.cuh"
#include "sst_internal.h"

namespace sst {

namespace {

constexpr int kFbThreads = 256;
constexpr int kFbWarps = kFbThreads / 32;

__device__ __forceinline__ float2 fmulc(float2 a, float2 b) {
    return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}

__device__ __forceinline__ unsigned brev_n(unsigned v, int lg) { return __brev(v) >> (32 - lg); }

}  // namespace

// ------------------------------------------------------------------------------ transform ----
// HH: the fold length H (compile time for the usual 4..64, unrolled; 0: runtime).  GSM: Gamma of the
// current window staged in shared memory (windows then processed one after the other).
template <int HH, bool GSM>
__global__ void __launch_bounds__(kFbThreads, 1) fb_transform_kernel(const FbArgs a) {
    extern __shared__ __align__(16) float2 fsm[];
    float2* X = fsm;                                         // [ns] spectrum of x_b (in place)
    float2* wb = X + a.ns;                                   // [warps][P] inverse-FFT buffers
    float2* stg = wb + kFbWarps * a.P;                       // [fb][kc][2] staging tile
    float2* gsm = stg + (size_t)a.fb * a.kc * 2;             // [ns] Gamma of one window (GSM)
    __shared__ float red[kFbWarps];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t nfr = a.frame_end - a.frame_begin;
    // blocks on the global frame grid (block b = frames [b Fb, b Fb + Fb)): the same blocks whatever
    // frame range a launch covers; only the launch's frames are stored
    const int64_t g0 = (a.frame_begin / a.fb + blockIdx.x) * a.fb;   // first frame of the block (global)
    const int64_t m0 = g0 - a.frame_begin;                   // ... within the launch (may be < 0)
    const int64_t n0 = g0 * a.hop - a.c;
    const int64_t v_lo = a.x_off > 0 ? a.x_off : 0;
    const int64_t v_hi = min(a.n, a.x_off + a.x_len);

    // x_b in bit-reversed order (in-place DIT), and ||x_b||^2 for the R23 error model
    float e2 = 0.0f;
    for (int n = tid; n < a.ns; n += kFbThreads) {
        const int64_t s = n0 + n;
        const float v = (s >= v_lo && s < v_hi) ? __ldg(a.x + (s - a.x_off)) : 0.0f;
        e2 = fmaf(v, v, e2);
        X[brev_n((unsigned)n, a.lg_ns)] = make_float2(v, 0.0f);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) e2 += __shfl_xor_sync(0xffffffffu, e2, o);
    if (lane == 0) red[warp] = e2;
    __syncthreads();
    // forward DFT (e^{-2 pi i f n / Ns}), radix-2 DIT, twiddles rounded from fp64 (twns[e] = W_Ns^e)
    for (int half = 1, st = a.ns >> 1; half < a.ns; half <<= 1, st >>= 1) {
        for (int t = tid; t < a.ns / 2; t += kFbThreads) {
            const int pos = t & (half - 1);
            const int i = ((t - pos) << 1) + pos, j = i + half;
            const float2 w = __ldg(a.twns + pos * st);
            const float2 u = X[i], v = fmulc(X[j], w);
            X[i] = make_float2(u.x + v.x, u.y + v.y);
            X[j] = make_float2(u.x - v.x, u.y - v.y);
        }
        __syncthreads();
    }
    float nrm2 = 0.0f;
#pragma unroll
    for (int w = 0; w < kFbWarps; ++w) nrm2 += red[w];
    const float eta = sqrtf(nrm2);                           // ||x_b||_2 (the plan's constants do the rest)

    float2* buf = wb + warp * a.P;
    const int H = HH ? HH : a.ns / a.P;
    for (int pass = 0; pass < (GSM ? 2 : 1); ++pass) {
    if constexpr (GSM) {
        const float2* src = pass ? a.gamd : a.gam;
        for (int i = tid; i < a.ns; i += kFbThreads) gsm[i] = __ldg(src + i);
        __syncthreads();
    }
    for (int kk0 = 0; kk0 < a.kb; kk0 += a.kc) {
        const int kn = min(a.kc, a.kb - kk0);
        for (int item = warp; item < (GSM ? 1 : 2) * kn; item += kFbWarps) {
            const int kk = kk0 + (GSM ? item : (item >> 1)), win = GSM ? pass : (item & 1);
            const int k = a.kb0 + kk;
            const float2* gam = GSM ? gsm : (win ? a.gamd : a.gam);
            // Y_k[q] = sum_{r < H} X_b[q + r P] Gamma[(q + r P - ratio k) mod Ns], placed in bit-reversed
            // order for the in-place DIT inverse transform
            const int sh = a.ratio * k;
            for (int q = lane; q < a.P; q += 32) {
                float2 acc = make_float2(0.0f, 0.0f);
                if constexpr (HH > 0) {
                    float2 xv[HH], gv[HH];
#pragma unroll
                    for (int r = 0; r < HH; ++r) {                // all loads first, then the fixed-order sum
                        const int f = q + r * a.P;
                        xv[r] = X[f];
                        gv[r] = GSM ? gam[(f - sh) & (a.ns - 1)] : __ldg(gam + ((f - sh) & (a.ns - 1)));
                    }
#pragma unroll
                    for (int r = 0; r < HH; ++r) {
                        acc.x = fmaf(xv[r].x, gv[r].x, fmaf(-xv[r].y, gv[r].y, acc.x));
                        acc.y = fmaf(xv[r].x, gv[r].y, fmaf(xv[r].y, gv[r].x, acc.y));
                    }
                } else {
                    for (int r = 0; r < H; ++r) {
                        const int f = q + r * a.P;
                        const float2 xv = X[f], gv = __ldg(gam + ((f - sh) & (a.ns - 1)));
                        acc.x = fmaf(xv.x, gv.x, fmaf(-xv.y, gv.y, acc.x));
                        acc.y = fmaf(xv.x, gv.y, fmaf(xv.y, gv.x, acc.y));
                    }
                }
                buf[brev_n((unsigned)q, a.lg_P)] = acc;
            }
            __syncwarp();
            // inverse DFT over P (e^{+2 pi i q m / P}), radix-2 DIT
            for (int half = 1, st = a.P >> 1; half < a.P; half <<= 1, st >>= 1) {
                for (int t = lane; t < a.P / 2; t += 32) {
                    const int pos = t & (half - 1);
                    const int i = ((t - pos) << 1) + pos, j = i + half;
                    const float2 w = __ldg(a.twp + pos * st);
                    const float2 u = buf[i], v = fmulc(buf[j], w);
                    buf[i] = make_float2(u.x + v.x, u.y + v.y);
                    buf[j] = make_float2(u.x - v.x, u.y - v.y);
                }
                __syncwarp();
            }
            const float2 ph = __ldg(a.ph + kk);               // e^{2 pi i k c / N_f} / Ns
            for (int m = lane; m < a.fb; m += 32)
                stg[((int64_t)m * a.kc + (kk - kk0)) * 2 + win] = fmulc(buf[m], ph);
            __syncwarp();
        }
        __syncthreads();
        // staging -> planes: row m0 + m, columns kk0 .. kk0 + kn (GSM: the pass's window only)
        for (int idx = tid; idx < a.fb * kn; idx += kFbThreads) {
            const int m = idx / kn, kk = idx - m * kn;
            const int64_t fr = m0 + m;
            if (fr >= 0 && fr < nfr) {
                if (!GSM || pass == 0) a.S[fr * a.kb + kk0 + kk] = stg[((int64_t)m * a.kc + kk) * 2 + 0];
                if (!GSM || pass == 1) a.Sd[fr * a.kb + kk0 + kk] = stg[((int64_t)m * a.kc + kk) * 2 + 1];
            }
        }
        __syncthreads();
    }
    }
    if (a.eta)
        for (int m = tid; m < a.fb; m += kFbThreads)
            if (m0 + m >= 0 && m0 + m < nfr) a.eta[m0 + m] = eta;
}

// ------------------------------------------------------------------------------ squeeze ------
// one warp per frame; list mode (a.flist) processes the listed frames with inline fp64 re-decision
template <int NBMAX>
__global__ void __launch_bounds__(kFbThreads) fb_squeeze_kernel(const FbArgs fb, const FwdArgs a) {
    extern __shared__ __align__(16) int lsm[];
    __shared__ unsigned cq_n;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int B = a.bins;
    int* acc = lsm + warp * 4 * B;                            // planar [hi_re | lo_re | hi_im | lo_im][B]
    const int64_t nfr = a.frame_end - a.frame_begin;
    const bool lmode = a.flist != nullptr;
    const int64_t nitems = lmode ? (int64_t)*a.flist_n : nfr;
    const int64_t K = a.nfft / 2 + 1;
    (void)K;
    float gam4 = a.gamma2x4;
    if (a.absmax_dev) {
        const float gm = a.gamma_rel * __ldg(a.absmax_dev);
        gam4 = 4.0f * gm * gm;
    }
    const double gam64 = launch_gamma64(a);
    const float alpha2 = 2.0f * fb.alpha;
    if (threadIdx.x == 0) cq_n = 0;
    for (int i = lane; i < 4 * B; i += 32) acc[i] = 0;
    __syncthreads();
    const int64_t v_lo = a.x_off > 0 ? a.x_off : 0;
    const int64_t v_hi = min(a.n, a.x_off + a.x_len);
    const int nb = (fb.kb + 31) / 32;                         // source bins per lane (<= NBMAX)

    for (int64_t it = (int64_t)blockIdx.x * kFbWarps + warp; it < nitems; it += (int64_t)gridDim.x * kFbWarps) {
        const int64_t fi = lmode ? (int64_t)__ldg(a.flist + it) : it;
        // per-frame margins (R23): eta = ||x_b||_2 of the frame's block
        const float eta = __ldg(fb.eta + fi);
        float cm = fb.cflag * eta, km = -1.0f;
        {
            const float kd = fb.kflag * eta;
            km = 4.0f * kd * fmaf(2.0f, 0.5f * sqrtf(fmaxf(gam4, 0.0f)), kd);
            if (!a.redecide) { cm = 0.0f; km = -1.0f; }
        }
        int bl[NBMAX];
        float br[NBMAX], bi[NBMAX];
        unsigned uns = 0u;
        float vmax = 0.0f;
#pragma unroll
        for (int j = 0; j < NBMAX; ++j) {
            bl[j] = -3;
            br[j] = bi[j] = 0.0f;
            if (j < nb) {
                const int kk = lane + 32 * j;
                const bool ok = kk < fb.kb;
                const float2 S = ok ? __ldg(fb.S + fi * fb.kb + kk) : make_float2(0.0f, 0.0f);
                const float2 Sd = ok ? __ldg(fb.Sd + fi * fb.kb + kk) : make_float2(0.0f, 0.0f);
                const float2 PQ = make_float2(2.0f * S.x, 2.0f * S.y);
                const float2 UV = make_float2(alpha2 * Sd.x, -alpha2 * Sd.y);
                float mag4;
                bool unsure;
                int l = bin_target_pq<true>(a, gam4, cm, km, fb.kb0 + kk, PQ, UV, mag4, unsure);
                if (!ok) { l = -3; unsure = false; }
                bl[j] = l;
                br[j] = S.x;
                bi[j] = S.y;
                if (unsure) uns |= 1u << j;
            }
        }
        // R23: deferred (queue) in the normal launch, inline in list mode / when the queue is full
        unsigned my = uns;
        if (a.gq && my) {
            const unsigned reg = a.gq_cap / gridDim.x;
            int4* cq = a.gq + (size_t)blockIdx.x * reg;
            while (my) {
                const int j = __ffs(my) - 1;
                int lj = 0;
#pragma unroll
                for (int jj = 0; jj < NBMAX; ++jj) lj = (jj == j) ? bl[jj] : lj;
                const unsigned q = atomicAdd(&cq_n, 1u);
                if (q >= reg) break;
                cq[q] = make_int4((int)fi, fb.kb0 + lane + 32 * j, lj, 0);
                my &= my - 1;
            }
        }
        while (true) {
            const unsigned ball = __ballot_sync(0xffffffffu, my != 0u);
            if (!ball) break;
            const int src = __ffs(ball) - 1;
            const int j = __ffs(__shfl_sync(0xffffffffu, my, src)) - 1;
            if (lane == src) my &= my - 1;
            const int k = fb.kb0 + src + 32 * j;
            const int64_t s0 = (a.frame_begin + fi) * a.hop - a.c;
            double sr, si, dr, di;
            stft_bin_fp64([&](int jj) -> float {
                const int64_t sj = s0 + jj;
                return (sj >= v_lo && sj < v_hi) ? __ldg(a.x + (sj - a.x_off)) : 0.0f;
            }, a.taps64, a.tw64, a.nfft, a.L, a.c, k, sr, si, dr, di);
            const int ln = decide_fp64(a, gam64, k, sr, si, dr, di);
            if (lane == 0 && !lmode) atomicAdd(a.r23_count, 1ull);
#pragma unroll
            for (int jj = 0; jj < NBMAX; ++jj)
                if (lane == src && jj == j) {
                    if (bl[jj] != ln && !lmode) atomicAdd(a.r23_count + 1, 1ull);
                    bl[jj] = ln;
                }
        }
        // a6: exact fixed-point sums (as the fused kernel): scale 2^(39 - ex), v_max < 2^ex over the kept
        // values of the frame; 32-bit limbs, at most K_b <= 1024 terms per target
#pragma unroll
        for (int j = 0; j < NBMAX; ++j)
            if (j < nb && bl[j] >= 0) vmax = fmaxf(vmax, fmaxf(fabsf(br[j]), fabsf(bi[j])));
        const unsigned vb = __reduce_max_sync(0xffffffffu, __float_as_uint(vmax));
        const int ex = max(-87, (int)((vb >> 23) & 0xff) - 126);
        const float scale = __uint_as_float((unsigned)(127 + 39 - ex) << 23);
        const float iscale = __uint_as_float((unsigned)(127 - 39 + ex) << 23);
#pragma unroll
        for (int j = 0; j < NBMAX; ++j) {
            if (j >= nb) break;
            const int l = bl[j];
            if (l >= 0) {
                SST_CHECK(l < B);
                long long xr, xi;
                asm volatile("cvt.rni.s64.f32 %0, %1;" : "=l"(xr) : "f"(br[j] * scale));
                asm volatile("cvt.rni.s64.f32 %0, %1;" : "=l"(xi) : "f"(bi[j] * scale));
                atomicAdd(acc + l, (int)(xr >> 20));
                atomicAdd(acc + B + l, (int)(xr & 0xFFFFF));
                atomicAdd(acc + 2 * B + l, (int)(xi >> 20));
                atomicAdd(acc + 3 * B + l, (int)(xi & 0xFFFFF));
            }
        }
        __syncwarp();
        float2* trow = a.T + fi * a.ldT;
        for (int l = lane; l < B; l += 32) {
            const float2 t = make_float2(limbs_to_float(acc[l], acc[B + l], iscale),
                                         limbs_to_float(acc[2 * B + l], acc[3 * B + l], iscale));
            acc[l] = acc[B + l] = acc[2 * B + l] = acc[3 * B + l] = 0;   // clear on read
            __stcs(trow + l, t);
        }
        __syncwarp();
    }
    if (a.gq) {
        __syncthreads();
        if (threadIdx.x == 0) a.gq_counts[blockIdx.x] = min(cq_n, a.gq_cap / gridDim.x);
    }
}

// ------------------------------------------------------------------------------ launchers ----
int fb_transform_smem(const FbArgs& a) { return (a.ns + kFbWarps * a.P + a.fb * a.kc * 2) * (int)sizeof(float2); }

template <int HH>
static cudaError_t launch_fbt(const FbArgs& a, unsigned blocks, cudaStream_t s) {
    const int base = fb_transform_smem(a);
    const bool gsm = base + a.ns * (int)sizeof(float2) <= 227 * 1024;
    const int smem = base + (gsm ? a.ns * (int)sizeof(float2) : 0);
    auto kern = gsm ? fb_transform_kernel<HH, true> : fb_transform_kernel<HH, false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    kern<<<blocks, kFbThreads, smem, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_fb_transform(const FbArgs& a, cudaStream_t s) {
    const int64_t nfr = a.frame_end - a.frame_begin;
    if (nfr <= 0) return cudaSuccess;
    const unsigned blocks = (unsigned)((a.frame_end - 1) / a.fb - a.frame_begin / a.fb + 1);
    switch (a.ns / a.P) {
        case 4: return launch_fbt<4>(a, blocks, s);
        case 8: return launch_fbt<8>(a, blocks, s);
        case 16: return launch_fbt<16>(a, blocks, s);
        case 32: return launch_fbt<32>(a, blocks, s);
        default: return launch_fbt<0>(a, blocks, s);
    }
}

int fb_squeeze_grid(int device) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    return 2 * sms;
}

template <int NBMAX>
static cudaError_t launch_fbs(const FbArgs& fb, const FwdArgs& a, int grid, cudaStream_t s) {
    const int smem = kFbWarps * 4 * a.bins * (int)sizeof(int);
    cudaError_t e = cudaFuncSetAttribute(fb_squeeze_kernel<NBMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    fb_squeeze_kernel<NBMAX><<<grid, kFbThreads, smem, s>>>(fb, a);
    return cudaGetLastError();
}

cudaError_t launch_fb_squeeze(const FbArgs& fb, const FwdArgs& a, int grid, cudaStream_t s) {
    const int nb = (fb.kb + 31) / 32;
    if (nb <= 2) return launch_fbs<2>(fb, a, grid, s);
    if (nb <= 4) return launch_fbs<4>(fb, a, grid, s);
    if (nb <= 8) return launch_fbs<8>(fb, a, grid, s);
    if (nb <= 16) return launch_fbs<16>(fb, a, grid, s);
    return launch_fbs<32>(fb, a, grid, s);
}

}  // namespace sst
