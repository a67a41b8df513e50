// sm_100a kernels of the fast downsampled SST (He & Cao, arXiv 2003.07065).
//
// Forward (one fused persistent kernel, rows a1-a7 of DESIGN.md §1):
//   frame m, packed buffer z[n] = x[m H + tau] (g[tau+c] + i alpha g'[tau+c]), n = tau mod N_f
//   (circular placement == Eq. 9's phase factor e^{i 2 pi k M/N_f});
//   N_f = 64 * N2 four-step FFT: N2 threads per frame, each thread a 64-point register DFT of
//   the decimated row n2 = thread, twiddle W_N^{n2 k1}, one padded shared-memory exchange,
//   then N2-point register DFTs of columns.  Columns are assigned in conjugate pairs
//   (k1, 64-k1) so that Z[k] and Z[N-k] meet in one thread (N2 <= 32), which makes the
//   unpack S = (Z[k] + conj Z[N-k])/2, S' = (Z[k] - conj Z[N-k])/(2 i alpha) register-only.
//   Per source bin: mask |S| > gamma (Eq. 13), r = -Im(S'/S) N/(2 pi) (Eq. 36), target
//   l = z(k-k1) + floor(z r + 1/2) (Eq. 28, R17), shared-memory atomics into the frame's band
//   accumulator (Eq. 27/28), coalesced store of the band row.
//
// Inverse (rows a9-a11): two frames per complex IFFT (Hermitian packing), the z N_f-point
//   band IDFT of P:L222 split into z N_f-point sub-transforms by residue b = j mod z, outer
//   phase e^{i 2 pi b tau/(z N)}, real/imag -> the two frames, x g[tau+c] / N_f, OLA in a
//   shared-memory ring per CTA (Eq. 26); samples shared with the neighbouring CTA go to a
//   seam buffer combined by a second tiny kernel.
#include <cuda_runtime.h>
#include <stdint.h>

#include "fft.cuh"
#include "sst_internal.h"

namespace sst {

cudaError_t upload_w64(const float2* w64_host) {
    return cudaMemcpyToSymbol(c_w64, w64_host, sizeof(float2) * 64);
}

template <int N2>
struct Geom {
    static constexpr int N = 64 * N2;
    static constexpr int G = kCtaThreads / N2;   // frames (forward) / frame pairs (inverse) per CTA
    static constexpr int STRIDE = N2 + 1;         // padded exchange row (odd -> conflict-free)
    static constexpr int CAP = 64 * STRIDE;       // float2 per group buffer
};

template <int N2>
__device__ __forceinline__ void group_sync(int group) {
    if constexpr (N2 <= 32) {
        __syncwarp();
    } else {
        asm volatile("bar.sync %0, %1;" ::"r"(1 + group), "r"(N2) : "memory");
    }
}

// ------------------------------------------------------------------------------- forward ------
struct BinCtx {
    float gam4, r_scale;
    int k1, bins, zoom, src_lo, src_hi;
};

// Per source bin k with Za = Z[k], Zb = Z[N-k]: returns target l (>= 0), -1 masked, -2 out of band.
// S = (P, Q)/2 with P = Re Za + Re Zb, Q = Im Za - Im Zb;  S' = (U, -V)/(2 alpha) with
// U = Im Za + Im Zb, V = Re Za - Re Zb;  -Im(S'/S) = (V P + U Q) / (alpha (P^2 + Q^2)).
__device__ __forceinline__ int bin_target(const BinCtx& b, int k, float2 za, float2 zb, float& P, float& Q,
                                          float& U, float& V, float& mag4) {
    P = za.x + zb.x;
    Q = za.y - zb.y;
    U = za.y + zb.y;
    V = za.x - zb.x;
    mag4 = fmaf(P, P, Q * Q);                       // 4 |S|^2
    if (!(mag4 > b.gam4) || k < b.src_lo || k >= b.src_hi) return -1;
    const float r = (fmaf(V, P, U * Q) / mag4) * b.r_scale;   // RF in coarse bins (Eq. 36)
    const float zr = (float)b.zoom * r;
    if (!(fabsf(zr) <= 1073741824.0f)) return -2;   // non-finite or huge (R17)
    int l;
    if (r >= -(float)k) l = b.zoom * (k - b.k1) + (int)floorf(zr + 0.5f);
    else                l = -b.zoom * (k + b.k1) + (int)floorf(0.5f - zr);   // |k + r| = -(k + r) (Eq. 13 abs)
    return (l >= 0 && l < b.bins) ? l : -2;
}

// BIG: the band row (B bins) does not fit the group's exchange buffer (B > CAP): bins are kept
// in registers and squeezed in chunks of CAP.  Otherwise (N2 <= 32) all column data is read
// into registers first and the exchange buffer is reused as the band accumulator.
template <int N2, int MODE, bool BIG>
__global__ void __launch_bounds__(kCtaThreads, (N2 <= 32 ? 3 : 2)) fwd_kernel(const FwdArgs a) {
    using Gm = Geom<N2>;
    constexpr int N = Gm::N;
    constexpr int STRIDE = Gm::STRIDE;
    constexpr int CAP = Gm::CAP;
    constexpr int G = Gm::G;
    constexpr int NB = 33;                         // source bins per thread (+1 Nyquist slot)
    extern __shared__ float2 smem[];
    const int group = threadIdx.x / N2;
    const int tg = threadIdx.x % N2;
    float2* buf = smem + group * CAP;

    BinCtx bc;
    if (a.absmax_dev) {
        const float gm = a.gamma_rel * __ldg(a.absmax_dev);
        bc.gam4 = 4.0f * gm * gm;
    } else {
        bc.gam4 = a.gamma2x4;
    }
    bc.r_scale = a.r_scale;
    bc.k1 = a.k1; bc.bins = a.bins; bc.zoom = a.zoom; bc.src_lo = a.src_lo; bc.src_hi = a.src_hi;

    const int64_t nfr = a.frame_end - a.frame_begin;
    const int64_t ntiles = (nfr + G - 1) / G;
    const int64_t tiles_per_cta = (ntiles + gridDim.x - 1) / gridDim.x;
    const int64_t t_begin = (int64_t)blockIdx.x * tiles_per_cta;
    const int64_t t_end = min(ntiles, t_begin + tiles_per_cta);
    const int last_in = a.L - 1 - a.c;             // largest tau
    float vmax = 0.0f;

    for (int64_t tile = t_begin; tile < t_end; ++tile) {
        const int64_t fi = tile * G + group;       // frame index within the launch
        const bool valid = fi < nfr;
        const int64_t sbase = (a.frame_begin + fi) * a.hop - a.x_off;   // x index of tau = 0

        // ---- a1: gather + pack (circular placement), a2 step 1: 64-point DFT of row tg
        float2 v[64];
#pragma unroll
        for (int n1 = 0; n1 < 64; ++n1) {
            const int n = N2 * n1 + tg;
            const int tau = (n <= last_in) ? n : n - N;
            float2 val = make_float2(0.0f, 0.0f);
            const int64_t s = sbase + tau + a.x_off;             // global sample
            if (valid && tau >= -a.c && s >= 0 && s < a.n) {
                const float xs = __ldg(a.x + (sbase + tau));
                const float2 w = __ldg(a.taps + (tau + a.c));
                val = make_float2(xs * w.x, xs * w.y);
            }
            v[n1] = val;
        }
        Fft<64, -1>::run(v);
#pragma unroll
        for (int k1 = 0; k1 < 64; ++k1) {
            float2 t = v[k1];
            if (k1 != 0) t = cmul(t, __ldg(a.tw + k1 * N2 + tg));   // W_N^{tg k1}, lane-contiguous
            buf[k1 * STRIDE + tg] = t;
        }
        group_sync<N2>(group);

        // ---- a2 step 2 + a3 unpack + a4/a5 per bin
        constexpr bool STORE = (MODE == kModeForward) && (BIG || N2 > 32);   // keep bins, squeeze later
        constexpr bool DIRECT = (MODE == kModeForward) && !STORE;           // squeeze while unpacking
        int bl[STORE ? NB : 1];
        float bsr[STORE ? NB : 1], bsi[STORE ? NB : 1];
        auto on_bin = [&](int idx, int k, float2 za, float2 zb, bool ok) {
            float P, Q, U, V, mag4;
            int l = bin_target(bc, k, za, zb, P, Q, U, V, mag4);
            if (!ok || !valid) l = -3;
            if constexpr (STORE) {
                bl[idx] = l;
                bsr[idx] = 0.5f * P;
                bsi[idx] = 0.5f * Q;
            } else if constexpr (DIRECT) {
                if (l >= 0) {
                    atomicAdd(&buf[l].x, 0.5f * P);                 // a6: T_acc[l] += S (Eq. 27/28)
                    atomicAdd(&buf[l].y, 0.5f * Q);
                }
            } else if constexpr (MODE == kModeStft) {
                if (l != -3) {
                    const int64_t o = fi * (int64_t)(N / 2 + 1) + k;
                    a.S[o] = make_float2(0.5f * P, 0.5f * Q);
                    a.Sd[o] = make_float2(U * a.inv_alpha2, -V * a.inv_alpha2);
                }
            } else if constexpr (MODE == kModeTargets) {
                if (l != -3) a.lout[fi * (int64_t)(N / 2 + 1) + k] = l;
            } else {
                if (l != -3) vmax = fmaxf(vmax, mag4);
            }
        };

        if constexpr (N2 <= 32) {
            constexpr int UNITS = 32 / N2;
            // pair-unit u of this thread: columns {j, 64-j} (j = tg + N2 u), unit 0 = {0, 32}
            auto unpack_unit = [&](int u, float2 (&A)[N2], float2 (&B)[N2]) {
                const int j = tg + N2 * u;
                const int cA = j;
                const int cB = (j == 0) ? 32 : 64 - j;
                Fft<N2, -1>::run(A);                      // A[k2] = Z[cA + 64 k2]
                Fft<N2, -1>::run(B);                      // B[k2] = Z[cB + 64 k2]
                const bool dc = (j == 0);
#pragma unroll
                for (int k2 = 0; k2 < N2 / 2; ++k2) {
                    // bin cA + 64 k2 pairs with N - k = cB + 64 (N2-1-k2)   [unit 0: 64 (N2 - k2)]
                    const float2 zbA = dc ? A[(N2 - k2) % N2] : B[N2 - 1 - k2];
                    on_bin(u * N2 + k2, cA + 64 * k2, A[k2], zbA, true);
                    // bin cB + 64 k2 pairs with cA + 64 (N2-1-k2)          [unit 0: 32 + 64 (N2-1-k2)]
                    const float2 zbB = dc ? B[N2 - 1 - k2] : A[N2 - 1 - k2];
                    on_bin(u * N2 + N2 / 2 + k2, cB + 64 * k2, B[k2], zbB, true);
                }
                if (u == 0) on_bin(NB - 1, N / 2, A[N2 / 2], A[N2 / 2], tg == 0);   // Nyquist
            };
            auto load_unit = [&](int u, float2 (&A)[N2], float2 (&B)[N2]) {
                const int j = tg + N2 * u;
                const int cA = j;
                const int cB = (j == 0) ? 32 : 64 - j;
#pragma unroll
                for (int n2 = 0; n2 < N2; ++n2) {
                    A[n2] = buf[cA * STRIDE + n2];
                    B[n2] = buf[cB * STRIDE + n2];
                }
            };
            if constexpr (DIRECT) {
                float2 A[UNITS][N2], B[UNITS][N2];
#pragma unroll
                for (int u = 0; u < UNITS; ++u) load_unit(u, A[u], B[u]);
                group_sync<N2>(group);
                for (int i = tg; i < a.bins; i += N2) buf[i] = make_float2(0.0f, 0.0f);
                group_sync<N2>(group);
#pragma unroll
                for (int u = 0; u < UNITS; ++u) unpack_unit(u, A[u], B[u]);
            } else {
#pragma unroll
                for (int u = 0; u < UNITS; ++u) {
                    float2 A[N2], B[N2];
                    load_unit(u, A, B);
                    unpack_unit(u, A, B);
                }
            }
        } else {
            // N2 == 64: column DFT per thread, then unpack through shared memory
            {
                float2 A[N2];
#pragma unroll
                for (int n2 = 0; n2 < N2; ++n2) A[n2] = buf[tg * STRIDE + n2];
                Fft<N2, -1>::run(A);
#pragma unroll
                for (int k2 = 0; k2 < N2; ++k2) buf[tg * STRIDE + k2] = A[k2];   // own column only
            }
            group_sync<N2>(group);
            const int j = tg & 31, h = tg >> 5;
            const int cA = j, cB = (j == 0) ? 32 : 64 - j;
            const bool dc = (j == 0);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int k2 = 16 * h + i;
                const float2 za = buf[cA * STRIDE + k2];
                const float2 zbA = dc ? buf[((N2 - k2) % N2)] : buf[cB * STRIDE + (N2 - 1 - k2)];
                on_bin(i, cA + 64 * k2, za, zbA, true);
                const float2 zb2 = buf[cB * STRIDE + k2];
                const float2 zbB = dc ? buf[32 * STRIDE + (N2 - 1 - k2)] : buf[cA * STRIDE + (N2 - 1 - k2)];
                on_bin(16 + i, cB + 64 * k2, zb2, zbB, true);
            }
            const float2 zn = buf[N2 / 2];             // column 0, k2 = N2/2: Nyquist
            on_bin(NB - 1, N / 2, zn, zn, tg == 0);
        }
        group_sync<N2>(group);

        // ---- a7 band store (DIRECT), or a6 + a7 in chunks of CAP bins (STORE)
        float2* trow = (MODE == kModeForward) ? reinterpret_cast<float2*>(a.T) + fi * a.ldT : nullptr;
        if constexpr (DIRECT) {
            if (valid)
                for (int i = tg; i < a.bins; i += N2) trow[i] = buf[i];
            group_sync<N2>(group);
        }
        if constexpr (STORE) {
            for (int l0 = 0; l0 < a.bins; l0 += CAP) {
                const int lc = min(CAP, a.bins - l0);
                for (int i = tg; i < lc; i += N2) buf[i] = make_float2(0.0f, 0.0f);
                group_sync<N2>(group);
#pragma unroll
                for (int i = 0; i < NB; ++i) {
                    const int l = bl[i] - l0;
                    if (bl[i] >= 0 && l >= 0 && l < lc) {
                        atomicAdd(&buf[l].x, bsr[i]);
                        atomicAdd(&buf[l].y, bsi[i]);
                    }
                }
                group_sync<N2>(group);
                if (valid)
                    for (int i = tg; i < lc; i += N2) trow[l0 + i] = buf[i];
                group_sync<N2>(group);
            }
        }
    }

    if constexpr (MODE == kModeAbsmax) {
        // block max of 4|S|^2 -> |S|
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
        __shared__ float red[kCtaThreads / 32];
        __syncthreads();
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = vmax;
        __syncthreads();
        if (threadIdx.x == 0) {
            float m = 0.0f;
            for (int w = 0; w < kCtaThreads / 32; ++w) m = fmaxf(m, red[w]);
            atomicMax(reinterpret_cast<unsigned int*>(a.absmax_out), __float_as_uint(0.5f * sqrtf(m)));
        }
    }
}

// ------------------------------------------------------------------------------- inverse ------
__device__ __forceinline__ float inv_norm(int64_t s, const InvArgs& a) {
    if (s < a.n_head) return __ldg(a.inv_head + s);
    if (s >= a.n - a.n_tail) return __ldg(a.inv_tail + (s - (a.n - a.n_tail)));
    return __ldg(a.inv_per + (int)((s + a.c) % a.hop));
}

template <int N2>
__global__ void __launch_bounds__(kCtaThreads, 2) inv_kernel(const InvArgs a) {
    using Gm = Geom<N2>;
    constexpr int N = Gm::N;
    constexpr int STRIDE = Gm::STRIDE;
    constexpr int CAP = Gm::CAP;
    constexpr int G = Gm::G;
    extern __shared__ float2 smem[];
    const int group = threadIdx.x / N2;
    const int tg = threadIdx.x % N2;
    float2* buf = smem + group * CAP;
    float* ring = reinterpret_cast<float*>(smem + G * CAP);
    const int64_t rmask = a.ring - 1;

    const int64_t F = a.frame_end - a.frame_begin;
    const int64_t f_lo = (int64_t)blockIdx.x * a.frames_per_cta;
    if (f_lo >= F) return;
    const int64_t f_hi = min(F, f_lo + a.frames_per_cta);
    const bool first_cta = (blockIdx.x == 0);
    const bool last_cta = (f_hi == F);
    const int64_t H = a.hop;
    const int last_in = a.L - 1 - a.c;

    for (int i = threadIdx.x; i < a.ring; i += kCtaThreads) ring[i] = 0.0f;
    __syncthreads();

    const int64_t g_lo = (a.frame_begin + f_lo) * H - a.c;           // first sample touched
    const int64_t left_end = g_lo + a.seam_len;                        // [g_lo, left_end) = left seam
    const int64_t right_start = (a.frame_begin + f_hi) * H - a.c;     // [right_start, ..) = right seam
    int64_t flushed = g_lo;
    const int k2band = a.k1 + a.bins / a.zoom;

    for (int64_t f0 = f_lo; f0 < f_hi; f0 += 2 * G) {
        const int64_t fA = f0 + 2 * group, fB = fA + 1;
        const bool vA = fA < f_hi, vB = fB < f_hi;
        const float2* TA = a.T + fA * a.ldT;
        const float2* TB = a.T + fB * a.ldT;
        const int64_t sA = (a.frame_begin + fA) * H, sB = sA + H;      // sample of tau = 0

        for (int b = 0; b < a.zoom; ++b) {
            // ---- a9: sub-spectrum G_b[q] = H_A[z q + b] + i H_B[z q + b] (Hermitian pair pack)
            float2 v[64];
#pragma unroll
            for (int n1 = 0; n1 < 64; ++n1) {
                const int q = N2 * n1 + tg;
                float2 val = make_float2(0.0f, 0.0f);
                if (q >= a.k1 && q < k2band) {
                    const int l = a.zoom * (q - a.k1) + b;
                    float2 ta = vA ? __ldg(TA + l) : make_float2(0.0f, 0.0f);
                    float2 tb = vB ? __ldg(TB + l) : make_float2(0.0f, 0.0f);
                    if (q == 0 && b == 0) { ta.y = 0.0f; tb.y = 0.0f; }    // DC: not doubled (R14)
                    val = make_float2(ta.x - tb.y, ta.y + tb.x);
                } else {
                    const int lm = a.zoom * (N - a.k1 - q) - b;            // conj mirror (R14)
                    if (lm >= 0 && lm < a.bins) {
                        const float2 ta = vA ? __ldg(TA + lm) : make_float2(0.0f, 0.0f);
                        const float2 tb = vB ? __ldg(TB + lm) : make_float2(0.0f, 0.0f);
                        val = make_float2(ta.x + tb.y, tb.x - ta.y);
                    }
                }
                v[n1] = val;
            }
            Fft<64, +1>::run(v);
#pragma unroll
            for (int k1 = 0; k1 < 64; ++k1) {
                float2 t = v[k1];
                if (k1 != 0) t = cmulc(t, __ldg(a.tw + k1 * N2 + tg));   // W_N^{-tg k1}
                buf[k1 * STRIDE + tg] = t;
            }
            group_sync<N2>(group);
            constexpr int COLS = 64 / N2;
#pragma unroll
            for (int ci = 0; ci < COLS; ++ci) {
                const int col = tg + N2 * ci;
                float2 u[N2];
#pragma unroll
                for (int n2 = 0; n2 < N2; ++n2) u[n2] = buf[col * STRIDE + n2];
                Fft<N2, +1>::run(u);
#pragma unroll
                for (int k2 = 0; k2 < N2; ++k2) {
                    const int p = col + 64 * k2;                 // output index tau mod N
                    const int tau = (p <= last_in) ? p : p - N;
                    if (tau < -a.c) continue;
                    float2 y = u[k2];
                    if (b != 0) y = cmul(y, __ldg(a.twz + (int64_t)(b - 1) * a.L + (tau + a.c)));   // e^{i2pi b tau/(zN)}
                    const float gw = __ldg(&a.taps[tau + a.c].x) * a.inv_n;
                    if (vA) atomicAdd(&ring[(sA + tau) & rmask], gw * y.x);
                    if (vB) atomicAdd(&ring[(sB + tau) & rmask], gw * y.y);
                }
            }
            group_sync<N2>(group);
        }
        __syncthreads();
        // ---- a10: flush completed samples
        const int64_t f_next = f0 + 2 * G;
        const int64_t next_lo = (f_next >= f_hi) ? (a.frame_begin + f_hi - 1) * H - a.c + a.L
                                                 : (a.frame_begin + f_next) * H - a.c;
        for (int64_t s = flushed + threadIdx.x; s < next_lo; s += kCtaThreads) {
            float* slot = &ring[s & rmask];
            const float val = *slot;
            *slot = 0.0f;
            if (s < 0 || s >= a.n) continue;
            if (!first_cta && s < left_end) {
                a.seam[((int64_t)blockIdx.x * 2 + 0) * a.seam_len + (s - g_lo)] = val;
            } else if (!last_cta && s >= right_start) {
                a.seam[((int64_t)blockIdx.x * 2 + 1) * a.seam_len + (s - right_start)] = val;
            } else if (a.normalize) {
                a.y[s - a.y_off] = val * inv_norm(s, a);
            } else {
                a.y[s - a.y_off] += val;
            }
        }
        flushed = next_lo;
        __syncthreads();
    }
}

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
        if (a.normalize) a.y[s - a.y_off] = val * inv_norm(s, a);
        else             a.y[s - a.y_off] += val;
    }
}

__global__ void finalize_kernel(float* y, int64_t y_off, int64_t y_len, InvArgs a) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < y_len; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = y_off + i;
        if (s < 0 || s >= a.n) continue;
        y[i] *= inv_norm(s, a);
    }
}

// ------------------------------------------------------------------------------- launchers ----
template <int N2>
static int fwd_smem() { return Geom<N2>::G * Geom<N2>::CAP * (int)sizeof(float2); }

template <int N2>
static int inv_smem(int hop, int L, int* ring_out) {
    const int span = (2 * Geom<N2>::G - 1) * hop + L;
    int ring = 1;
    while (ring < span) ring <<= 1;
    if (ring_out) *ring_out = ring;
    return Geom<N2>::G * Geom<N2>::CAP * (int)sizeof(float2) + ring * (int)sizeof(float);
}

template <int N2, int MODE, bool BIG>
static cudaError_t launch_fwd_b(const FwdArgs& a, int grid, cudaStream_t s) {
    const int smem = fwd_smem<N2>();
    cudaError_t e = cudaFuncSetAttribute(fwd_kernel<N2, MODE, BIG>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    fwd_kernel<N2, MODE, BIG><<<grid, kCtaThreads, smem, s>>>(a);
    return cudaGetLastError();
}

template <int N2, int MODE>
static cudaError_t launch_fwd_t(const FwdArgs& a, int grid, cudaStream_t s) {
    if (MODE == kModeForward && N2 <= 32 && a.bins > Geom<N2>::CAP) return launch_fwd_b<N2, MODE, true>(a, grid, s);
    return launch_fwd_b<N2, MODE, false>(a, grid, s);
}

template <int N2>
static cudaError_t launch_fwd_mode(const FwdArgs& a, int mode, int grid, cudaStream_t s) {
    switch (mode) {
        case kModeForward: return launch_fwd_t<N2, kModeForward>(a, grid, s);
        case kModeStft: return launch_fwd_t<N2, kModeStft>(a, grid, s);
        case kModeTargets: return launch_fwd_t<N2, kModeTargets>(a, grid, s);
        case kModeAbsmax: return launch_fwd_t<N2, kModeAbsmax>(a, grid, s);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_forward(const FwdArgs& a, int mode, int grid, cudaStream_t s) {
    switch (a.nfft) {
        case 128: return launch_fwd_mode<2>(a, mode, grid, s);
        case 256: return launch_fwd_mode<4>(a, mode, grid, s);
        case 512: return launch_fwd_mode<8>(a, mode, grid, s);
        case 1024: return launch_fwd_mode<16>(a, mode, grid, s);
        case 2048: return launch_fwd_mode<32>(a, mode, grid, s);
        case 4096: return launch_fwd_mode<64>(a, mode, grid, s);
    }
    return cudaErrorInvalidValue;
}

int forward_smem_bytes(int nfft) {
    switch (nfft) {
        case 128: return fwd_smem<2>();
        case 256: return fwd_smem<4>();
        case 512: return fwd_smem<8>();
        case 1024: return fwd_smem<16>();
        case 2048: return fwd_smem<32>();
        case 4096: return fwd_smem<64>();
    }
    return -1;
}

template <int N2>
static int occ_fwd(int device) {
    int nb = 0, sms = 0;
    const int smem = fwd_smem<N2>();
    cudaFuncSetAttribute(fwd_kernel<N2, kModeForward, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fwd_kernel<N2, kModeForward, false>, kCtaThreads, smem);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    return (nb > 0 ? nb : 1) * sms;
}

int forward_max_grid(int nfft, int device) {
    switch (nfft) {
        case 128: return occ_fwd<2>(device);
        case 256: return occ_fwd<4>(device);
        case 512: return occ_fwd<8>(device);
        case 1024: return occ_fwd<16>(device);
        case 2048: return occ_fwd<32>(device);
        case 4096: return occ_fwd<64>(device);
    }
    return -1;
}

template <int N2>
static cudaError_t launch_inv_t(const InvArgs& a, int grid, cudaStream_t s) {
    const int smem = inv_smem<N2>(a.hop, a.L, nullptr);
    cudaError_t e = cudaFuncSetAttribute(inv_kernel<N2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    inv_kernel<N2><<<grid, kCtaThreads, smem, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_inverse(const InvArgs& a, int grid, cudaStream_t s) {
    switch (a.nfft) {
        case 128: return launch_inv_t<2>(a, grid, s);
        case 256: return launch_inv_t<4>(a, grid, s);
        case 512: return launch_inv_t<8>(a, grid, s);
        case 1024: return launch_inv_t<16>(a, grid, s);
        case 2048: return launch_inv_t<32>(a, grid, s);
        case 4096: return launch_inv_t<64>(a, grid, s);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_inverse_seams(const InvArgs& a, int ctas, cudaStream_t s) {
    if (ctas < 2 || a.seam_len <= 0) return cudaSuccess;
    const int64_t total = (int64_t)(ctas - 1) * a.seam_len;
    const int threads = 256;
    const int blocks = (int)((total + threads - 1) / threads < 4096 ? (total + threads - 1) / threads : 4096);
    seam_kernel<<<blocks, threads, 0, s>>>(a, ctas);
    return cudaGetLastError();
}

cudaError_t launch_finalize(float* y, int64_t y_off, int64_t y_len, int64_t n, int32_t hop, int32_t c,
                            const float* inv_head, int32_t n_head, const float* inv_tail, int32_t n_tail,
                            const float* inv_per, cudaStream_t s) {
    InvArgs a{};
    a.n = n; a.hop = hop; a.c = c;
    a.inv_head = inv_head; a.n_head = n_head; a.inv_tail = inv_tail; a.n_tail = n_tail; a.inv_per = inv_per;
    const int threads = 256;
    const int blocks = (int)((y_len + threads - 1) / threads < 2368 ? (y_len + threads - 1) / threads : 2368);
    if (blocks <= 0) return cudaSuccess;
    finalize_kernel<<<blocks, threads, 0, s>>>(y, y_off, y_len, a);
    return cudaGetLastError();
}

int inverse_smem_bytes(int nfft, int hop, int L, int* ring_out) {
    switch (nfft) {
        case 128: return inv_smem<2>(hop, L, ring_out);
        case 256: return inv_smem<4>(hop, L, ring_out);
        case 512: return inv_smem<8>(hop, L, ring_out);
        case 1024: return inv_smem<16>(hop, L, ring_out);
        case 2048: return inv_smem<32>(hop, L, ring_out);
        case 4096: return inv_smem<64>(hop, L, ring_out);
    }
    return -1;
}

template <int N2>
static int occ_inv(int hop, int L, int device) {
    int nb = 0, sms = 0;
    const int smem = inv_smem<N2>(hop, L, nullptr);
    cudaFuncSetAttribute(inv_kernel<N2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, inv_kernel<N2>, kCtaThreads, smem);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    return (nb > 0 ? nb : 1) * sms;
}

int inverse_max_grid(int nfft, int hop, int L, int device) {
    switch (nfft) {
        case 128: return occ_inv<2>(hop, L, device);
        case 256: return occ_inv<4>(hop, L, device);
        case 512: return occ_inv<8>(hop, L, device);
        case 1024: return occ_inv<16>(hop, L, device);
        case 2048: return occ_inv<32>(hop, L, device);
        case 4096: return occ_inv<64>(hop, L, device);
    }
    return -1;
}

}  // namespace sst
