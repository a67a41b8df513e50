// Fused inverse kernel (rows a9-a11 of DESIGN.md §1): two frames per complex IFFT (Hermitian
//   packing), the z N_f-point band IDFT of P:L222 split into z N_f-point sub-transforms by residue
//   b = j mod z; work item = (frame pair, b), one per group; outer phase e^{i 2 pi b tau/(z N)}; the
//   CTA sums a pair's items, windows by g[tau+c]/N_f and overlap-adds frame A (real part) and frame
//   B (imaginary part) into a shared-memory ring (Eq. 26).  Samples shared with the neighbouring
//   CTA go to a seam buffer combined by seam_kernel (sst_kernels.cu).
#pragma once

#include "common.cuh"

namespace sst {

// Work item = (frame pair, residue b).  A tile holds P = max(1, G/z) consecutive frame pairs, so
// its P z items occupy the G groups in ceil(P z / G) passes (one pass for every config here).
// Per item the group computes V_b = IDFT_N of the Hermitian-packed sub-spectrum
// G_b[q] = H_A[z q + b] + i H_B[z q + b] and leaves e^{i 2 pi b tau/(z N)} V_b[p] in its buffer
// (indexed by p = tau mod N).  The CTA then sums the items of each pair over b, windows by
// g[tau + c]/N and adds frame A (real part) and frame B (imaginary part) into the OLA ring.
// RM: every nonzero sub-spectrum entry q (band [k1, k2) or mirror [N - k2, N)) has
// q / N2 in [0, RM) or [64 - RM, 64) (i.e. ceil(k2 / N2) <= RM): other rows of the step-1
// input are compile-time zeros and cost nothing (narrow bands: C2, C3 use RM = 5, C4 RM = 8).
// RM = kRmFull: the full band (k1 = 0, B = z N/2, e.g. C5): every row is live and the T index of
// an entry is affine in its row, so the loads need no per-entry index arithmetic.
// ZONE: the mode-retrieval zone is applied to the T loads (a.zone_path); a separate
// instantiation, so the plain inverse carries no zone arithmetic
constexpr int kRmFull = 0;

template <int N2, bool FULLWIN, int RM, bool ZONE>
__global__ void __launch_bounds__(Geom<N2, false>::TPB, Geom<N2, false>::TPB == 256 ? 1 : 2) inv_kernel(const InvArgs a) {
    using Gm = Geom<N2, false>;
    constexpr int N = Gm::N;
    constexpr int TPB = Gm::TPB;
    constexpr int STRIDE = Gm::STRIDE;
    constexpr int CAP = Gm::CAP;
    constexpr int G = Gm::G;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float2* smem = reinterpret_cast<float2*>(smem_raw);
    float* g_s = reinterpret_cast<float*>(smem_raw + a.lay.g_off);
    float* ring = reinterpret_cast<float*>(smem_raw + a.lay.ring_off);
    const int group = threadIdx.x / N2;
    const int tg = threadIdx.x % N2;
    float2* buf = smem + group * CAP;
    const int rmask = a.lay.ring - 1;

    const int64_t F = a.frame_end - a.frame_begin;
    const int64_t f_lo = (int64_t)blockIdx.x * a.frames_per_cta;
    if (f_lo >= F) return;
    const int64_t f_hi = min(F, f_lo + a.frames_per_cta);
    const bool first_cta = (blockIdx.x == 0);
    const bool last_cta = (f_hi == F);
    const int64_t H = a.hop;
    const int c = a.c;
    const int last_in = a.L - 1 - c;
    const int zoom = a.zoom;
    const int P = a.lay.pairs;                            // frame pairs per tile
    const int items = P * zoom;
    const int k1 = a.k1;
    const int nr = a.bins / zoom;                          // N_r
    const float inv_n = a.inv_n;

    for (int i = threadIdx.x; i < a.lay.ring; i += TPB) ring[i] = 0.0f;
    for (int i = threadIdx.x; i < a.L; i += TPB) g_s[i] = __ldg(&a.taps[i].x) * inv_n;
    __syncthreads();

    const int64_t g_lo = (a.frame_begin + f_lo) * H - c;            // first sample touched
    const int64_t left_end = g_lo + a.seam_len;                      // [g_lo, left_end) = left seam
    const int64_t right_start = (a.frame_begin + f_hi) * H - c;     // [right_start, ..) = right seam
    int64_t flushed = g_lo;

    for (int64_t f0 = f_lo; f0 < f_hi; f0 += 2 * P) {
        {
            // L2 prefetch of the next tile's T rows (2P rows of B complex values): their DRAM
            // latency overlaps this tile's transforms
            const int64_t fn = f0 + 2 * P;
            const int nrows = (int)min((int64_t)(2 * P), f_hi - fn);
            const int lines = (a.bins * 8 + 127) >> 7;
            for (int i = threadIdx.x; i < nrows * lines; i += TPB) {
                const int r = i / lines, q = i - r * lines;
                const char* ptr = reinterpret_cast<const char*>(a.T + (fn + r) * a.ldT) + q * 128;
                asm volatile("prefetch.global.L2 [%0];" ::"l"(ptr));
            }
        }
        for (int it0 = 0; it0 < items; it0 += G) {
            // ---------------- per-group item: sub-IFFT of one (pair, b)
            const int item = it0 + group;
            const int pair = item / zoom, b = item - pair * zoom;
            const int64_t fA = f0 + 2 * pair;
            const bool vA = item < items && fA < f_hi;
            const bool vB = vA && fA + 1 < f_hi;
            const float2* TA = a.T + (vA ? fA : f_lo) * a.ldT;
            const float2* TB = vB ? TA + a.ldT : TA;
            // mode retrieval zone: centre bins of frames A and B (none: keep everything)
            const int zA = ZONE && vA ? __ldg(a.zone_path + fA) : 0;
            const int zB = ZONE && vB ? __ldg(a.zone_path + fA + 1) : 0;
            float2 v[64];
            if constexpr (RM == kRmFull) {
                // full band (k1 = 0, B = z N/2): rows n1 < 32 hold the band entries q = N2 n1 + tg
                // (li = z q + b), rows n1 >= 32 the mirror entries (li = z (N - q) - b); li is affine
                // in n1, so each entry is one load at a fixed stride from a per-thread base, with no
                // index arithmetic or range tests.  The one empty entry is q = N/2 at b = 0 (li = B).
                const int zs = zoom * N2;
                // no validity predicates: an invalid item (vA false) is never combined, and with no
                // frame B, TB = TA makes H_B Hermitian, so frame A's real part is unaffected and the
                // imaginary part is not added (hasB false); every address stays inside row f_lo / fA
                const float2* pA = TA + (zoom * tg + b);
                const float2* pB = TB + (zoom * tg + b);
#pragma unroll
                for (int n1 = 0; n1 < 32; ++n1) {
                    SST_CHECK(zoom * (N2 * n1 + tg) + b < a.bins);
                    float2 ta = __ldg(pA + n1 * zs);
                    float2 tb = __ldg(pB + n1 * zs);
                    if (n1 == 0 && tg == 0 && b == 0) { ta.y = 0.0f; tb.y = 0.0f; }   // DC: real part only (R14)
                    v[n1] = __fadd2_rn(ta, make_float2(-tb.y, tb.x));                // H_A + i H_B
                }
                const float2* mA = TA + (zoom * (N / 2 - tg) - b);                 // li at n1 = 32
                const float2* mB = TB + (zoom * (N / 2 - tg) - b);
                const bool m0 = tg != 0 || b != 0;                                  // q = N/2, b = 0: none
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const bool ok = j > 0 || m0;
                    SST_CHECK(!ok || (zoom * (N / 2 - tg) - b - j * zs >= 0 && zoom * (N / 2 - tg) - b - j * zs < a.bins));
                    const float2 ta = ok ? __ldg(mA - j * zs) : make_float2(0.0f, 0.0f);
                    const float2 tb = ok ? __ldg(mB - j * zs) : make_float2(0.0f, 0.0f);
                    v[32 + j] = __fadd2_rn(make_float2(ta.x, tb.x), make_float2(tb.y, -ta.y));   // conj H_A + i conj H_B
                }
            } else {
                // band entries q in [k1, k2): l = z (q - k1) + b; mirror entries: l' = z (N - k1 - q) - b
                const int zstep = zoom * N2;                           // l step per row n1
                const int lbase = zoom * (tg - k1) + b;                // band l at n1 = 0
                const int mbase = zoom * (N - k1 - tg) - b;            // mirror l at n1 = 0
#pragma unroll
                for (int n1 = 0; n1 < 64; ++n1) {
                    if (n1 >= RM && n1 < 64 - RM) {                   // outside band and mirror
                        v[n1] = make_float2(0.0f, 0.0f);
                        continue;
                    }
                    const int q = N2 * n1 + tg;                       // sub-spectrum index (coarse bin)
                    // RM < 32: rows below RM can only hold band entries, rows above 64 - RM only mirror
                    // entries (k2 <= RM N2 and N - k2 >= (64 - RM) N2)
                    const bool lower = (RM < 32) ? (n1 < RM) : true;
                    const bool upper = (RM < 32) ? (n1 >= 64 - RM) : true;
                    const bool inb = lower && (unsigned)(q - k1) < (unsigned)nr;
                    const int lm = mbase - n1 * zstep;
                    const bool inm = upper && !inb && q > 0 && (unsigned)lm < (unsigned)a.bins;
                    const int li = inb ? lbase + n1 * zstep : lm;
                    float2 ta = make_float2(0.0f, 0.0f), tb = make_float2(0.0f, 0.0f);
                    SST_CHECK(!(inb || inm) || (li >= 0 && li < a.bins));
                    const bool okA = !ZONE || ((abs(li - zA) <= a.zone_half) == (bool)a.zone_keep);
                    const bool okB = !ZONE || ((abs(li - zB) <= a.zone_half) == (bool)a.zone_keep);
                    if ((inb || inm) && vA && okA) ta = __ldg(TA + li);
                    if ((inb || inm) && vB && okB) tb = __ldg(TB + li);
                    if (n1 == 0 && q == 0 && b == 0) { ta.y = 0.0f; tb.y = 0.0f; }  // DC: real part only (R14)
                    if (n1 == 32 && q == N / 2 && b == 0) { ta.y = 0.0f; tb.y = 0.0f; }   // Nyquist (full band only)
                    v[n1] = inb ? make_float2(ta.x - tb.y, ta.y + tb.x)    // H_A + i H_B
                                : make_float2(ta.x + tb.y, tb.x - ta.y);   // conj H_A + i conj H_B
                }
            }
            if constexpr (RM != kRmFull && RM < 32) FftSparse64<+1, RM>::run(v);   // zero rows skipped
            else Fft<64, +1>::run(v);
#pragma unroll
            for (int kk = 0; kk < 64; ++kk) {
                float2 t = v[kk];
                if (kk != 0) t = cmulc(t, __ldg(a.tw + kk * N2 + tg));   // W_N^{-tg kk}
                SST_CHECK(kk * STRIDE + tg < CAP);
                buf[kk * STRIDE + tg] = t;
            }
            group_sync<N2>(group);
            if constexpr (N2 == 128) {
                // N_f = 8192: 128-point column IDFT of column c split over (c, hh) as in the forward
                const int c = tg & 63, hh = tg >> 6;
                {
                    float2 A[64];
#pragma unroll
                    for (int m = 0; m < 64; ++m) A[m] = buf[c * STRIDE + 2 * m + hh];
                    group_sync<N2>(group);
                    Fft<64, +1>::run(A);
#pragma unroll
                    for (int k = 0; k < 64; ++k) {
                        float2 t = A[k];
                        if (hh && k) t = cmulc(t, __ldg(a.tw + k * N2 + 64));   // W_128^{-k}
                        buf[c * STRIDE + 64 * hh + k] = t;
                    }
                }
                group_sync<N2>(group);
                float2 Y[64];                                     // outputs p = c + 64 k2, k2 = 64 hh + k
#pragma unroll
                for (int k = 0; k < 64; ++k) {
                    const float2 e = buf[c * STRIDE + k], o = buf[c * STRIDE + 64 + k];
                    Y[k] = hh ? csub(e, o) : cadd(e, o);
                }
                group_sync<N2>(group);
                const bool rot = b != 0;
                const float2* pb = a.phz + b * (64 + 2 * N2);          // phase tables of residue b
                const float2 fb = __ldg(pb + c);                        // e(b c)
#pragma unroll
                for (int k = 0; k < 64; ++k) {
                    const int k2 = 64 * hh + k;
                    const int p = c + 64 * k2;
                    float2 y = Y[k];
                    const bool wrap = p > last_in;                      // tau = p - N
                    if (rot && (!wrap || p - N >= -a.c))
                        y = cmul(y, cmul(fb, __ldg(pb + 64 + (wrap ? N2 : 0) + k2)));   // e^{i 2 pi b tau/(z N)}
                    buf[p] = y;
                }
            } else {
                constexpr int COLS = 64 / N2;
                float2 u[COLS][N2];
#pragma unroll
                for (int ci = 0; ci < COLS; ++ci)
#pragma unroll
                    for (int n2 = 0; n2 < N2; ++n2) u[ci][n2] = buf[(tg + N2 * ci) * STRIDE + n2];
                group_sync<N2>(group);
                const bool rot = b != 0;
                const float2* pb = a.phz + b * (64 + 2 * N2);              // phase tables of residue b
#pragma unroll
                for (int ci = 0; ci < COLS; ++ci) {
                    const int col = tg + N2 * ci;
                    Fft<N2, +1>::run(u[ci]);
                    const float2 fb = __ldg(pb + col);                      // e(b col)
                    // FULLWIN: the phase e(b tau) of consecutive k2 advances by e(64 b): a recurrence started
                    // from the table at k2 = 0 and again at the wrap k2 = N2/2 (tau = p - N), <= N2/2 steps
                    const float2 step = __ldg(pb + 64 + 1);                 // e(64 b)
                    float2 ph = fb;
#pragma unroll
                    for (int k2 = 0; k2 < N2; ++k2) {
                        const int p = col + 64 * k2;                  // output index tau mod N
                        float2 y = u[ci][k2];
                        if constexpr (FULLWIN) {
                            // tau = p (k2 < N2/2) or p - N: e(b tau) = e(b col) e(b (64 k2 [- N]))
                            if (k2 == N2 / 2) ph = cmul(fb, __ldg(pb + 64 + N2 + k2));
                            if (rot) {
                                y = cmul(y, ph);
                                if (k2 + 1 < N2) ph = cmul(ph, step);
                            }
                        } else {
                            const bool wrap = p > last_in;
                            if (rot && (!wrap || p - N >= -c)) y = cmul(y, cmul(fb, __ldg(pb + 64 + (wrap ? N2 : 0) + k2)));
                        }
                        buf[p] = y;
                    }
                }
            }
            __syncthreads();
            // ---------------- combine the items of each pair over b, window, OLA into the ring.
            // Each thread owns positions p = threadIdx.x + TPB j; frame A (real part) and frame B
            // (imaginary part, H samples later) are added in two barrier-separated phases, so
            // every ring slot has a single writer per phase (no atomics).
            constexpr int PPT = (N + TPB - 1) / TPB;
            const int pr_lo = it0 / zoom, pr_hi = min(P, (it0 + G + zoom - 1) / zoom);
            for (int pr = pr_lo; pr < pr_hi; ++pr) {
                const int64_t fa = f0 + 2 * pr;
                if (fa >= f_hi) break;                         // CTA-uniform
                const bool hasB = fa + 1 < f_hi;
                const int i_lo = max(it0, pr * zoom) - it0, i_hi = min(it0 + G, pr * zoom + zoom) - it0;
                const int64_t sA = (a.frame_begin + fa) * H;
                float2 y[PPT];
                int slot[PPT];
                // sum of the pair's items (compile-time count for the usual z = 1, 2, 4, 8)
                auto combine = [&](auto nic) {
                    constexpr int NI = decltype(nic)::value;
#pragma unroll
                    for (int jj = 0; jj < PPT; ++jj) {
                        const int p = threadIdx.x + TPB * jj;
                        const int tau = (p <= last_in) ? p : p - N;
                        const bool ok = (FULLWIN || (p < N && tau >= -c));
                        float2 acc = make_float2(0.0f, 0.0f);
                        if (ok) {
                            const float2* sp = smem + i_lo * CAP + p;
                            if constexpr (NI > 0) {
                                acc = sp[0];
#pragma unroll
                                for (int i = 1; i < NI; ++i) acc = cadd(acc, sp[i * CAP]);
                            } else {
                                for (int i = 0; i < i_hi - i_lo; ++i) acc = cadd(acc, sp[i * CAP]);
                            }
                            acc = cscale(acc, g_s[tau + c]);
                        }
                        y[jj] = acc;
                        slot[jj] = ok ? (int)((sA + tau) & rmask) : -1;
                    }
                };
                switch (i_hi - i_lo) {
                    case 1: combine(IntC<1>{}); break;
                    case 2: combine(IntC<2>{}); break;
                    case 4: combine(IntC<4>{}); break;
                    case 8: combine(IntC<8>{}); break;
                    default: combine(IntC<0>{}); break;
                }
#pragma unroll
                for (int jj = 0; jj < PPT; ++jj)
                    if (slot[jj] >= 0) {
                        SST_CHECK(slot[jj] < a.lay.ring);
                        ring[slot[jj]] += y[jj].x;
                    }
                __syncthreads();
                if (hasB) {
#pragma unroll
                    for (int jj = 0; jj < PPT; ++jj)
                        if (slot[jj] >= 0) ring[(slot[jj] + (int)H) & rmask] += y[jj].y;
                }
                __syncthreads();
            }
        }
        // ---------------- a10: flush completed samples
        const int64_t f_next = f0 + 2 * P;
        const int64_t next_lo = (f_next >= f_hi) ? (a.frame_begin + f_hi - 1) * H - c + a.L
                                                 : (a.frame_begin + f_next) * H - c;
        for (int64_t s = flushed + threadIdx.x; s < next_lo; s += TPB) {
            float* slot = &ring[(int)(s & rmask)];
            const float val = *slot;
            *slot = 0.0f;
            if (s < 0 || s >= a.n) continue;
            if (!first_cta && s < left_end) {
                SST_CHECK(s - g_lo >= 0 && s - g_lo < a.seam_len);
                a.seam[((int64_t)blockIdx.x * 2 + 0) * a.seam_len + (s - g_lo)] = val;
            } else if (!last_cta && s >= right_start) {
                SST_CHECK(s - right_start >= 0 && s - right_start < a.seam_len);
                a.seam[((int64_t)blockIdx.x * 2 + 1) * a.seam_len + (s - right_start)] = val;
            } else if (a.normalize) {
                // (a per-sample 32-bit mod_pos here measured 4 % slower on C4: one more live register)
                SST_CHECK(s - a.y_off >= 0 && s - a.y_off < a.y_len);
                a.y[s - a.y_off] = val * inv_norm(s, a) * a.out_scale;
            } else {
                SST_CHECK(s - a.y_off >= 0 && s - a.y_off < a.y_len);
                a.y[s - a.y_off] += val;
            }
        }
        flushed = next_lo;
        __syncthreads();
    }
}

template <int N2, bool FULLWIN, int RM, bool ZONE = false>
static cudaError_t launch_inv_b(const InvArgs& a, int grid, cudaStream_t s) {
    auto kern = inv_kernel<N2, FULLWIN, RM, ZONE>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, a.lay.total);
    if (e != cudaSuccess) return e;
    kern<<<grid, Geom<N2, false>::TPB, a.lay.total, s>>>(a);
    return cudaGetLastError();
}

template <int N2, bool FULLWIN>
static cudaError_t launch_inv_r(const InvArgs& a, int grid, cudaStream_t s) {
    if (a.zone_path) return launch_inv_b<N2, FULLWIN, 64, true>(a, grid, s);   // mode retrieval (f1)
    if (a.k1 == 0 && a.bins == a.zoom * (Geom<N2, false>::N / 2)) return launch_inv_b<N2, FULLWIN, kRmFull>(a, grid, s);   // C5
    const int rows = (a.k1 + a.bins / a.zoom + N2 - 1) / N2;   // ceil(k2 / N2)
    if (rows <= 5) return launch_inv_b<N2, FULLWIN, 5>(a, grid, s);   // C2, C3
    if (rows <= 8) return launch_inv_b<N2, FULLWIN, 8>(a, grid, s);
    if (rows <= 16) return launch_inv_b<N2, FULLWIN, 16>(a, grid, s);
    return launch_inv_b<N2, FULLWIN, 64>(a, grid, s);
}

template <int N2>
static cudaError_t launch_inv_t(const InvArgs& a, int grid, cudaStream_t s) {
    if (a.L == Geom<N2, false>::N && a.c == Geom<N2, false>::N / 2) return launch_inv_r<N2, true>(a, grid, s);
    return launch_inv_r<N2, false>(a, grid, s);
}

template <int N2>
static int occ_inv(int hop, int L, int zoom, int device) {
    int nb = 0, sms = 0;
    const int smem = inv_layout(N2, L, hop, zoom).total;
    auto kern = inv_kernel<N2, true, 64, false>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, Geom<N2, false>::TPB, smem);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    return (nb > 0 ? nb : 1) * sms;
}

}  // namespace sst
