// sm_100a kernels of the fast downsampled SST (He & Cao, arXiv 2003.07065).
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

#include "decide.cuh"
#include "fft.cuh"
#include "sst_internal.h"

#ifdef SST_DEV_N2
#define SST_HAS(n2) ((n2) == SST_DEV_N2)
#else
#define SST_HAS(n2) 1
#endif

namespace sst {

cudaError_t upload_w64(const float2* w64_host) {
    return cudaMemcpyToSymbol(c_w64, w64_host, sizeof(float2) * 64);
}

template <int V>
struct IntC {
    static constexpr int value = V;
};

template <int N2, bool FWD>
struct Geom {
    static constexpr int N = 64 * N2;
    static constexpr int TPB = tpb_of(N2, FWD);
    static constexpr int G = groups_of(N2, FWD);
    static constexpr int STRIDE = N2 + 1;         // padded exchange row (odd -> conflict-free)
    static constexpr int CAP = cap_of(N2);        // float2 per group buffer
};

template <int N2>
__device__ __forceinline__ void group_sync(int group) {
    if constexpr (N2 <= 32) {
        __syncwarp();
    } else {
        asm volatile("bar.sync %0, %1;" ::"r"(1 + group), "r"(N2) : "memory");
    }
}

// ------------------------------------------------------------------------ TMA bulk copy helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// one-dimensional bulk copy global -> shared, completion counted on bar (bytes % 16 == 0)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// ------------------------------------------------------------------------------- forward ------
// Tile t of a CTA covers frames [fb + t G, fb + t G + G) and input samples [s_lo, s_hi).  It is
// fetched with one bulk copy when the 16-byte aligned span lies inside the valid x slice;
// otherwise (record / slice edges, misaligned x) the CTA loads it cooperatively with zero fill.
struct TileIn {
    int64_t s_lo, a_lo;   // first sample; first copied x index (aligned)
    int pad, bytes;       // s_lo - (x_off + a_lo); bytes of the bulk copy
    bool bulk;
};

template <int G>
__device__ __forceinline__ TileIn tile_in(const FwdArgs& a, int64_t t, bool x_aligned) {
    TileIn ti;
    const int64_t f = a.frame_begin + t * G;
    ti.s_lo = f * a.hop - a.c;
    const int64_t s_hi = (f + G - 1) * a.hop - a.c + a.L;
    const int64_t v_lo = a.x_off > 0 ? a.x_off : 0;
    const int64_t v_hi = min(a.n, a.x_off + a.x_len);
    const int64_t d0 = ti.s_lo - a.x_off;
    ti.a_lo = d0 - (((d0 % 4) + 4) % 4);
    const int64_t a_hi = (s_hi - a.x_off + 3) / 4 * 4;
    ti.pad = (int)(d0 - ti.a_lo);
    ti.bytes = (int)((a_hi - ti.a_lo) * 4);
    ti.bulk = x_aligned && a.x_off + ti.a_lo >= v_lo && a.x_off + a_hi <= v_hi && a_hi - ti.a_lo <= a.lay.xcap;
    return ti;
}

// BIG: the band row (B bins) does not fit the group's exchange buffer (B > CAP): bins are kept
// in registers and squeezed in chunks of CAP.  Otherwise (N2 <= 32) all column data is read into
// registers first and the exchange buffer is reused as the band accumulator.
// FULLWIN: L == N_f and c == N_f/2 (all of C2-C5): the packed index n = N2 n1 + tg maps to
// tau = n (n1 < 32) or n - N (n1 >= 32) at compile time, so the gather has no checks.
template <int N2, int MODE, bool BIG, bool FULLWIN>
__global__ void __launch_bounds__(Geom<N2, true>::TPB, Geom<N2, true>::TPB == 256 ? 1 : 2) fwd_kernel(const FwdArgs a) {
    using Gm = Geom<N2, true>;
    constexpr int N = Gm::N;
    constexpr int TPB = Gm::TPB;
    constexpr int STRIDE = Gm::STRIDE;
    constexpr int CAP = Gm::CAP;
    constexpr int G = Gm::G;
    constexpr int NB = 33;                         // source bins per thread (+1 Nyquist slot)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float2* smem = reinterpret_cast<float2*>(smem_raw);
    float2* taps_s = reinterpret_cast<float2*>(smem_raw + a.lay.taps_off);
    float* xbuf = reinterpret_cast<float*>(smem_raw + a.lay.xb_off);
    uint64_t* mbar = reinterpret_cast<uint64_t*>(smem_raw + a.lay.mbar_off);
    const int group = threadIdx.x / N2;
    const int tg = threadIdx.x % N2;
    float2* buf = smem + group * CAP;

    float gam4 = a.gamma2x4;
    if (a.absmax_dev) {
        const float gm = a.gamma_rel * __ldg(a.absmax_dev);
        gam4 = 4.0f * gm * gm;
    }

    const int64_t nfr = a.frame_end - a.frame_begin;
    const int64_t ntiles = (nfr + G - 1) / G;
    const int64_t tiles_per_cta = (ntiles + gridDim.x - 1) / gridDim.x;
    const int64_t t_begin = (int64_t)blockIdx.x * tiles_per_cta;
    const int64_t t_end = min(ntiles, t_begin + tiles_per_cta);
    const int last_in = a.L - 1 - a.c;             // largest tau
    const bool x_aligned = (reinterpret_cast<uintptr_t>(a.x) & 15) == 0;
    float vmax = 0.0f;

    for (int i = threadIdx.x; i < a.L; i += TPB) taps_s[i] = __ldg(a.taps + i);
    if (threadIdx.x == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0 && t_begin < t_end) {
        const TileIn ti = tile_in<G>(a, t_begin, x_aligned);
        if (ti.bulk) {
            mbar_arrive_tx(&mbar[0], ti.bytes);
            bulk_g2s(xbuf, a.x + ti.a_lo, ti.bytes, &mbar[0]);
        }
    }
    uint32_t phase = 0;                            // bit b = parity of buffer b's next completion

    for (int64_t tile = t_begin; tile < t_end; ++tile) {
        const int bsel = (int)((tile - t_begin) & 1);
        float* xb = xbuf + bsel * a.lay.xcap;
        // prefetch tile + 1 into the other buffer (freed by the barrier that ended tile - 1)
        if (threadIdx.x == 0 && tile + 1 < t_end) {
            const TileIn tn = tile_in<G>(a, tile + 1, x_aligned);
            if (tn.bulk) {
                fence_proxy_async();
                mbar_arrive_tx(&mbar[bsel ^ 1], tn.bytes);
                bulk_g2s(xbuf + (bsel ^ 1) * a.lay.xcap, a.x + tn.a_lo, tn.bytes, &mbar[bsel ^ 1]);
            }
        }
        const TileIn ti = tile_in<G>(a, tile, x_aligned);
        int pad = ti.pad;
        if (ti.bulk) {
            mbar_wait(&mbar[bsel], (phase >> bsel) & 1);
            phase ^= 1u << bsel;
        } else {
            const int64_t v_lo = a.x_off > 0 ? a.x_off : 0;
            const int64_t v_hi = min(a.n, a.x_off + a.x_len);
            const int span = (G - 1) * a.hop + a.L;
            for (int i = threadIdx.x; i < span; i += TPB) {
                const int64_t s = ti.s_lo + i;
                xb[i] = (s >= v_lo && s < v_hi) ? __ldg(a.x + (s - a.x_off)) : 0.0f;
            }
            pad = 0;
            __syncthreads();
        }

        const int64_t fi = tile * G + group;       // frame index within the launch
        const bool valid = fi < nfr;
        const float* xw = xb + pad + group * a.hop; // x[m H - c + j], j = 0..L-1 (j = tau + c)

        // ---- a1: gather + pack (circular placement), a2 step 1: 64-point DFT of row tg
        float2 v[64];
        if constexpr (FULLWIN) {
            const float* xt = xw + tg;
            const float2* wt = taps_s + tg;
#pragma unroll
            for (int n1 = 0; n1 < 64; ++n1) {
                const int j = N2 * n1 + (n1 < 32 ? N / 2 : -N / 2);   // tau + c - tg (compile time)
                v[n1] = cscale(wt[j], xt[j]);
            }
        } else {
#pragma unroll
            for (int n1 = 0; n1 < 64; ++n1) {
                const int n = N2 * n1 + tg;
                const int j = ((n <= last_in) ? n : n - N) + a.c;
                float2 val = make_float2(0.0f, 0.0f);
                if (j >= 0) val = cscale(taps_s[j], xw[j]);
                v[n1] = val;
            }
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
        // forward: bins are computed branch-free into registers (phase 1), then squeezed with
        // predicated shared-memory atomics in chunks of CAP bins (phase 2; one chunk unless BIG)
        constexpr bool STORE = (MODE == kModeForward);
        int bl[STORE ? NB : 1];
        float bsr[STORE ? NB : 1], bsi[STORE ? NB : 1];
        auto on_bin = [&](int idx, int k, float2 za, float2 zb, bool ok) {
            float2 PQ, UV;
            float mag4;
            int l = bin_target(a, gam4, k, za, zb, PQ, UV, mag4);
            if (!ok || !valid) l = -3;
            if constexpr (STORE) {
                bl[idx] = l;
                const float2 S = cscale(PQ, 0.5f);
                bsr[idx] = S.x;
                bsi[idx] = S.y;
            } else if constexpr (MODE == kModeStft) {
                if (l != -3) {
                    const int64_t o = fi * (int64_t)(N / 2 + 1) + k;
                    a.S[o] = cscale(PQ, 0.5f);
                    a.Sd[o] = __fmul2_rn(UV, make_float2(a.inv_alpha2, -a.inv_alpha2));
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
#pragma unroll
            for (int u = 0; u < UNITS; ++u) {
                float2 A[N2], B[N2];
                load_unit(u, A, B);
                unpack_unit(u, A, B);
            }
        } else if constexpr (N2 == 128) {
            // N_f = 8192: the 128-point column DFT of column c is split between threads (c, hh):
            // hh = 0 takes the even rows, hh = 1 the odd rows (times W_128^k); the buffer then holds
            // E_c[k] | W O_c[k] and Z[c + 64 k2] = E + W O (k2 < 64), E - W O (k2 >= 64)
            {
                const int c = tg & 63, hh = tg >> 6;
                float2 A[64];
#pragma unroll
                for (int m = 0; m < 64; ++m) A[m] = buf[c * STRIDE + 2 * m + hh];
                group_sync<N2>(group);
                Fft<64, -1>::run(A);
#pragma unroll
                for (int k = 0; k < 64; ++k) {
                    float2 t = A[k];
                    if (hh && k) t = cmul(t, __ldg(a.tw + k * N2 + 64));   // W_N^{64 k} = W_128^k
                    buf[c * STRIDE + 64 * hh + k] = t;
                }
            }
            group_sync<N2>(group);
            auto Xp = [&](int c, int k) { return cadd(buf[c * STRIDE + k], buf[c * STRIDE + 64 + k]); };  // X_c[k]
            auto Xm = [&](int c, int k) { return csub(buf[c * STRIDE + k], buf[c * STRIDE + 64 + k]); };  // X_c[64 + k]
            const int j = tg & 31, h = tg >> 5;
            const int cA = j, cB = (j == 0) ? 32 : 64 - j;
            const bool dc = (j == 0);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int k2 = 16 * h + i;                  // < 64: bins cA + 64 k2 <= N/2
                const float2 za = Xp(cA, k2);
                // partner N - k: column cB, index 127 - k2 (DC column: column 0, index 128 - k2)
                const float2 zbA = dc ? (k2 == 0 ? Xp(0, 0) : Xm(0, 64 - k2)) : Xm(cB, 63 - k2);
                on_bin(i, cA + 64 * k2, za, zbA, true);
                const float2 zb2 = Xp(cB, k2);
                const float2 zbB = dc ? Xm(32, 63 - k2) : Xm(cA, 63 - k2);
                on_bin(16 + i, cB + 64 * k2, zb2, zbB, true);
            }
            const float2 zn = Xm(0, 0);                     // column 0, k2 = 64: Nyquist
            on_bin(NB - 1, N / 2, zn, zn, tg == 0);
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
        float2* trow = (MODE == kModeForward) ? a.T + fi * a.ldT : nullptr;
        if constexpr (STORE) {
            // a6 as exact fixed-point integer sums with native shared-memory integer atomics
            // (float atomics on shared memory are compare-and-swap loops on sm_100a).  Per warp and
            // tile, v_max bounds the kept |Re S|, |Im S|; every value is scaled by 2^(39 - e)
            // (v_max < 2^e, a power of two: exact) and rounded to a 64-bit integer X, |X| < 2^39, which
            // is added as two 32-bit limbs hi = X >> 20 (signed) and lo = X & (2^20 - 1).  With at
            // most K <= 2049 contributions per target the limb sums cannot overflow
            // (sum|hi| < 2^30.01, sum lo < 2^31.01): the integer sum is exact whatever the order (quantum
            // v_max 2^-39), so the band value is bitwise reproducible.
            // N2 = 64: each of the frame's two warps squeezes into its own half of the group buffer.
            constexpr int WPG = (N2 > 32) ? N2 / 32 : 1;   // warps per group
            // band bins per pass (4 int32 each); groups sharing a warp offset their planes by up to
            // 28 ints so that the warp's 32-bit accesses spread over the banks
            constexpr int CH = ((N2 < 32 ? 2 * CAP - 32 : 2 * CAP) / 4 / WPG) & ~3;
            static_assert(CH % 4 == 0 && CH > 0, "int4 zeroing");
            const int lane = threadIdx.x & 31;
            const int wib = (WPG > 1) ? (tg >> 5) : 0;     // warp within the group
            const int ebank = (N2 < 32) ? ((32 - ((lane / N2) * N2) % 32) % 32) & ~3 : 0;
            int* acc = reinterpret_cast<int*>(buf) + ebank + wib * 4 * CH;   // planar [hi_re|lo_re|hi_im|lo_im][CH]
            __shared__ float wscale[TPB / 32];
            float vmax = 0.0f;
#pragma unroll
            for (int i = 0; i < NB; ++i)
                if (bl[i] >= 0) vmax = fmaxf(vmax, fmaxf(fabsf(bsr[i]), fabsf(bsi[i])));
            const unsigned vb = __reduce_max_sync(0xffffffffu, __float_as_uint(vmax));
            const int ex = max(-87, (int)((vb >> 23) & 0xff) - 126);   // v_max < 2^ex
            const float scale = __uint_as_float((unsigned)(127 + 39 - ex) << 23);
            const float iscale = __uint_as_float((unsigned)(127 - 39 + ex) << 23);
            if (WPG > 1 && lane == 0) wscale[threadIdx.x >> 5] = iscale;
            for (int l0 = 0; l0 < a.bins; l0 += CH) {
                const int lc = min(CH, a.bins - l0);
                {
                    int4* z4 = reinterpret_cast<int4*>(reinterpret_cast<int*>(buf) + ebank);
                    const int lc4 = (lc + 3) >> 2;
#pragma unroll
                    for (int q = 0; q < 4 * WPG; ++q)
                        for (int i = tg; i < lc4; i += N2) z4[q * (CH / 4) + i] = make_int4(0, 0, 0, 0);
                }
                group_sync<N2>(group);
#pragma unroll
                for (int i = 0; i < NB; ++i) {
                    const int lr = bl[i] - l0;
                    const bool in = bl[i] >= 0 && lr >= 0 && lr < lc;
                    if (!__any_sync(0xffffffffu, in)) continue;      // warp-uniform: nothing lands here
                    // lanes hitting the same target (a ridge's run of source bins) are serialised by the
                    // shared-memory atomic unit; a warp scan merging runs first measured slower
                    const float vr = bsr[i] * scale, vi = bsi[i] * scale;
                    if (in) {                                         // a6: T_acc[l] += S (Eq. 27/28)
                        // volatile: keep the conversions inside this rarely-taken branch
                        long long xr, xi;
                        asm volatile("cvt.rni.s64.f32 %0, %1;" : "=l"(xr) : "f"(vr));
                        asm volatile("cvt.rni.s64.f32 %0, %1;" : "=l"(xi) : "f"(vi));
                        atomicAdd(acc + lr, (int)(xr >> 20));
                        atomicAdd(acc + CH + lr, (int)(xr & 0xFFFFF));
                        atomicAdd(acc + 2 * CH + lr, (int)(xi >> 20));
                        atomicAdd(acc + 3 * CH + lr, (int)(xi & 0xFFFFF));
                    }
                }
                group_sync<N2>(group);
                if (valid)
                    for (int i = tg; i < lc; i += N2) {
                        const int* a0 = reinterpret_cast<const int*>(buf) + ebank;
                        float2 t;
                        if constexpr (WPG > 1) {
                            const int w0 = (threadIdx.x >> 5) - wib;   // first warp of this group
                            float sr = 0.0f, si = 0.0f;
#pragma unroll
                            for (int h = 0; h < WPG; ++h) {
                                const int* ah = a0 + h * 4 * CH;
                                const float is = wscale[w0 + h];
                                sr += limbs_to_float(ah[i], ah[CH + i], is);
                                si += limbs_to_float(ah[2 * CH + i], ah[3 * CH + i], is);
                            }
                            t = make_float2(sr, si);
                        } else {
                            t = make_float2(limbs_to_float(a0[i], a0[CH + i], iscale),
                                            limbs_to_float(a0[2 * CH + i], a0[3 * CH + i], iscale));
                        }
                        trow[l0 + i] = t;
                    }
                group_sync<N2>(group);
            }
        }
        __syncthreads();   // tile input buffer and group buffers free for the next tile
    }

    if constexpr (MODE == kModeAbsmax) {
        // block max of 4|S|^2 -> |S|
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
        __shared__ float red[TPB / 32];
        __syncthreads();
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = vmax;
        __syncthreads();
        if (threadIdx.x == 0) {
            float m = 0.0f;
            for (int w = 0; w < TPB / 32; ++w) m = fmaxf(m, red[w]);
            atomicMax(reinterpret_cast<unsigned int*>(a.absmax_out), __float_as_uint(0.5f * sqrtf(m)));
        }
    }
}

// ------------------------------------------------------------------------------- inverse ------
// 1/(C d[s]) given r = (s + c) mod hop
__device__ __forceinline__ float inv_norm_r(int64_t s, int r, const InvArgs& a) {
    if (s < a.n_head) return __ldg(a.inv_head + s);
    if (s >= a.n - a.n_tail) return __ldg(a.inv_tail + (s - (a.n - a.n_tail)));
    return __ldg(a.inv_per + r);
}

__device__ __forceinline__ float inv_norm(int64_t s, const InvArgs& a) {
    if (s < a.n_head) return __ldg(a.inv_head + s);
    if (s >= a.n - a.n_tail) return __ldg(a.inv_tail + (s - (a.n - a.n_tail)));
    return __ldg(a.inv_per + (int)((s + a.c) % a.hop));
}

// Work item = (frame pair, residue b).  A tile holds P = max(1, G/z) consecutive frame pairs, so
// its P z items occupy the G groups in ceil(P z / G) passes (one pass for every config here).
// Per item the group computes V_b = IDFT_N of the Hermitian-packed sub-spectrum
// G_b[q] = H_A[z q + b] + i H_B[z q + b] and leaves e^{i 2 pi b tau/(z N)} V_b[p] in its buffer
// (indexed by p = tau mod N).  The CTA then sums the items of each pair over b, windows by
// g[tau + c]/N and adds frame A (real part) and frame B (imaginary part) into the OLA ring.
// RM: every nonzero sub-spectrum entry q (band [k1, k2) or mirror [N - k2, N)) has
// q / N2 in [0, RM) or [64 - RM, 64) (i.e. ceil(k2 / N2) <= RM): other rows of the step-1
// input are compile-time zeros and cost nothing (narrow bands: C2, C3 use RM = 5, C4 RM = 8).
template <int N2, bool FULLWIN, int RM>
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
            float2 v[64];
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
                if ((inb || inm) && vA) ta = __ldg(TA + li);
                if ((inb || inm) && vB) tb = __ldg(TB + li);
                if (n1 == 0 && q == 0 && b == 0) { ta.y = 0.0f; tb.y = 0.0f; }  // DC: real part only (R14)
                if (n1 == 32 && q == N / 2 && b == 0) { ta.y = 0.0f; tb.y = 0.0f; }   // Nyquist (full band only)
                v[n1] = inb ? make_float2(ta.x - tb.y, ta.y + tb.x)    // H_A + i H_B
                            : make_float2(ta.x + tb.y, tb.x - ta.y);   // conj H_A + i conj H_B
            }
            if constexpr (RM < 32) FftSparse64<+1, RM>::run(v);   // zero rows skipped
            else Fft<64, +1>::run(v);
#pragma unroll
            for (int kk = 0; kk < 64; ++kk) {
                float2 t = v[kk];
                if (kk != 0) t = cmulc(t, __ldg(a.tw + kk * N2 + tg));   // W_N^{-tg kk}
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
#pragma unroll
                    for (int k2 = 0; k2 < N2; ++k2) {
                        const int p = col + 64 * k2;                  // output index tau mod N
                        float2 y = u[ci][k2];
                        if constexpr (FULLWIN) {
                            // tau = p (k2 < N2/2) or p - N: compile-time split; e(b tau) = e(b col) e(b (64 k2 [- N]))
                            if (rot) y = cmul(y, cmul(fb, __ldg(pb + 64 + (k2 < N2 / 2 ? 0 : N2) + k2)));
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
                    if (slot[jj] >= 0) ring[slot[jj]] += y[jj].x;
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
                a.seam[((int64_t)blockIdx.x * 2 + 0) * a.seam_len + (s - g_lo)] = val;
            } else if (!last_cta && s >= right_start) {
                a.seam[((int64_t)blockIdx.x * 2 + 1) * a.seam_len + (s - right_start)] = val;
            } else if (a.normalize) {
                // (a per-sample 32-bit mod_pos here measured 4 % slower on C4: one more live register)
                a.y[s - a.y_off] = val * inv_norm(s, a) * a.out_scale;
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
        if (a.normalize) a.y[s - a.y_off] = val * inv_norm(s, a) * a.out_scale;
        else             a.y[s - a.y_off] += val;
    }
}

__global__ void finalize_kernel(float* y, int64_t y_off, int64_t y_len, InvArgs a) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    // r = (s + c) mod hop, advanced incrementally (one 64-bit modulo per thread)
    int r = (int)(((y_off + i + a.c) % a.hop + a.hop) % a.hop);
    const int step = (int)(stride % a.hop);
    for (; i < y_len; i += stride) {
        const int64_t s = y_off + i;
        if (s >= 0 && s < a.n) y[i] *= inv_norm_r(s, r, a) * a.out_scale;
        r += step;
        r -= (r >= a.hop) ? a.hop : 0;
    }
}

// ------------------------------------------------------------------------------- launchers ----
template <int N2, int MODE, bool BIG, bool FULLWIN>
static cudaError_t launch_fwd_b(const FwdArgs& a, int grid, cudaStream_t s) {
    auto kern = fwd_kernel<N2, MODE, BIG, FULLWIN>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, a.lay.total);
    if (e != cudaSuccess) return e;
    kern<<<grid, Geom<N2, true>::TPB, a.lay.total, s>>>(a);
    return cudaGetLastError();
}

template <int N2, int MODE, bool BIG>
static cudaError_t launch_fwd_w(const FwdArgs& a, int grid, cudaStream_t s) {
    if (a.L == Geom<N2, true>::N && a.c == Geom<N2, true>::N / 2) return launch_fwd_b<N2, MODE, BIG, true>(a, grid, s);
    return launch_fwd_b<N2, MODE, BIG, false>(a, grid, s);
}

template <int N2, int MODE>
static cudaError_t launch_fwd_t(const FwdArgs& a, int grid, cudaStream_t s) {
    if constexpr (MODE == kModeForward && N2 <= 32) {
        if (a.bins > Geom<N2, true>::CAP) return launch_fwd_w<N2, MODE, true>(a, grid, s);
    }
    return launch_fwd_w<N2, MODE, false>(a, grid, s);
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
        case 128: if constexpr (SST_HAS(2)) return launch_fwd_mode<2>(a, mode, grid, s); break;
        case 256: if constexpr (SST_HAS(4)) return launch_fwd_mode<4>(a, mode, grid, s); break;
        case 512: if constexpr (SST_HAS(8)) return launch_fwd_mode<8>(a, mode, grid, s); break;
        case 1024: if constexpr (SST_HAS(16)) return launch_fwd_mode<16>(a, mode, grid, s); break;
        case 2048: if constexpr (SST_HAS(32)) return launch_fwd_mode<32>(a, mode, grid, s); break;
        case 4096: if constexpr (SST_HAS(64)) return launch_fwd_mode<64>(a, mode, grid, s); break;
        case 8192: if constexpr (SST_HAS(128)) return launch_fwd_mode<128>(a, mode, grid, s); break;
    }
    return cudaErrorInvalidValue;
}

template <int N2>
static int occ_fwd(int L, int H, int device) {
    int nb = 0, sms = 0;
    const int smem = fwd_layout(N2, L, H).total;
    auto kern = fwd_kernel<N2, kModeForward, false, true>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, Geom<N2, true>::TPB, smem);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    return (nb > 0 ? nb : 1) * sms;
}

int forward_max_grid(int nfft, int L, int H, int device) {
    switch (nfft) {
        case 128: if constexpr (SST_HAS(2)) return occ_fwd<2>(L, H, device); break;
        case 256: if constexpr (SST_HAS(4)) return occ_fwd<4>(L, H, device); break;
        case 512: if constexpr (SST_HAS(8)) return occ_fwd<8>(L, H, device); break;
        case 1024: if constexpr (SST_HAS(16)) return occ_fwd<16>(L, H, device); break;
        case 2048: if constexpr (SST_HAS(32)) return occ_fwd<32>(L, H, device); break;
        case 4096: if constexpr (SST_HAS(64)) return occ_fwd<64>(L, H, device); break;
        case 8192: if constexpr (SST_HAS(128)) return occ_fwd<128>(L, H, device); break;
    }
    return -1;
}

template <int N2, bool FULLWIN, int RM>
static cudaError_t launch_inv_b(const InvArgs& a, int grid, cudaStream_t s) {
    auto kern = inv_kernel<N2, FULLWIN, RM>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, a.lay.total);
    if (e != cudaSuccess) return e;
    kern<<<grid, Geom<N2, false>::TPB, a.lay.total, s>>>(a);
    return cudaGetLastError();
}

template <int N2, bool FULLWIN>
static cudaError_t launch_inv_r(const InvArgs& a, int grid, cudaStream_t s) {
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

cudaError_t launch_inverse(const InvArgs& a, int grid, cudaStream_t s) {
    switch (a.nfft) {
        case 128: if constexpr (SST_HAS(2)) return launch_inv_t<2>(a, grid, s); break;
        case 256: if constexpr (SST_HAS(4)) return launch_inv_t<4>(a, grid, s); break;
        case 512: if constexpr (SST_HAS(8)) return launch_inv_t<8>(a, grid, s); break;
        case 1024: if constexpr (SST_HAS(16)) return launch_inv_t<16>(a, grid, s); break;
        case 2048: if constexpr (SST_HAS(32)) return launch_inv_t<32>(a, grid, s); break;
        case 4096: if constexpr (SST_HAS(64)) return launch_inv_t<64>(a, grid, s); break;
        case 8192: if constexpr (SST_HAS(128)) return launch_inv_t<128>(a, grid, s); break;
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_inverse_seams(const InvArgs& a, int ctas, cudaStream_t s) {
    if (ctas < 2 || a.seam_len <= 0) return cudaSuccess;
    const int64_t total = (int64_t)(ctas - 1) * a.seam_len;
    const int threads = 256;
    const int64_t want = (total + threads - 1) / threads;
    const int blocks = (int)(want < 4096 ? want : 4096);
    seam_kernel<<<blocks, threads, 0, s>>>(a, ctas);
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
                            const float* inv_per, float out_scale, cudaStream_t s) {
    InvArgs a{};
    a.out_scale = out_scale;
    a.n = n; a.hop = hop; a.c = c;
    a.inv_head = inv_head; a.n_head = n_head; a.inv_tail = inv_tail; a.n_tail = n_tail; a.inv_per = inv_per;
    const int threads = 256;
    const int64_t want = (y_len + threads - 1) / threads;
    const int blocks = (int)(want < 2368 ? want : 2368);
    if (blocks <= 0) return cudaSuccess;
    finalize_kernel<<<blocks, threads, 0, s>>>(y, y_off, y_len, a);
    return cudaGetLastError();
}

template <int N2>
static int occ_inv(int hop, int L, int zoom, int device) {
    int nb = 0, sms = 0;
    const int smem = inv_layout(N2, L, hop, zoom).total;
    auto kern = inv_kernel<N2, true, 64>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, Geom<N2, false>::TPB, smem);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    return (nb > 0 ? nb : 1) * sms;
}

int inverse_max_grid(int nfft, int hop, int L, int zoom, int device) {
    switch (nfft) {
        case 128: if constexpr (SST_HAS(2)) return occ_inv<2>(hop, L, zoom, device); break;
        case 256: if constexpr (SST_HAS(4)) return occ_inv<4>(hop, L, zoom, device); break;
        case 512: if constexpr (SST_HAS(8)) return occ_inv<8>(hop, L, zoom, device); break;
        case 1024: if constexpr (SST_HAS(16)) return occ_inv<16>(hop, L, zoom, device); break;
        case 2048: if constexpr (SST_HAS(32)) return occ_inv<32>(hop, L, zoom, device); break;
        case 4096: if constexpr (SST_HAS(64)) return occ_inv<64>(hop, L, zoom, device); break;
        case 8192: if constexpr (SST_HAS(128)) return occ_inv<128>(hop, L, zoom, device); break;
    }
    return -1;
}

}  // namespace sst
