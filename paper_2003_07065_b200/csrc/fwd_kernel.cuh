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

#pragma once

#include "common.cuh"

namespace sst {

// ------------------------------------------------------------------------------- forward ------
// Tile t of a CTA covers frames [fb + t G, fb + t G + G) and input samples [s_lo, s_hi).  It is
// fetched with one bulk copy when the 16-byte aligned span lies inside the valid x slice;
// otherwise (record / slice edges, misaligned x) the CTA loads it cooperatively with zero fill.
struct TileIn {
    int64_t s_lo, a_lo;   // first sample; first copied x index (aligned)
    int pad, bytes;       // s_lo - (x_off + a_lo); bytes of the bulk copy
    bool bulk;
};

// frames [f, f + g) (global indices) of one tile
__device__ __forceinline__ TileIn tile_in(const FwdArgs& a, int64_t f, int g, bool x_aligned) {
    TileIn ti;
    ti.s_lo = f * a.hop - a.c;
    const int64_t s_hi = (f + g - 1) * a.hop - a.c + a.L;
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
    constexpr bool KEEPL = (MODE == kModeForward || MODE == kModeTargets);   // targets kept in registers
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ float wnrm[TPB / 32];               // per-warp ||z_m||^2 partials (groups of > 1 warp)
    __shared__ unsigned cq_n;                      // R23 deferral: entries this CTA queued
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
    // list mode (R23 repair): tile t is the single frame flist[t] (group 0), inline re-decision
    // list mode (R23 repair): tile t holds the frames flist[t G .. t G + G) (within the launch, one per
    // group), gathered straight from global memory (bounds-checked); inline re-decision
    const bool lmode = a.flist != nullptr;
    const int64_t nlist = lmode ? (int64_t)*a.flist_n : 0;
    const int64_t ntiles = lmode ? (nlist + G - 1) / G : (nfr + G - 1) / G;
    const int64_t v_lo_x = a.x_off > 0 ? a.x_off : 0;
    const int64_t v_hi_x = min(a.n, a.x_off + a.x_len);
    auto xglob = [&](int64_t frame, int j) -> float {           // sample j of frame (within the launch)
        const int64_t sj = (a.frame_begin + frame) * a.hop - a.c + j;
        return (sj >= v_lo_x && sj < v_hi_x) ? __ldg(a.x + (sj - a.x_off)) : 0.0f;
    };
    const int64_t tiles_per_cta = (ntiles + gridDim.x - 1) / gridDim.x;
    const int64_t t_begin = (int64_t)blockIdx.x * tiles_per_cta;
    const int64_t t_end = min(ntiles, t_begin + tiles_per_cta);
    const int last_in = a.L - 1 - a.c;             // largest tau
    const bool x_aligned = (reinterpret_cast<uintptr_t>(a.x) & 15) == 0;
    float vmax = 0.0f;

    for (int i = threadIdx.x; i < a.L; i += TPB) taps_s[i] = __ldg(a.taps + i);
    if (threadIdx.x == 0) {
        cq_n = 0;
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0 && t_begin < t_end && !lmode) {
        const TileIn ti = tile_in(a, a.frame_begin + t_begin * G, G, x_aligned);
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
        if (threadIdx.x == 0 && tile + 1 < t_end && !lmode) {
            const TileIn tn = tile_in(a, a.frame_begin + (tile + 1) * G, G, x_aligned);
            if (tn.bulk) {
                fence_proxy_async();
                mbar_arrive_tx(&mbar[bsel ^ 1], tn.bytes);
                bulk_g2s(xbuf + (bsel ^ 1) * a.lay.xcap, a.x + tn.a_lo, tn.bytes, &mbar[bsel ^ 1]);
            }
        }
        const TileIn ti = tile_in(a, a.frame_begin + tile * G, G, x_aligned);
        int pad = ti.pad;
        if (lmode) {
            pad = 0;
        } else if (ti.bulk) {
            mbar_wait(&mbar[bsel], (phase >> bsel) & 1);
            phase ^= 1u << bsel;
        } else {
            const int64_t v_lo = a.x_off > 0 ? a.x_off : 0;
            const int64_t v_hi = min(a.n, a.x_off + a.x_len);
            const int span = (G - 1) * a.hop + a.L;
            for (int i = threadIdx.x; i < span; i += TPB) {
                const int64_t s = ti.s_lo + i;
                SST_CHECK(i < a.lay.xcap && (s < v_lo || s >= v_hi || (s - a.x_off >= 0 && s - a.x_off < a.x_len)));
                xb[i] = (s >= v_lo && s < v_hi) ? __ldg(a.x + (s - a.x_off)) : 0.0f;
            }
            pad = 0;
            __syncthreads();
        }

        const int64_t li = tile * G + group;
        const int64_t fi = lmode ? (li < nlist ? (int64_t)__ldg(a.flist + li) : nfr) : li;   // frame within the launch
        const bool valid = fi < nfr;
        const float* xw = xb + pad + group * a.hop; // x[m H - c + j], j = 0..L-1 (j = tau + c)

        // ---- a1: gather + pack (circular placement), a2 step 1: 64-point DFT of row tg
        float2 v[64];
        float2 nacc = make_float2(0.0f, 0.0f);          // ||z_m||^2 partial (R23 margins)
        if (lmode) {
#pragma unroll
            for (int n1 = 0; n1 < 64; ++n1) {
                const int n = N2 * n1 + tg;
                const int j = ((n <= last_in) ? n : n - N) + a.c;
                float2 val = make_float2(0.0f, 0.0f);
                if (j >= 0 && valid) val = cscale(taps_s[j], xglob(fi, j));
                v[n1] = val;
                if constexpr (KEEPL) nacc = __ffma2_rn(val, val, nacc);
            }
        } else if constexpr (FULLWIN) {
            const float* xt = xw + tg;
            const float2* wt = taps_s + tg;
#pragma unroll
            for (int n1 = 0; n1 < 64; ++n1) {
                const int j = N2 * n1 + (n1 < 32 ? N / 2 : -N / 2);   // tau + c - tg (compile time)
                v[n1] = cscale(wt[j], xt[j]);
                if constexpr (KEEPL) nacc = __ffma2_rn(v[n1], v[n1], nacc);
            }
        } else {
#pragma unroll
            for (int n1 = 0; n1 < 64; ++n1) {
                const int n = N2 * n1 + tg;
                const int j = ((n <= last_in) ? n : n - N) + a.c;
                float2 val = make_float2(0.0f, 0.0f);
                if (j >= 0) val = cscale(taps_s[j], xw[j]);
                v[n1] = val;
                if constexpr (KEEPL) nacc = __ffma2_rn(val, val, nacc);
            }
        }
        float nrm2 = 0.0f;
        if constexpr (KEEPL) {
            nrm2 = nacc.x + nacc.y;
#pragma unroll
            for (int o = (N2 < 32 ? N2 : 32) / 2; o > 0; o >>= 1) nrm2 += __shfl_xor_sync(0xffffffffu, nrm2, o);
            if constexpr (N2 > 32) {
                if ((threadIdx.x & 31) == 0) wnrm[threadIdx.x >> 5] = nrm2;
            }
        }
        Fft<64, -1>::run(v);
#pragma unroll
        for (int k1 = 0; k1 < 64; ++k1) {
            float2 t = v[k1];
            if (k1 != 0) t = cmul(t, __ldg(a.tw + k1 * N2 + tg));   // W_N^{tg k1}, lane-contiguous
            SST_CHECK(k1 * STRIDE + tg < CAP);
            buf[k1 * STRIDE + tg] = t;
        }
        group_sync<N2>(group);

        // ---- a2 step 2 + a3 unpack + a4/a5 per bin
        // forward: bins are computed branch-free into registers (phase 1), then squeezed with
        // predicated shared-memory atomics in chunks of CAP bins (phase 2; one chunk unless BIG)
        constexpr bool STORE = (MODE == kModeForward);
        int bl[KEEPL ? NB : 1];
        float bsr[STORE ? NB : 1], bsi[STORE ? NB : 1];
        unsigned long long uns = 0ull;                 // R23: bit idx = bin idx needs the fp64 decision
        float cm = 0.0f, km = -1.0f;
        if constexpr (KEEPL) {
            if constexpr (N2 > 32) {
                nrm2 = 0.0f;
                const int w0 = (threadIdx.x >> 5) & ~(N2 / 32 - 1);
#pragma unroll
                for (int h = 0; h < N2 / 32; ++h) nrm2 += wnrm[w0 + h];
            }
            fwd_margins(a, gam4, nrm2, cm, km);
        }
        auto on_bin = [&](int idx, int k, float2 za, float2 zb, bool ok) {
            float2 PQ, UV;
            float mag4;
            bool unsure;
            int l = bin_target(a, gam4, cm, km, k, za, zb, PQ, UV, mag4, unsure);
            if (!ok || !valid) { l = -3; unsure = false; }
            if constexpr (KEEPL) {
                bl[idx] = l;
                if (unsure) uns |= 1ull << idx;
            }
            if constexpr (STORE) {
                const float2 S = cscale(PQ, 0.5f);
                bsr[idx] = S.x;
                bsi[idx] = S.y;
            } else if constexpr (MODE == kModeStft) {
                if (l != -3) {
                    const int64_t o = fi * (int64_t)(N / 2 + 1) + k;
                    a.S[o] = cscale(PQ, 0.5f);
                    a.Sd[o] = __fmul2_rn(UV, make_float2(a.inv_alpha2, -a.inv_alpha2));
                }
            } else if constexpr (MODE == kModeAbsmax) {
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

        // ---- R23: bins whose fp32 decision the FFT error could have moved are re-decided in fp64
        // (direct Eq. 8 sum over the tile's input in shared memory), one warp-cooperative sum each
        if constexpr (KEEPL) {
            auto bin_k = [&](int i) -> int {               // source bin of register slot i (see on_bin)
                if (i == NB - 1) return N / 2;
                if constexpr (N2 <= 32) {
                    const int u = i / N2, r = i % N2;
                    const int j = tg + N2 * u;
                    return r < N2 / 2 ? j + 64 * r : ((j == 0) ? 32 : 64 - j) + 64 * (r - N2 / 2);
                } else {
                    const int j = tg & 31, h = tg >> 5;
                    return i < 16 ? j + 64 * (16 * h + i) : ((j == 0) ? 32 : 64 - j) + 64 * (16 * h + i - 16);
                }
            };
            // Deferred (the common path): the flagged bins stay squeezed at their fp32 targets and are
            // queued in this CTA's region of the queue (shared-memory index) for redecide_kernel; no CTA
            // barrier here, so warps keep their own pace through the tile.  Inline fallback (region full,
            // or the list-mode repair launch): one warp-uniform loop per warp with a single copy of the
            // warp-cooperative fp64 sum.
            unsigned long long my = uns;
            if (a.gq && my) {
                const unsigned reg = a.gq_cap / gridDim.x;
                int4* cq = a.gq + (size_t)blockIdx.x * reg;
#pragma unroll 1
                while (my) {
                    const int i = __ffsll((long long)my) - 1;
                    int li = 0;
#pragma unroll
                    for (int ii = 0; ii < NB; ++ii) li = (ii == i) ? bl[ii] : li;
                    const unsigned q = atomicAdd(&cq_n, 1u);
                    if (q >= reg) break;                               // region full: inline below
                    SST_CHECK((size_t)blockIdx.x * reg + q < a.gq_cap && fi < nfr);
                    cq[q] = make_int4((int)fi, bin_k(i), li, 0);
                    my &= my - 1;
                }
            }
            if (__any_sync(0xffffffffu, my != 0ull)) {
                const double gam64 = launch_gamma64(a);
                const int lane = threadIdx.x & 31;
                const int wbase = threadIdx.x & ~31;
#pragma unroll 1
                while (true) {
                    const unsigned ball = __ballot_sync(0xffffffffu, my != 0ull);
                    if (!ball) break;
                    const int src = __ffs(ball) - 1;
                    const int i = __ffsll((long long)__shfl_sync(0xffffffffu, my, src)) - 1;
                    if (lane == src) my &= my - 1;
                    const int k = __shfl_sync(0xffffffffu, bin_k(i), src);
                    const float* xs = xb + pad + ((wbase + src) / N2) * a.hop;
                    const int64_t fsrc = __shfl_sync(0xffffffffu, fi, src);
                    double sr, si, dr, di;
                    stft_bin_fp64([&](int j) { return lmode ? xglob(fsrc, j) : xs[j]; }, a.taps64, a.tw64, N, a.L,
                                  a.c, k, sr, si, dr, di);
                    const int ln = decide_fp64(a, gam64, k, sr, si, dr, di);
                    if (lane == 0 && !lmode) atomicAdd(a.r23_count, 1ull);
#pragma unroll
                    for (int ii = 0; ii < NB; ++ii)
                        if (lane == src && ii == i) {
                            if (bl[ii] != ln && !lmode) atomicAdd(a.r23_count + 1, 1ull);
                            bl[ii] = ln;
                        }
                }
            }
            if constexpr (MODE == kModeTargets) {
#pragma unroll
                for (int i = 0; i < NB; ++i)
                    if (bl[i] != -3) {
                        SST_CHECK(fi < nfr && bin_k(i) <= N / 2);
                        a.lout[fi * (int64_t)(N / 2 + 1) + bin_k(i)] = bl[i];
                    }
            }
        }

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
            // planar [hi_re|lo_re|hi_im|lo_im][CH], or (IL: the dense bands of the BIG path, whose
            // zeroing and readout of CH bins per pass bound it on the L1/shared pipe) interleaved
            // [CH][re, im] with ONE int32 limb per component: at most K = N/2 + 1 <= 2^KB - 1 sources
            // land on a target, so with |X| <= 2^QB, QB = 31 - KB, the int32 sum cannot overflow and
            // is still exact and order-free (quantum v_max 2^-QB instead of 2^-39: C5 2^-22, far
            // below the north star's 1e-3 relative L2); half the bytes of four limbs per bin
            constexpr bool IL = BIG && WPG == 1;
            constexpr int KB = ceil_log2_c(N / 2 + 2);     // 2^KB - 1 >= N/2 + 1
            constexpr int QB = IL ? 31 - KB : 39;
            constexpr int LPB = IL ? 2 : 4;                 // int32 limbs per bin
            // band bins per pass; groups sharing a warp offset their planes by up to 28 ints so that
            // the warp's 32-bit accesses spread over the banks
            constexpr int CH = ((N2 < 32 ? 2 * CAP - 32 : 2 * CAP) / LPB / WPG) & ~3;
            static_assert(CH % 4 == 0 && CH > 0, "int4 zeroing");
            const int lane = threadIdx.x & 31;
            const int wib = (WPG > 1) ? (tg >> 5) : 0;     // warp within the group
            // (IL: 8-byte bins; group buffers start CAP float2 = 16 banks (mod 32) apart, so the groups of a
            // half-warp already read disjoint banks in the readout -- an offset would make them collide)
            const int ebank = (N2 < 32 && !IL) ? ((32 - ((lane / N2) * N2) % 32) % 32) & ~3 : 0;
            int* acc = reinterpret_cast<int*>(buf) + ebank + wib * 4 * CH;
            __shared__ float wscale[TPB / 32];
            float vmax = 0.0f;
#pragma unroll
            for (int i = 0; i < NB; ++i)
                if (bl[i] >= 0) vmax = fmaxf(vmax, fmaxf(fabsf(bsr[i]), fabsf(bsi[i])));
            const unsigned vb = __reduce_max_sync(0xffffffffu, __float_as_uint(vmax));
            const int ex = max(-87, (int)((vb >> 23) & 0xff) - 126);   // v_max < 2^ex
            const float scale = __uint_as_float((unsigned)(127 + QB - ex) << 23);
            const float iscale = __uint_as_float((unsigned)(127 - QB + ex) << 23);
            if (WPG > 1 && lane == 0) wscale[threadIdx.x >> 5] = iscale;
            for (int l0 = 0; l0 < a.bins; l0 += CH) {
                const int lc = min(CH, a.bins - l0);
                {
                    int4* z4 = reinterpret_cast<int4*>(reinterpret_cast<int*>(buf) + ebank);
                    if constexpr (IL) {
                        // (clearing on read in the readout instead, zeroing only before the first pass,
                        // measured slower: C5 26.98 -> 28.59 ms per 2^24 samples)
                        for (int i = tg; i < (lc + 1) >> 1; i += N2) z4[i] = make_int4(0, 0, 0, 0);
                    } else {
                        const int lc4 = (lc + 3) >> 2;
#pragma unroll
                        for (int q = 0; q < 4 * WPG; ++q)
                            for (int i = tg; i < lc4; i += N2) z4[q * (CH / 4) + i] = make_int4(0, 0, 0, 0);
                    }
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
                        if constexpr (IL) {
                            int xr, xi;
                            asm volatile("cvt.rni.s32.f32 %0, %1;" : "=r"(xr) : "f"(vr));
                            asm volatile("cvt.rni.s32.f32 %0, %1;" : "=r"(xi) : "f"(vi));
                            SST_CHECK(lr >= 0 && lr < CH && (int)(acc - reinterpret_cast<int*>(buf)) + 2 * lr + 1 < 2 * CAP);
                            atomicAdd(acc + 2 * lr, xr);
                            atomicAdd(acc + 2 * lr + 1, xi);
                        } else {
                            long long xr, xi;
                            asm volatile("cvt.rni.s64.f32 %0, %1;" : "=l"(xr) : "f"(vr));
                            asm volatile("cvt.rni.s64.f32 %0, %1;" : "=l"(xi) : "f"(vi));
                            SST_CHECK(lr >= 0 && lr < CH && (int)(acc - reinterpret_cast<int*>(buf)) + 3 * CH + lr < 2 * CAP);
                            atomicAdd(acc + lr, (int)(xr >> 20));
                            atomicAdd(acc + CH + lr, (int)(xr & 0xFFFFF));
                            atomicAdd(acc + 2 * CH + lr, (int)(xi >> 20));
                            atomicAdd(acc + 3 * CH + lr, (int)(xi & 0xFFFFF));
                        }
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
                        } else if constexpr (IL) {
                            // (two bins per lane with 16-byte loads and stores measured slower: C5
                            // forward 21.37 -> 22.12 ms per 2^24 samples)
                            const int2 v = reinterpret_cast<const int2*>(a0)[i];
                            t = make_float2((float)v.x * iscale, (float)v.y * iscale);
                        } else {
                            t = make_float2(limbs_to_float(a0[i], a0[CH + i], iscale),
                                            limbs_to_float(a0[2 * CH + i], a0[3 * CH + i], iscale));
                        }
                        SST_CHECK(fi < nfr && l0 + i < a.bins);
                        __stcs(trow + l0 + i, t);           // streaming: T is written once, read by the inverse later
                    }
                group_sync<N2>(group);
            }
        }
        __syncthreads();   // tile input buffer and group buffers free for the next tile
    }

    if constexpr (KEEPL) {
        if (a.gq) {
            __syncthreads();
            if (threadIdx.x == 0) a.gq_counts[blockIdx.x] = min(cq_n, a.gq_cap / gridDim.x);
        }
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

}  // namespace sst
