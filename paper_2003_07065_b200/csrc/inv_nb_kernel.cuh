// Narrow-band inverse kernel (rows a9-a10 of DESIGN.md §1) for full windows and bands whose
// sub-spectrum rows fit RM <= 8 of 64 (C2, C3).  Same result as inv_kernel.cuh (Eq. 25-26, P:L182,
// P:L186); a different factorisation of the z N_f-point band IDFT:
//
//   j = J j_hi + j_lo (J = z N2, j_hi in [0, 64)),  tau = tau_lo + 64 tau_hi (tau_lo in [0, 64))
//   stage 1, per column j_lo:  P[j_lo][tau_lo] = e(j_lo tau_lo) sum_{j_hi} G[J j_hi + j_lo] e^{i 2 pi j_hi tau_lo / 64}
//   stage 2, per row tau_lo:   Y[tau] = sum_b e^{i 2 pi b tau_hi / J} sum_t P[z t + b][tau_lo] e^{i 2 pi t tau_hi / N2}
//
// with e(x) = e^{i 2 pi x / (z N)} and G = H_A + i H_B the Hermitian-packed spectra of a frame pair.
// One CTA of J threads owns a contiguous frame range and walks it a pair at a time.  Stage 1: thread
// t = column j_lo holds its 2 RM nonzero inputs (the band and mirror rows) in registers and computes
// the 64 outputs chunk by chunk (N2 of the 64 rows per chunk, an 8 x 8 DIT composite whose first
// 8-point sums run over the nonzero rows only), into a shared chunk buffer.  Stage 2: thread
// (row, b) runs the N2-point DFT of residue b, multiplies by e(b tau), and the z threads of a row
// sum over b by a reduce-scatter of warp shuffles, so each ends with N2/z finished outputs that it
// windows and overlap-adds into the CTA's OLA ring (frame A = real part, frame B = imaginary part,
// two barrier-separated phases).  The sum over residues never touches shared memory, which is
// where the residue-split kernel spends a 2 x 16 KB round trip per item.
#pragma once

#include "common.cuh"

namespace sst {

// resident warps per SM the register budget is sized for (16: <= 128 registers; measured on C3: 16 warps
// with one T staging buffer 8.81 ms, 12 warps with two 9.02 ms)
#ifndef SST_NB_WARPS
#define SST_NB_WARPS 16
#endif


template <int N2, int Z, bool FULL>
struct NbGeom {
    static constexpr int N = 64 * N2;
    static constexpr int J = Z * N2;          // columns j_lo = threads per CTA
    static constexpr int TPB = J;
    // narrow band: N2 rows per chunk (one stage-2 task per thread); full band: 32 rows per chunk,
    // 32 / N2 tasks per thread
    static constexpr int RPC = FULL ? 32 : N2;
    static constexpr int KPC = RPC / 8;       // DIT indices k1' per chunk (rows tau_lo = k1' + 8 k2)
    static constexpr int CH = 64 / RPC;       // chunks per frame pair
    static constexpr int TPT = RPC * Z / TPB; // stage-2 tasks per thread and chunk
    static constexpr int S = J + Z;           // padded row stride (float2): conflict-free stage-2 reads
    static constexpr int OPL = N2 / Z;        // outputs per task after the residue sum
    static constexpr int LOGZ = Z == 1 ? 0 : Z == 2 ? 1 : Z == 4 ? 2 : 3;
    // OLA ring bank skew.  After the residue sum, lane b of a row holds outputs k = b + Z i, i.e.
    // tau = tau_lo + 64 b + 64 Z i: the Z lanes of a row are 64 b apart, the same bank.  A warp's
    // 32/Z rows have tau_lo offsets {0..KPC-1} + 8 {0..R-1} (R = (32/Z)/KPC).  Slot s is stored at
    // phys(s) = s + sum_j o_j bit(s, 6 + j) + SUPER (s >> (6 + LOGZ)): o_j = KPC 2^j for the first
    // log2(8/KPC) bits of b, then 8 R 2^j', so that the warp's banks tile the 32 banks; each o_j
    // exceeds the sum of the smaller ones and SUPER (a multiple of 32) exceeds them all, so phys is
    // monotone (injective), and s -> s + 64 Z moves phys by 64 Z + SUPER (a lane's consecutive
    // outputs are one constant stride apart).  Off when 8 R > 32 (C2's geometry).
    static constexpr int R = (32 / Z) / KPC > 0 ? (32 / Z) / KPC : 1;
    static constexpr int LOGK = KPC == 1 ? 3 : KPC == 2 ? 2 : KPC == 4 ? 1 : 0;   // log2(8 / KPC)
    static constexpr bool SKEW = Z > 1 && 8 * R <= 32;
    __host__ __device__ static constexpr int o(int j) { return j < LOGK ? KPC << j : (8 * R) << (j - LOGK); }
    static constexpr int SUPER = SKEW ? 32 : 0;
    static constexpr int QB = 6 + LOGZ;                   // phys adds SUPER per 2^QB slots
    __device__ __forceinline__ static int phys(int s) {
        if constexpr (!SKEW) {
            return s;
        } else {
            int f = s + (s >> QB) * SUPER;
#pragma unroll
            for (int j = 0; j < LOGZ; ++j) f += ((s >> (6 + j)) & 1) * o(j);
            return f;
        }
    }
};

// RM <= 8: narrow band (T rows staged by TMA); RM = kNbFull: full band (k1 = 0, B = z N/2: every row
// nonzero, one full 64-point DFT per column, T loaded straight into registers)
constexpr int kNbFull = 32;

template <int N2, int Z, int RM>
__global__ void __launch_bounds__(NbGeom<N2, Z, RM == kNbFull>::TPB,
                                  ((RM == kNbFull ? (SST_NB_FULL_TMA ? 8 : 12) : SST_NB_WARPS) * 32 / NbGeom<N2, Z, RM == kNbFull>::TPB < 16
                                       ? (RM == kNbFull ? (SST_NB_FULL_TMA ? 8 : 12) : SST_NB_WARPS) * 32 / NbGeom<N2, Z, RM == kNbFull>::TPB : 16))
inv_nb_kernel(const InvArgs a) {
    constexpr bool FULL = RM == kNbFull;
    using Gm = NbGeom<N2, Z, FULL>;
    constexpr int N = Gm::N, J = Gm::J, TPB = Gm::TPB, KPC = Gm::KPC, CH = Gm::CH, S = Gm::S, OPL = Gm::OPL;
    constexpr int TPT = Gm::TPT, RPC = Gm::RPC;
    static_assert((FULL || (RM >= 1 && RM <= 8)) && N2 >= 8 && Z <= 8 && (TPB >= 32 || Z == 1), "narrow-band geometry");
    static_assert(!Gm::SKEW || (Z < 2 || Gm::o(0) >= 1) && (Z < 4 || Gm::o(1) > Gm::o(0)) &&
                                   (Z < 8 || Gm::o(2) > Gm::o(0) + Gm::o(1)) && Gm::SUPER > Gm::o(0) + (Z >= 4 ? Gm::o(1) : 0) + (Z >= 8 ? Gm::o(2) : 0),
                  "skew must be monotone");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float2* buf = reinterpret_cast<float2*>(smem_raw);
    float* ring = reinterpret_cast<float*>(smem_raw + a.lay.ring_off);
    const int t = threadIdx.x;
    const int tq = t / Z;                     // stage 1: column j_lo = t = Z tq + (t % Z)
    const int b = t % Z;                      // stage 2: residue b of rows t / Z + (TPB / Z) it

    const int64_t F = a.frame_end - a.frame_begin;
    const int64_t f_lo = (int64_t)blockIdx.x * a.frames_per_cta;
    if (f_lo >= F) return;
    const int64_t f_hi = min(F, f_lo + a.frames_per_cta);
    const bool first_cta = (blockIdx.x == 0);
    const bool last_cta = (f_hi == F);
    const int64_t H = a.hop;
    const int c = a.c;
    const int k1 = a.k1;
    const int B = a.bins;

    // OLA ring: sample s -> slot (s - g_lo) mod Rr -> ring[phys(slot)]; Rr is a multiple of 64 Z, so a
    // wrap by Rr moves phys by the constant Rp
    const int Rr = a.lay.ring;
    const int Rp = Gm::phys(Rr);
    for (int i = t; i < Rp + 64; i += TPB) ring[i] = 0.0f;
    __syncthreads();

    const int64_t g_lo = (a.frame_begin + f_lo) * H - c;            // first sample touched
    const int64_t left_end = g_lo + a.seam_len;                      // [g_lo, left_end) = left seam
    const int64_t right_start = (a.frame_begin + f_hi) * H - c;     // [right_start, ..) = right seam
    int64_t flushed = g_lo;
    // a10: completed samples [flushed, upto) leave the ring (normalised, or to the seam buffer)
    auto flush = [&](int64_t upto) {
        for (int64_t s = flushed + t; s < upto; s += TPB) {
            const int sl = (int)((s - g_lo) % Rr);
            float* slot = &ring[Gm::phys(sl)];
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
                SST_CHECK(s - a.y_off >= 0 && s - a.y_off < a.y_len);
                a.y[s - a.y_off] = val * inv_norm(s, a) * a.out_scale;
            } else {
                SST_CHECK(s - a.y_off >= 0 && s - a.y_off < a.y_len);
                a.y[s - a.y_off] += val;
            }
        }
        flushed = upto;
    };

    const float2* pb = a.phz + b * (64 + 2 * N2);     // e(b col) | e(64 b k) | e(b (64 k - N))
    // narrow band: T rows of a pair are staged in shared memory: one TMA bulk copy per row, issued a
    // pair ahead (two buffers) or after the previous pair's last stage-1 read (one buffer), completed on
    // the buffer's mbarrier; cooperative loads where the rows are not 16-byte aligned / sized
    const int Bp = (B + 2) & ~1;                          // row stride; entries [B, Bp) stay zero
    float2* tst = reinterpret_cast<float2*>(smem_raw + a.lay.g_off);
    uint64_t* mbar = reinterpret_cast<uint64_t*>(smem_raw + a.lay.g_off + (FULL ? 1 : SST_NB_TBUF) * 2 * Bp * 8);
    const bool bulk = (!FULL || SST_NB_FULL_TMA) && ((reinterpret_cast<uintptr_t>(a.T) & 15) == 0) && (a.ldT % 2 == 0) &&
                      (B % 2 == 0);
    auto issue = [&](int64_t f, int sel) {                // thread 0: rows f, f + 1 (< f_hi) -> buffer sel
        const int nrows = (f + 1 < f_hi) ? 2 : 1;
        fence_proxy_async();
        mbar_arrive_tx(&mbar[sel], (uint32_t)(nrows * B * 8));
        for (int r = 0; r < nrows; ++r) bulk_g2s(tst + (2 * sel + r) * Bp, a.T + (f + r) * a.ldT, (uint32_t)(B * 8), &mbar[sel]);
    };
    if constexpr (!FULL) {
        for (int i = t; i < 2 * SST_NB_TBUF * (Bp - B); i += TPB) tst[(i / (Bp - B)) * Bp + B + i % (Bp - B)] = make_float2(0.0f, 0.0f);
        if (t == 0) {
            mbar_init(&mbar[0], 1);
            mbar_init(&mbar[1], 1);
            fence_mbar_init();
        }
        __syncthreads();
        if (bulk && t == 0) issue(f_lo, 0);
    } else if constexpr (SST_NB_FULL_TMA) {
        if (t == 0) {
            mbar_init(&mbar[0], 1);
            fence_mbar_init();
        }
        __syncthreads();
        if (bulk && t == 0) issue(f_lo, 0);
    }
    uint32_t phase = 0;                                   // bit s = parity of buffer s's next completion
    int base0 = 0;                                        // slot of the pair's first sample sA - c
    for (int64_t f0 = f_lo; f0 < f_hi; f0 += 2, base0 = (base0 + 2 * (int)H) % Rr) {
        const bool hasB = f0 + 1 < f_hi;
        const int sel = SST_NB_TBUF == 2 ? (int)(((f0 - f_lo) >> 1) & 1) : 0;
        const float2* tA = tst + 2 * sel * Bp;
        const float2* tB = tA + Bp;
        float2 vf[FULL ? 64 : 1];                         // full band: the column's 64 stage-1 outputs
        if constexpr (FULL) {
          if (bulk) {
            // T rows staged by TMA (issued after the previous pair's inputs were read)
            mbar_wait(&mbar[0], phase & 1);
            phase ^= 1u;
            const float2* sB = hasB ? tA + Bp : tA;
#pragma unroll
            for (int jh = 0; jh < 32; ++jh) {
                float2 ta = tA[J * jh + t], tb = sB[J * jh + t];
                if (jh == 0 && t == 0) { ta.y = 0.0f; tb.y = 0.0f; }         // DC (j = 0): real part only (R14)
                vf[jh] = __fadd2_rn(ta, make_float2(-tb.y, tb.x));           // H_A + i H_B
            }
#pragma unroll
            for (int jh = 32; jh < 64; ++jh) {
                const int l = (jh == 32 && t == 0) ? B - J : J * (64 - jh) - t;
                float2 ta = tA[l], tb = sB[l];
                if (jh == 32 && t == 0) { ta = make_float2(0.0f, 0.0f); tb = ta; }   // l = B: none
                vf[jh] = __fadd2_rn(make_float2(ta.x, tb.x), make_float2(tb.y, -ta.y));   // conj H_A + i conj H_B
            }
            Fft<64, +1>::run(vf);
#pragma unroll
            for (int tl = 1; tl < 64; ++tl) vf[tl] = cmulc(vf[tl], __ldg(a.tw + tl * N2 + tq));   // e^{i 2 pi tq tau_lo / N}
          } else {
            {
                // L2 prefetch of the next pair's T rows (their DRAM latency overlaps this pair)
                const int64_t fn = f0 + 2;
                const int nrows = (int)min((int64_t)2, f_hi - fn);
                const int lines = (B * 8 + 127) >> 7;
                for (int i = t; i < nrows * lines; i += TPB) {
                    const int r = i / lines, q = i - r * lines;
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(a.T + (fn + r) * a.ldT) + q * 128));
                }
            }
            // column j_lo = t: rows j_hi < 32 band (l = j = J j_hi + t), rows >= 32 mirror (l = z N - j);
            // l = B (row 32, t = 0: the Nyquist bin, outside the half-open band) is zero.  Without a frame
            // B the pair reads frame A twice: G = (1 + i) H_A, whose IDFT has real part y_A (H_A is
            // Hermitian) and an imaginary part that is never added
            const float2* TA = a.T + f0 * a.ldT;
            const float2* TB = hasB ? TA + a.ldT : TA;
#pragma unroll
            for (int jh = 0; jh < 32; ++jh) {
                SST_CHECK(J * jh + t < B);
                float2 ta = __ldg(TA + J * jh + t), tb = __ldg(TB + J * jh + t);
                if (jh == 0 && t == 0) { ta.y = 0.0f; tb.y = 0.0f; }         // DC (j = 0): real part only (R14)
                vf[jh] = __fadd2_rn(ta, make_float2(-tb.y, tb.x));           // H_A + i H_B
            }
            {
                const float2* pA = TA + B - t;                               // l = J (64 - j_hi) - t
                const float2* pB = TB + B - t;
#pragma unroll
                for (int jh = 32; jh < 64; ++jh) {
                    const int off = -J * (jh - 32);
                    float2 ta = __ldg(pA + (jh == 32 ? (t ? 0 : -J) : off)), tb = __ldg(pB + (jh == 32 ? (t ? 0 : -J) : off));
                    if (jh == 32 && t == 0) { ta = make_float2(0.0f, 0.0f); tb = ta; }   // l = B: none
                    SST_CHECK(jh == 32 || (B - t + off >= 0 && B - t + off < B));
                    vf[jh] = __fadd2_rn(make_float2(ta.x, tb.x), make_float2(tb.y, -ta.y));   // conj H_A + i conj H_B
                }
            }
            Fft<64, +1>::run(vf);
#pragma unroll
            for (int tl = 1; tl < 64; ++tl) vf[tl] = cmulc(vf[tl], __ldg(a.tw + tl * N2 + tq));   // e^{i 2 pi tq tau_lo / N}
          }
        } else if (bulk) {
            if (SST_NB_TBUF == 2 && t == 0 && f0 + 2 < f_hi) issue(f0 + 2, sel ^ 1);
            mbar_wait(&mbar[sel], (phase >> sel) & 1);
            phase ^= 1u << sel;
        } else {
            float2* dst = tst + 2 * sel * Bp;
            for (int i = t; i < B; i += TPB) {
                dst[i] = __ldg(a.T + f0 * a.ldT + i);
                if (hasB) dst[Bp + i] = __ldg(a.T + (f0 + 1) * a.ldT + i);
            }
            __syncthreads();
        }
        // ---- narrow band, inputs of column j_lo = t: band rows j_hi < RM (G = T_A + i T_B at
        // l = j - z k1) and mirror rows j_hi >= 64 - RM (G = conj T_A + i conj T_B at l = z N - j - z k1),
        // read from the staged rows for every chunk so that they are not live across stage 2
        // (entries outside the band, and frame B of a last odd frame, read the zero at index B)
        constexpr int NIN = FULL ? 1 : 2 * RM;
        auto load_inputs = [&](float2 (&in)[NIN]) {
            if constexpr (!FULL) {
#pragma unroll
                for (int i = 0; i < RM; ++i) {
                    const int l = J * i + t - Z * k1;
                    const bool ok = (unsigned)l < (unsigned)B;
                    float2 ta = tA[ok ? l : B], tb = tB[ok && hasB ? l : B];
                    if (i == 0 && t == 0) { ta.y = 0.0f; tb.y = 0.0f; }      // DC (j = 0): real part only (R14)
                    in[i] = __fadd2_rn(ta, make_float2(-tb.y, tb.x));        // H_A + i H_B
                }
#pragma unroll
                for (int i = 0; i < RM; ++i) {
                    const int l = J * (RM - i) - t - Z * k1;                  // j = J (64 - RM + i) + t
                    const bool ok = (unsigned)l < (unsigned)B;
                    const float2 ta = tA[ok ? l : B], tb = tB[ok && hasB ? l : B];
                    in[RM + i] = __fadd2_rn(make_float2(ta.x, tb.x), make_float2(tb.y, -ta.y));   // conj H_A + i conj H_B
                }
            }
        };
        const int64_t sA = (a.frame_begin + f0) * H;

#pragma unroll
        for (int ch = 0; ch < CH; ++ch) {
            // ---- stage 1: rows tau_lo = k1' + 8 k2, k1' in [KPC ch, KPC ch + KPC) (compile time)
            if constexpr (FULL) {
#pragma unroll
                for (int r = 0; r < RPC; ++r) {
                    const int tau_lo = KPC * ch + (r % KPC) + 8 * (r / KPC);
                    buf[r * S + t] = vf[tau_lo];
                }
            } else {
                float2 in[NIN];
                load_inputs(in);
#pragma unroll
                for (int kk = 0; kk < KPC; ++kk) {
                    const int k1p = KPC * ch + kk;
                    float2 v[8];
#pragma unroll
                    for (int n2 = 0; n2 < 8; ++n2) {
                        // nonzero inputs of the 8-point sum over n1: n1 = 0 (row n2 < RM), n1 = 7 (row 56 + n2 >= 64 - RM)
                        float2 acc = make_float2(0.0f, 0.0f);
                        bool any = false;
                        if (n2 < RM) { acc = in[n2]; any = true; }
                        if (n2 >= 8 - RM) {
                            const float2 u = mul_w8<+1>(in[2 * RM + n2 - 8], 7 * k1p);
                            acc = any ? cadd(acc, u) : u;
                            any = true;
                        }
                        v[n2] = (n2 * k1p == 0 || !any) ? acc : cmul(acc, twiddle<64, +1>(n2 * k1p));
                    }
                    Fft<8, +1>::run(v);
#pragma unroll
                    for (int k2 = 0; k2 < 8; ++k2) {
                        const int tau_lo = k1p + 8 * k2;
                        float2 y = v[k2];
                        // e(j_lo tau_lo) = e^{i 2 pi tq tau_lo / N} e(b' tau_lo): the first factor here, the
                        // second (constant per stage-2 item) with the output phase below
                        if (tau_lo != 0) y = cmulc(y, __ldg(a.tw + tau_lo * N2 + tq));
                        SST_CHECK((kk + KPC * k2) * S + t < RPC * S);
                        buf[(kk + KPC * k2) * S + t] = y;
                    }
                }
            }
            __syncthreads();
            if (ch == 0) flush(sA - c);                                       // earlier pairs are complete
            if (!FULL && SST_NB_TBUF == 1 && ch == CH - 1 && bulk && t == 0 && f0 + 2 < f_hi) issue(f0 + 2, 0);   // inputs read
            if (FULL && ch == 0 && bulk && t == 0 && f0 + 2 < f_hi) issue(f0 + 2, 0);                          // inputs read

            // ---- stage 2, task it: row r2 = t / Z + (TPB / Z) it (tau_lo = KPC ch + r2 % KPC + 8 (r2 / KPC)),
            // residue b; frame A (real part) is overlap-added now, frame B (imaginary part, H samples
            // later) after the barrier (chunks and pairs are ordered by the barriers)
            float yb[TPT][OPL];
            int sb0[TPT][2];
#pragma unroll
            for (int it = 0; it < TPT; ++it) {
                const int r2 = t / Z + (TPB / Z) * it;
                const int tau_lo = KPC * ch + (r2 % KPC) + 8 * (r2 / KPC);
                float2 x[N2];
#pragma unroll
                for (int i = 0; i < N2; ++i) x[i] = buf[r2 * S + Z * i + b];
                Fft<N2, +1>::run(x);
                if constexpr (Z > 1) {
                    // output phase e(b tau) = e(b tau_lo) e(64 b k'), k' = k (k < N2/2) or k - N2: two runs of
                    // a recurrence in e(64 b) started from the table (<= N2/2 - 1 steps each)
                    const float2 cb = __ldg(pb + tau_lo);
                    const float2 step = __ldg(pb + 64 + 1);
                    float2 ph = cb;
                    float2 ph2 = cmul(cb, __ldg(pb + 64 + N2 + N2 / 2));
#pragma unroll
                    for (int k = 0; k < N2 / 2; ++k) {
                        x[k] = cmul(x[k], ph);
                        x[k + N2 / 2] = cmul(x[k + N2 / 2], ph2);
                        if (k + 1 < N2 / 2) {
                            ph = cmul(ph, step);
                            ph2 = cmul(ph2, step);
                        }
                    }
                    // reduce-scatter over the Z lanes of the row (bits of k from the top bit of b down): lane b
                    // ends with outputs k = b + Z i in x[Z i]
#pragma unroll
                    for (int lvl = 0; lvl < Gm::LOGZ; ++lvl) {
                        const int m = Z >> (lvl + 1);
                        const bool up = (b & m) != 0;
#pragma unroll
                        for (int k = 0; k < N2; ++k) {
                            if ((k & (Z - 1)) & ~(2 * m - 1)) continue;   // k's lower bits above m already reduced away
                            if (k & m) continue;
                            const float2 snd = up ? x[k] : x[k | m];
                            const float2 kp = up ? x[k | m] : x[k];
                            float2 rcv;
                            rcv.x = __shfl_xor_sync(0xffffffffu, snd.x, m);
                            rcv.y = __shfl_xor_sync(0xffffffffu, snd.y, m);
                            x[k] = cadd(kp, rcv);
                        }
                    }
                }
                // window g[tau + c] / N.  Output i of this lane: k = b + Z i, tau = tau_lo + 64 k - (k >= N2/2 ?
                // N : 0).  OPL >= 2: two runs of consecutive slots 64 Z apart (i < OPL/2, i >= OPL/2), each
                // addressed from its first slot (phys stride 64 Z + SUPER, minus Rp once the run wraps the
                // ring); OPL = 1: one output, wrapped by the lane's b
                constexpr int HALF = (OPL + 1) / 2;        // first output of the second run (tau < 0)
                constexpr int DP = 64 * Z + Gm::SUPER;
                const int u0 = tau_lo + 64 * b + c;        // tau + c of output 0 (before the wrap)
                int pa0[2];
#pragma unroll
                for (int run = 0; run < (OPL > 1 ? 2 : 1); ++run) {
                    const int i0 = run ? HALF : 0;
                    const bool wrap = OPL > 1 ? (run == 1) : (b >= N2 / 2);
                    int sl = base0 + u0 + 64 * Z * i0 - (wrap ? N : 0);
                    if (sl >= Rr) sl -= Rr;
                    sb0[it][run] = sl;
                    pa0[run] = Gm::phys(sl);
                }
#pragma unroll
                for (int i = 0; i < OPL; ++i) {
                    const int run = (OPL > 1 && i >= HALF) ? 1 : 0, di = i - (run ? HALF : 0);
                    const bool wrap = OPL > 1 ? (run == 1) : (b >= N2 / 2);
                    const int u = u0 + 64 * Z * i - (wrap ? N : 0);   // tau + c in [0, L)
                    SST_CHECK(u >= 0 && u < a.L);
                    const float gw = __ldg(a.gwin + u);                        // g / N_f
                    const int s = sb0[it][run] + 64 * Z * di;
                    const int p = pa0[run] + DP * di - (s >= Rr ? Rp : 0);
                    SST_CHECK(p == Gm::phys(s % Rr));
                    const float2 yv = cscale(x[Z * i], gw);
                    ring[p] += yv.x;
                    yb[it][i] = yv.y;
                }
            }
            __syncthreads();
            if (hasB) {
#pragma unroll
                for (int it = 0; it < TPT; ++it) {
                    constexpr int NRUN = OPL > 1 ? 2 : 1;
                    int s0[NRUN], p0[NRUN];
#pragma unroll
                    for (int run = 0; run < NRUN; ++run) {
                        s0[run] = sb0[it][run] + (int)H;
                        if (s0[run] >= Rr) s0[run] -= Rr;
                        p0[run] = Gm::phys(s0[run]);
                    }
#pragma unroll
                    for (int i = 0; i < OPL; ++i) {
                        const int run = (OPL > 1 && i >= ((OPL + 1) / 2)) ? 1 : 0, di = i - (run ? ((OPL + 1) / 2) : 0);
                        const int s = s0[run] + 64 * Z * di;
                        const int p = p0[run] + (64 * Z + Gm::SUPER) * di - (s >= Rr ? Rp : 0);
                        SST_CHECK(p == Gm::phys(s % Rr));
                        ring[p] += yb[it][i];
                    }
                }
            }
        }
    }
    __syncthreads();
    flush((a.frame_begin + f_hi - 1) * H - c + a.L);
}

template <int N2, int Z, int RM>
static cudaError_t launch_nb_b(const InvArgs& a, int grid, cudaStream_t s) {
    auto kern = inv_nb_kernel<N2, Z, RM>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, a.lay.total);
    if (e != cudaSuccess) return e;
    kern<<<grid, NbGeom<N2, Z, RM == kNbFull>::TPB, a.lay.total, s>>>(a);
    return cudaGetLastError();
}

template <int N2, int Z>
static cudaError_t launch_nb_z(const InvArgs& a, int grid, cudaStream_t s) {
    if constexpr (N2 == 8) {
        if constexpr (Z >= 4) return launch_nb_b<N2, Z, kNbFull>(a, grid, s);   // C5
        return cudaErrorInvalidValue;
    } else {
        if (inv_nb_rows(N2, a.k1, a.bins, a.zoom) <= 5) return launch_nb_b<N2, Z, 5>(a, grid, s);   // C2, C3
        return launch_nb_b<N2, Z, 8>(a, grid, s);
    }
}

template <int N2>
static cudaError_t launch_nb(const InvArgs& a, int grid, cudaStream_t s) {
    if constexpr (N2 == 8 || N2 == 16 || N2 == 32) {
        switch (a.zoom) {
            case 1: return launch_nb_z<N2, 1>(a, grid, s);
            case 2: return launch_nb_z<N2, 2>(a, grid, s);
            case 4: return launch_nb_z<N2, 4>(a, grid, s);
            case 8: return launch_nb_z<N2, 8>(a, grid, s);
        }
    }
    return cudaErrorInvalidValue;
}

template <int N2, int Z>
static int occ_nb_z(int smem, int device) {
    constexpr int RM = N2 == 8 ? kNbFull : 5;
    if constexpr (N2 == 8 && Z < 4) {
        return 0;
    } else {
        int nb = 0, sms = 0;
        auto kern = inv_nb_kernel<N2, Z, RM>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, NbGeom<N2, Z, RM == kNbFull>::TPB, smem);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
        return (nb > 0 ? nb : 1) * sms;
    }
}

template <int N2>
static int occ_nb(int hop, int L, int zoom, int k1, int bins, int device) {
    if (!inv_nb_applicable(64 * N2, L, 64 * N2 / 2, hop, zoom, k1, bins)) return 0;
    if constexpr (N2 == 8 || N2 == 16 || N2 == 32) {
        const int smem = inv_nb_layout(N2, L, hop, zoom, bins).total;
        if (smem > 227 * 1024) return 0;
        switch (zoom) {
            case 1: return occ_nb_z<N2, 1>(smem, device);
            case 2: return occ_nb_z<N2, 2>(smem, device);
            case 4: return occ_nb_z<N2, 4>(smem, device);
            case 8: return occ_nb_z<N2, 8>(smem, device);
        }
    }
    return 0;
}

}  // namespace sst
