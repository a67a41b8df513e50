// Per-bin decision shared by the fused forward (sst_kernels.cu) and the multi-pass large-N_f
// forward (multipass.cu): unpack (a3), mask (Eq. 13), reassignment frequency (Eq. 36) and target
// bin (Eq. 28, R10, R17), so both paths take every integer decision with the same arithmetic.
//
// Reading R23: the fp32 decision is final only where the fp32 packed FFT provably
// cannot have moved it.  Each decision carries an error margin from the FFT's error model
// (R21: one bin of the packed fp32 FFT of frame m is off by at most eta = 4 u sqrt(log2 N_f) ||z_m||,
// calibrated on the configs at <= 0.95 of the model, taken 8 x here); a bin whose fp32 target lies
// closer than that margin to a rounding boundary (Eq. 28) or whose |S| lies that close to gamma
// (Eq. 13) is re-decided from S, S' recomputed in fp64 by the direct Eq. 8 sum --
// warp-cooperative, rare (measured well under one bin per frame on C2-C5).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "sst_internal.h"

namespace sst {

// (hi 2^20 + lo) * s for the squeeze's limb sums: one fused rounding of the two converted limbs
// (|hi| < 2^30, 0 <= lo < 2^31.01), i.e. within an fp32 ulp of the exact integer sum
__device__ __forceinline__ float limbs_to_float(int hi, int lo, float s) {
    return fmaf((float)hi, 1048576.0f, (float)(unsigned)lo) * s;
}

__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ float rsqrt_approx(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// Per source bin k with Za = Z[k], Zb = Z[N-k]: returns target l (>= 0), -1 masked, -2 out of band.
// S = (P, Q)/2 with P = Re Za + Re Zb, Q = Im Za - Im Zb;  S' = (U, -V)/(2 alpha) with
// U = Im Za + Im Zb, V = Re Za - Re Zb;  -Im(S'/S) = (V P + U Q) / (alpha (P^2 + Q^2)).
// Branch-free (the bins of a thread interleave): select chains instead of early returns.
// cm, km: the frame's R23 margins (see fwd_margins); unsure = the fp32 result is not final.
// FULLWARP: every lane of the warp calls it together (the fused kernel); else the vote uses the
// active mask (the multi-pass kernel's strided bin loop).
// Core on (P, Q) = 2 S and (U, V) = 2 alpha (Re S', -Im S') (shared with the filter-bank path, which
// has S and S' directly).
template <bool FULLWARP = true>
__device__ __forceinline__ int bin_target_pq(const FwdArgs& a, float gam4, float cm, float km, int k, float2 PQ,
                                             float2 UV, float& mag4, bool& unsure) {
    const float2 sq = __fmul2_rn(PQ, PQ);
    mag4 = sq.x + sq.y;                                                      // 4 |S|^2
    const bool src = k >= a.src_lo && k < a.src_hi;
    const bool keep = (mag4 > gam4) && src;                                  // mask (Eq. 13)
    const float2 vu = __fmul2_rn(make_float2(UV.y, UV.x), PQ);              // (V P, U Q)
    // z r: RF in fine bins (Eq. 36), r = -Im(S'/S) N_f/(2 pi) = (V P + U Q)/(P^2 + Q^2) * N_f/(2 pi alpha)
    const float rsq = rcp_approx(mag4);
    const float zr = (vu.x + vu.y) * rsq * a.zr_scale;
    const bool fin = fabsf(zr) <= 1073741824.0f;                             // non-finite or huge (R17)
    const bool pos = zr >= -(float)(a.zoom * k);                             // k + r >= 0
    const int base = pos ? a.zoom * (k - a.k1) : -a.zoom * (k + a.k1);      // |k + r| = -(k + r) otherwise
    const float t = pos ? zr + 0.5f : 0.5f - zr;                            // fine position - base
    const float fl = floorf(t);
    const int l = base + (int)fl;                                            // Eq. 28 (R10, R17)
    const int lin = ((unsigned)l < (unsigned)a.bins && fin) ? l : -2;
    // R23 margin of the fine position: z delta r = cm (1/|2S| + (|U|+|V|)/|2S|^2) (R21 error model);
    // only targets in [-1, B] can cross into / inside the band (margins of coefficients the north
    // star's location clause covers, |S| >= 1e-2 max|S|, stay far below half a bin).  Evaluated only
    // when some lane of the warp has such a target (warp-uniform skip: most source bins of a narrow
    // band's plane land far outside it).
    const bool cand = src && (unsigned)(l + 1) <= (unsigned)a.bins + 1u && fin;
    unsure = false;
    if (__any_sync(FULLWARP ? 0xffffffffu : __activemask(), cand)) {
        // branch-free (bitwise &, |): a margin below the flush-to-zero range only under-flags bins whose
        // |S| ~ 1e-19 ||z_m||, far below any threshold that matters
        const float rs = rsqrt_approx(mag4);
        const float mg = cm * fmaf(fabsf(UV.x) + fabsf(UV.y), rsq, rs);
        const float fr = t - fl;
        unsure = cand & ((keep & (fabsf(fr - 0.5f) > 0.5f - mg)) | (fabsf(mag4 - gam4) < km));
    }
    return keep ? lin : -1;
}

template <bool FULLWARP = true>
__device__ __forceinline__ int bin_target(const FwdArgs& a, float gam4, float cm, float km, int k, float2 za,
                                          float2 zb, float2& PQ, float2& UV, float& mag4, bool& unsure) {
    PQ = __fadd2_rn(za, make_float2(zb.x, -zb.y));                           // (P, Q) = 2 S
    UV = __fadd2_rn(make_float2(za.y, za.x), make_float2(zb.y, -zb.x));      // (U, V) = 2 alpha (Re, -Im) S'
    return bin_target_pq<FULLWARP>(a, gam4, cm, km, k, PQ, UV, mag4, unsure);
}

// R23 margins of one frame from its packed-input norm ||z_m||_2 (nrm2 = ||z_m||^2):
//   cm: margin factor of the fine position (cflag = 8 zr_scale 4 u sqrt(log2 N_f), set by the plan);
//   km: margin of 4|S|^2 around 4 gamma^2 (|S| off by at most kd = 8 * 2 u sqrt(log2 N_f) ||z_m||).
__device__ __forceinline__ void fwd_margins(const FwdArgs& a, float gam4, float nrm2, float& cm, float& km) {
    const float nrm = sqrtf(nrm2);
    cm = a.cflag * nrm;
    const float kd = a.kflag * nrm;
    km = 4.0f * kd * fmaf(2.0f, 0.5f * sqrtf(fmaxf(gam4, 0.0f)), kd);
    if (!a.redecide) { cm = 0.0f; km = -1.0f; }
}

// fp64 S, S' of bin k of one frame by the direct Eq. 8 sum
//   S[m,k] = sum_{j=0}^{L-1} x[m H - c + j] g[j] e^{-i 2 pi k (j - c)/N_f}   (and g' for S'),
// warp-cooperative: all 32 lanes call it with the same k and frame.  Lane l takes taps
// j = l + 32 t; with W = e^{-2 pi i/N_f}, W^{k (j - c)} = W^{k (l - c)} W^{32 k t}, so the per-tap
// twiddle W^{32 k t} is the same for every lane (one broadcast load) and the lane factor
// W^{k (l - c)} multiplies the lane's partial sums once; fixed xor-tree reduction (deterministic).
// xat(j) returns the frame's sample j as float (zero outside the record).  taps64[j] = (g[j], g'[j]);
// tw64[e] = W^e, both fp64.
template <class XF>
__device__ __forceinline__ void stft_bin_fp64(XF xat, const double2* __restrict__ taps64,
                                              const double2* __restrict__ tw64, int nfft, int L, int c, int k,
                                              double& sr, double& si, double& dr, double& di) {
    const int lane = threadIdx.x & 31;
    const unsigned msk = (unsigned)nfft - 1u;
    const unsigned step = (32u * (unsigned)k) & msk;
    double ar = 0.0, ai = 0.0, br = 0.0, bi = 0.0;
    unsigned e = 0;
#pragma unroll 4
    for (int j = lane; j < L; j += 32) {
        const double xv = (double)xat(j);
        const double2 w = __ldg(taps64 + j);
        const double2 t = __ldg(tw64 + e);                                   // W^{32 k t}: warp-uniform
        const double p = xv * w.x, q = xv * w.y;
        ar = fma(p, t.x, ar);
        ai = fma(p, t.y, ai);
        br = fma(q, t.x, br);
        bi = fma(q, t.y, bi);
        e = (e + step) & msk;
    }
    const double2 f = __ldg(tw64 + (((unsigned)k * (unsigned)(lane - c)) & msk));   // W^{k (l - c)}
    sr = ar * f.x - ai * f.y;
    si = ar * f.y + ai * f.x;
    dr = br * f.x - bi * f.y;
    di = br * f.y + bi * f.x;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        sr += __shfl_xor_sync(0xffffffffu, sr, o);
        si += __shfl_xor_sync(0xffffffffu, si, o);
        dr += __shfl_xor_sync(0xffffffffu, dr, o);
        di += __shfl_xor_sync(0xffffffffu, di, o);
    }
}

// One part of the same sum: virtual warp `part` of `parts` (a fixed decomposition of the taps, so
// the fp64 result does not depend on how many real warps share the work): lane l takes taps
// j = 32 part + l + 32 parts t, so W^{k (j - c)} = W^{k (32 part + l - c)} W^{32 parts k t}: one
// table load per thread and a uniform per-tap factor generated by the recurrence w <- w W^{32 parts k}
// (<= L / (32 parts) steps of fp64 complex products, ~1e-14 relative).  tap64(j) returns (g[j], g'[j])
// in fp64.  Returns the part's sums (Re S, Im S, Re S', Im S') on every lane (fixed xor tree).
template <class XF, class TF>
__device__ __forceinline__ double4 stft_bin_fp64_part(XF xat, TF tap64, const double2* __restrict__ tw64,
                                                      int nfft, int L, int c, int k, int part, int parts) {
    const int lane = threadIdx.x & 31;
    const unsigned msk = (unsigned)nfft - 1u;
    const int j0 = 32 * part + lane, stride = 32 * parts;
    const double2 st = __ldg(tw64 + (((unsigned)stride * (unsigned)k) & msk));
    const double2 f = __ldg(tw64 + (((unsigned)k * (unsigned)(j0 - c)) & msk));
    double ar = 0.0, ai = 0.0, br = 0.0, bi = 0.0;
    double wr = 1.0, wi = 0.0;
#pragma unroll 4
    for (int j = j0; j < L; j += stride) {
        const double xv = (double)xat(j);
        const double2 w = tap64(j);
        const double p = xv * w.x, q = xv * w.y;
        ar = fma(p, wr, ar);
        ai = fma(p, wi, ai);
        br = fma(q, wr, br);
        bi = fma(q, wi, bi);
        const double nr = fma(wr, st.x, -wi * st.y);
        wi = fma(wr, st.y, wi * st.x);
        wr = nr;
    }
    double s0 = ar * f.x - ai * f.y, s1 = ar * f.y + ai * f.x;
    double s2 = br * f.x - bi * f.y, s3 = br * f.y + bi * f.x;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        s3 += __shfl_xor_sync(0xffffffffu, s3, o);
    }
    return make_double4(s0, s1, s2, s3);
}

// The oracle's decision (Eq. 13, 36, 28; R8, R10) in fp64 on the fp64 S, S'.
__device__ __forceinline__ int decide_fp64(const FwdArgs& a, double gamma, int k, double sr, double si, double dr,
                                           double di) {
    if (!(k >= a.src_lo && k < a.src_hi)) return -1;
    const double mag = sr * sr + si * si;
    if (!(mag > gamma * gamma)) return -1;                                   // |S| > gamma (Eq. 13)
    const double im = di * sr - dr * si;                                     // Im(S' conj S)
    const double r = -im / mag * ((double)a.nfft / 6.283185307179586476925);   // Eq. 36
    const double fh = fabs((double)k + r);                                   // Eq. 13 (R8)
    const double p = (double)a.zoom * (fh - (double)a.k1) + 0.5;             // Eq. 28 (R10)
    if (!(p >= 0.0 && p < (double)a.bins)) return -2;
    return (int)floor(p);
}

// gamma of the launch in fp64 (absolute, or relative to the device max |S|)
__device__ __forceinline__ double launch_gamma64(const FwdArgs& a) {
    return a.absmax_dev ? a.gamma_rel_d * (double)__ldg(a.absmax_dev) : a.gamma_d;
}

}  // namespace sst
