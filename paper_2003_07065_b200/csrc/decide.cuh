// Per-bin decision shared by the fused forward (sst_kernels.cu) and the multi-pass large-N_f
// forward (multipass.cu): unpack (a3), mask (Eq. 13), reassignment frequency (Eq. 36) and target
// bin (Eq. 28, R10, R17), so both paths take every integer decision with the same fp32 arithmetic.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "sst_internal.h"

namespace sst {

// Per source bin k with Za = Z[k], Zb = Z[N-k]: returns target l (>= 0), -1 masked, -2 out of band.
// S = (P, Q)/2 with P = Re Za + Re Zb, Q = Im Za - Im Zb;  S' = (U, -V)/(2 alpha) with
// U = Im Za + Im Zb, V = Re Za - Re Zb;  -Im(S'/S) = (V P + U Q) / (alpha (P^2 + Q^2)).
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

// Branch-free (the 33 bins of a thread interleave): select chains instead of early returns.
__device__ __forceinline__ int bin_target(const FwdArgs& a, float gam4, int k, float2 za, float2 zb, float2& PQ,
                                          float2& UV, float& mag4) {
    PQ = __fadd2_rn(za, make_float2(zb.x, -zb.y));                           // (P, Q) = 2 S
    UV = __fadd2_rn(make_float2(za.y, za.x), make_float2(zb.y, -zb.x));      // (U, V) = 2 alpha (Re, -Im) S'
    const float2 sq = __fmul2_rn(PQ, PQ);
    mag4 = sq.x + sq.y;                                                      // 4 |S|^2
    const bool keep = (mag4 > gam4) && k >= a.src_lo && k < a.src_hi;        // mask (Eq. 13)
    const float2 vu = __fmul2_rn(make_float2(UV.y, UV.x), PQ);              // (V P, U Q)
    // z r: RF in fine bins (Eq. 36), r = -Im(S'/S) N_f/(2 pi) = (V P + U Q)/(P^2 + Q^2) * N_f/(2 pi alpha)
    const float zr = (vu.x + vu.y) * rcp_approx(mag4) * a.zr_scale;
    const bool fin = fabsf(zr) <= 1073741824.0f;                             // non-finite or huge (R17)
    const bool pos = zr >= -(float)(a.zoom * k);                             // k + r >= 0
    const int base = pos ? a.zoom * (k - a.k1) : -a.zoom * (k + a.k1);      // |k + r| = -(k + r) otherwise
    const int l = base + __float2int_rd(pos ? zr + 0.5f : 0.5f - zr);       // Eq. 28 (R10, R17)
    const int lin = ((unsigned)l < (unsigned)a.bins && fin) ? l : -2;
    return keep ? lin : -1;
}

}  // namespace sst
