// In-register complex DFTs for the SST kernels (sm_100a).
//
// fft<N, DIR>(a): a[0..N) in natural order -> DFT in natural order, N in {1,2,4,8,16,32,64},
// DIR = -1 forward (e^{-2 pi i nk/N}), +1 inverse (no 1/N).  All indices are compile-time,
// so the composite (four-step) orderings are pure register renaming: no data movement.
// Twiddles W_64^e come from constant memory with compile-time offsets (operand c[][] form).
#pragma once

#include <cuda_runtime.h>

namespace sst {

// Uploaders of every translation unit's constant twiddle table (sst_api.cu calls them all once per
// device).  The kernels are compiled as several separate CUDA modules (one per N2 and direction, for
// a parallel build), each with its own copy of c_w64.
void register_w64_uploader(cudaError_t (*fn)(const float2*));

namespace {
__constant__ float2 c_w64[64];   // W_64^e = exp(-2 pi i e / 64), rounded from fp64 (set at plan creation)
cudaError_t upload_w64_this_tu(const float2* w) { return cudaMemcpyToSymbol(c_w64, w, sizeof(float2) * 64); }
struct W64Registrar {
    W64Registrar() { register_w64_uploader(&upload_w64_this_tu); }
};
const W64Registrar w64_registrar;
}  // namespace

// Complex arithmetic on sm_100a's packed FP32x2 pipe (FADD2 / FMUL2 / FFMA2): one instruction per
// complex add, two per complex multiply; swaps and sign flips fold into operand modifiers.
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ float2 cscale(float2 a, float s) { return __fmul2_rn(a, make_float2(s, s)); }
// a * b = b.x (a.x, a.y) + b.y (-a.y, a.x)
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return __ffma2_rn(make_float2(-a.y, a.x), make_float2(b.y, b.y), __fmul2_rn(a, make_float2(b.x, b.x)));
}
// a * conj(b) = b.x (a.x, a.y) + b.y (a.y, -a.x)
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {
    return __ffma2_rn(make_float2(a.y, -a.x), make_float2(b.y, b.y), __fmul2_rn(a, make_float2(b.x, b.x)));
}
// multiply by exp(DIR * i pi/2): DIR=-1 -> -i, DIR=+1 -> +i
template <int DIR>
__device__ __forceinline__ float2 rot90(float2 a) {
    return DIR < 0 ? make_float2(a.y, -a.x) : make_float2(-a.y, a.x);
}
// W_N^e for the transform direction (compile-time e, N | 64)
template <int N, int DIR>
__device__ __forceinline__ float2 twiddle(int e) {
    float2 w = c_w64[(e * (64 / N)) & 63];
    return DIR < 0 ? w : make_float2(w.x, -w.y);
}

template <int N, int DIR>
struct Fft;

template <int DIR>
struct Fft<1, DIR> {
    __device__ __forceinline__ static void run(float2 (&)[1]) {}
};

template <int DIR>
struct Fft<2, DIR> {
    __device__ __forceinline__ static void run(float2 (&a)[2]) {
        float2 t = a[0];
        a[0] = cadd(t, a[1]);
        a[1] = csub(t, a[1]);
    }
};

template <int DIR>
struct Fft<4, DIR> {
    __device__ __forceinline__ static void run(float2 (&a)[4]) {
        float2 t0 = cadd(a[0], a[2]), t1 = csub(a[0], a[2]);
        float2 t2 = cadd(a[1], a[3]), t3 = rot90<DIR>(csub(a[1], a[3]));
        a[0] = cadd(t0, t2);
        a[2] = csub(t0, t2);
        a[1] = cadd(t1, t3);
        a[3] = csub(t1, t3);
    }
};

template <int DIR>
struct Fft<8, DIR> {
    __device__ __forceinline__ static void run(float2 (&a)[8]) {
        const float h = 0.70710678118654752440f;
        float2 e[4] = {a[0], a[2], a[4], a[6]};
        float2 o[4] = {a[1], a[3], a[5], a[7]};
        Fft<4, DIR>::run(e);
        Fft<4, DIR>::run(o);
        // o[k] *= W_8^k
        // W_8 = h (1 - i) (DIR = -1) or h (1 + i); W_8^3 = -h (1 + i) or h (-1 + i)
        const float2 o1 = o[1], o3 = o[3];
        if (DIR < 0) {
            o[1] = cscale(cadd(o1, make_float2(o1.y, -o1.x)), h);
            o[3] = cscale(cadd(make_float2(o3.y, -o3.x), make_float2(-o3.x, -o3.y)), h);
        } else {
            o[1] = cscale(cadd(o1, make_float2(-o1.y, o1.x)), h);
            o[3] = cscale(cadd(make_float2(-o3.y, o3.x), make_float2(-o3.x, -o3.y)), h);
        }
        o[2] = rot90<DIR>(o[2]);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            a[k] = cadd(e[k], o[k]);
            a[k + 4] = csub(e[k], o[k]);
        }
    }
};

// composite N = R1 * R2 (four-step, registers only):
//   n = R2 n1 + n2, k = k1 + R1 k2
//   X[k1 + R1 k2] = sum_n2 W_R2^{n2 k2} W_N^{n2 k1} sum_n1 x[R2 n1 + n2] W_R1^{n1 k1}
template <int N, int R1, int DIR>
struct FftComposite {
    static constexpr int R2 = N / R1;
    __device__ __forceinline__ static void run(float2 (&a)[N]) {
        float2 b[R2][R1];
#pragma unroll
        for (int n2 = 0; n2 < R2; ++n2) {
            float2 t[R1];
#pragma unroll
            for (int n1 = 0; n1 < R1; ++n1) t[n1] = a[R2 * n1 + n2];
            Fft<R1, DIR>::run(t);
#pragma unroll
            for (int k1 = 0; k1 < R1; ++k1) {
                const int e = n2 * k1;
                b[n2][k1] = (e == 0) ? t[k1] : cmul(t[k1], twiddle<N, DIR>(e));
            }
        }
#pragma unroll
        for (int k1 = 0; k1 < R1; ++k1) {
            float2 u[R2];
#pragma unroll
            for (int n2 = 0; n2 < R2; ++n2) u[n2] = b[n2][k1];
            Fft<R2, DIR>::run(u);
#pragma unroll
            for (int k2 = 0; k2 < R2; ++k2) a[k1 + R1 * k2] = u[k2];
        }
    }
};

// x * W_8^e for the transform direction (compile-time e): swaps / sign flips and at most one
// add + scale, W_8^{odd} = h (+-1 +- i)
template <int DIR>
__device__ __forceinline__ float2 mul_w8(float2 x, int e) {
    const float h = 0.70710678118654752440f;
    switch (e & 7) {
        case 0: return x;
        case 2: return rot90<DIR>(x);
        case 4: return make_float2(-x.x, -x.y);
        case 6: { const float2 r = rot90<DIR>(x); return make_float2(-r.x, -r.y); }
        case 1: return cscale(cadd(x, rot90<DIR>(x)), h);
        case 3: return cscale(csub(rot90<DIR>(x), x), h);
        case 5: return cscale(cadd(x, rot90<DIR>(x)), -h);
        default: return cscale(csub(x, rot90<DIR>(x)), h);
    }
}

// 64-point DFT of an input that is zero outside rows [0, RM) and [64 - RM, 64) (the inverse's
// narrow-band sub-spectra): as FftComposite<64, 8>, but each first-stage 8-point sub-DFT
// (inputs a[8 n1 + n2], n1 = 0..7) is a direct sum over its nonzero inputs only -- the packed
// FP32x2 intrinsics are opaque to the compiler, so it would not drop the zero terms by itself.
template <int DIR, int RM>
struct FftSparse64 {
    __device__ __forceinline__ static void run(float2 (&a)[64]) {
        float2 b[8][8];
#pragma unroll
        for (int n2 = 0; n2 < 8; ++n2) {
#pragma unroll
            for (int k1 = 0; k1 < 8; ++k1) {
                float2 acc = make_float2(0.0f, 0.0f);
                bool first = true;
#pragma unroll
                for (int n1 = 0; n1 < 8; ++n1) {
                    const int n = 8 * n1 + n2;
                    if (n >= RM && n < 64 - RM) continue;             // compile-time zero row
                    const float2 t = mul_w8<DIR>(a[n], n1 * k1);
                    acc = first ? t : cadd(acc, t);
                    first = false;
                }
                const int e = n2 * k1;
                b[n2][k1] = (e == 0 || first) ? acc : cmul(acc, twiddle<64, DIR>(e));
            }
        }
#pragma unroll
        for (int k1 = 0; k1 < 8; ++k1) {
            float2 u[8];
#pragma unroll
            for (int n2 = 0; n2 < 8; ++n2) u[n2] = b[n2][k1];
            Fft<8, DIR>::run(u);
#pragma unroll
            for (int k2 = 0; k2 < 8; ++k2) a[k1 + 8 * k2] = u[k2];
        }
    }
};

template <int DIR>
struct Fft<16, DIR> {
    __device__ __forceinline__ static void run(float2 (&a)[16]) { FftComposite<16, 4, DIR>::run(a); }
};
template <int DIR>
struct Fft<32, DIR> {
    __device__ __forceinline__ static void run(float2 (&a)[32]) { FftComposite<32, 8, DIR>::run(a); }
};
template <int DIR>
struct Fft<64, DIR> {
    __device__ __forceinline__ static void run(float2 (&a)[64]) { FftComposite<64, 8, DIR>::run(a); }
};

}  // namespace sst
