// Shared device helpers of the fused kernels (forward fwd_kernel.cuh, inverse inv_kernel.cuh):
// CTA geometry, group barriers, TMA bulk-copy / mbarrier PTX wrappers, normalisation lookup.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "decide.cuh"
#include "fft.cuh"
#include "sst_internal.h"

namespace sst {

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
#ifdef SST_BOUNDS
    // bounded spin: a TMA completion that never arrives (bad byte count / address) traps
    for (long long spin = 0;; ++spin) {
        uint32_t done;
        asm volatile(
            "{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
            : "=r"(done) : "r"(smem_u32(bar)), "r"(parity) : "memory");
        if (done) return;
        SST_CHECK(spin < (1ll << 26));
    }
#endif
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

}  // namespace sst
