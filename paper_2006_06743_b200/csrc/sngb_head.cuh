// sngb_head.cuh -- device helpers of the head filter (sngb_head.cu), shared with
// the fused Floyd + head gather kernel (sngb_floyd_bloom.cuh).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "sngb_epstest.cuh"
#include "sngb_internal.cuh"

namespace sngb {

__device__ __forceinline__ F4x2 ldg_row2_ef(const float4* p, uint64_t pol) {
    F4x2 r;
    asm("ld.global.nc.L2::cache_hint.v2.b64 {%0, %1}, [%2], %3;" : "=l"(r.lo), "=l"(r.hi) : "l"(p), "l"(pol));
    return r;
}

// the head's Q = sum dq^2: exact (integer) for 8-bit heads, fp32 for 16-bit ones
template <int KIND>
__device__ __forceinline__ float head_q(uint32_t a, uint32_t b) {
    if constexpr (KIND == kHeadU16x2) {
        const float dx = (float)((int)(a & 0xffffu) - (int)(b & 0xffffu));
        const float dy = (float)((int)(a >> 16) - (int)(b >> 16));
        return __fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy));
    } else {
        const uint32_t ad = __vabsdiffu4(a, b);
        return (float)__dp4a(ad, ad, 0u);
    }
}
template <int KIND>
__device__ __forceinline__ uint32_t head_load(const void* h, uint32_t r) {
    if constexpr (KIND == kHeadU8x2) return __ldg(static_cast<const unsigned short*>(h) + r);
    else return __ldg(static_cast<const uint32_t*>(h) + r);
}

// The same load with a 32-bit row index scaled in one IMAD.WIDE (the plain
// pointer arithmetic above compiles to a 64-bit add chain when r is a select).
template <int KIND>
__device__ __forceinline__ uint32_t head_load32(const void* h, uint32_t r) {
    const unsigned long long base = reinterpret_cast<unsigned long long>(h);
    unsigned long long a;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(a) : "r"(r), "r"(KIND == kHeadU8x2 ? 2u : 4u), "l"(base));
    if constexpr (KIND == kHeadU8x2) return __ldg(reinterpret_cast<const unsigned short*>(a));
    else return __ldg(reinterpret_cast<const uint32_t*>(a));
}

}  // namespace sngb
