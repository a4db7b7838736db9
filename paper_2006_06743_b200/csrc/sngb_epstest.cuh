// sngb_epstest.cuh -- the exact eps-test shared by the gather kernels:
// row loads, fp32 accumulate, guard-band decision, fp64 recheck in the
// reference's operation order (distance.hpp:75-83).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "sngb_device.cuh"
#include "sngb_internal.cuh"

namespace sngb {

__device__ __forceinline__ float4 ldg_row(const float4* p) { return __ldg(p); }
__device__ __forceinline__ float2 ldg_row(const float2* p) { return __ldg(p); }
// Query rows are read once per vertex (per phase): keep them out of L1 and
// mark them evict-first in L2 so they do not displace partner rows.
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ float4 ldg_stream(const float4* p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p), "l"(evict_first_policy()));
    return r;
}
__device__ __forceinline__ float2 ldg_stream(const float2* p) {
    float2 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;"
                 : "=f"(r.x), "=f"(r.y) : "l"(p), "l"(evict_first_policy()));
    return r;
}
template <typename Vec>
__device__ __forceinline__ Vec vzero();
template <>
__device__ __forceinline__ float4 vzero<float4>() { return make_float4(0.f, 0.f, 0.f, 0.f); }
template <>
__device__ __forceinline__ float2 vzero<float2>() { return make_float2(0.f, 0.f); }

__device__ __forceinline__ float diff2(float4 a, float4 b, float acc) {
    float t = a.x - b.x;
    acc = fmaf(t, t, acc);
    t = a.y - b.y;
    acc = fmaf(t, t, acc);
    t = a.z - b.z;
    acc = fmaf(t, t, acc);
    t = a.w - b.w;
    return fmaf(t, t, acc);
}
__device__ __forceinline__ float diff2(float2 a, float2 b, float acc) {
    float t = a.x - b.x;
    acc = fmaf(t, t, acc);
    t = a.y - b.y;
    return fmaf(t, t, acc);
}

// Packed-pair variant (sm_100 FADD2/FFMA2): a 16-byte row chunk as two
// f32x2 registers; half the FP instructions of diff2 and two independent
// accumulator pairs instead of one serial chain.  Any summation order and
// fusing is inside the guard band (make_test).
struct F4x2 {
    unsigned long long lo, hi;  // {x, y}, {z, w}
};
__device__ __forceinline__ F4x2 ldg_row2(const float4* p) {
    F4x2 r;
    asm("ld.global.nc.v2.b64 {%0, %1}, [%2];" : "=l"(r.lo), "=l"(r.hi) : "l"(p));
    return r;
}
__device__ __forceinline__ F4x2 to_x2(float4 v) {
    F4x2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r.lo) : "f"(v.x), "f"(v.y));
    asm("mov.b64 %0, {%1, %2};" : "=l"(r.hi) : "f"(v.z), "f"(v.w));
    return r;
}
// 8-byte rows (d <= 2): one f32x2 register per row.
__device__ __forceinline__ unsigned long long ldg_b64(const float2* p) {
    unsigned long long r;
    asm("ld.global.nc.b64 %0, [%1];" : "=l"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ unsigned long long ldg_b64(const float4*) { return 0; }  // unused
__device__ __forceinline__ F4x2 ldg_row2(const float2*) { return F4x2{0, 0}; }      // unused
__device__ __forceinline__ unsigned long long to_x1(float2 v) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(v.x), "f"(v.y));
    return r;
}
__device__ __forceinline__ unsigned long long to_x1(float4) { return 0; }  // unused
__device__ __forceinline__ F4x2 to_x2(float2) { return F4x2{0, 0}; }       // unused
__device__ __forceinline__ void diff1x2(unsigned long long a, unsigned long long b,
                                        unsigned long long& acc) {
    unsigned long long d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(acc) : "l"(d));
}
__device__ __forceinline__ float acc1_sum(unsigned long long acc) {
    float x, y;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(acc));
    return x + y;
}
struct Acc2 {
    unsigned long long xy = 0, zw = 0;  // two f32x2 accumulators (+0.0f each)
};
__device__ __forceinline__ void diff2x2(const F4x2& a, const F4x2& b, Acc2& acc) {
    unsigned long long d0, d1;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d0) : "l"(a.lo), "l"(b.lo));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d1) : "l"(a.hi), "l"(b.hi));
    asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(acc.xy) : "l"(d0));
    asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(acc.zw) : "l"(d1));
}
__device__ __forceinline__ float acc2_sum(const Acc2& acc) {
    float x, y, z, w;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(acc.xy));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(z), "=f"(w) : "l"(acc.zw));
    return (x + y) + (z + w);
}

// Canonical key of the undirected edge {u, v} (graph.cpp:183-186: min, max).
__device__ __forceinline__ unsigned long long edge_key(uint64_t u, uint64_t v, uint32_t nb) {
    const uint64_t a = u < v ? u : v, b = u < v ? v : u;
    return (a << nb) | b;
}

// distance.hpp:75-83 verbatim in fp64: s += (a_k - b_k)^2 sequentially in k,
// no contraction (explicit _rn intrinsics), then s <= eps*eps.
// fp64 input: on the caller's fp64 rows, exactly as the reference does.
static __device__ __noinline__ bool exact_within(const TestParams tp, uint64_t u, uint64_t v) {
    double s = 0.0;
    if (tp.pts64) {
        const double* a = tp.pts64 + u * tp.d;
        const double* b = tp.pts64 + v * tp.d;
        for (uint32_t k = 0; k < tp.d; ++k) {
            const double t = __dsub_rn(a[k], b[k]);
            s = __dadd_rn(s, __dmul_rn(t, t));
        }
    } else {
        const float* a = tp.pts + u * tp.stride;
        const float* b = tp.pts + v * tp.stride;
        for (uint32_t k = 0; k < tp.d; ++k) {
            const double t = __dsub_rn((double)a[k], (double)b[k]);
            s = __dadd_rn(s, __dmul_rn(t, t));
        }
    }
    return s <= tp.eps2;
}

struct TestStats {
    unsigned long long pairs = 0, band = 0, band6 = 0, flips = 0;
};

// Decide one pair per G-lane group.  `s` is group-uniform.  Returns the exact
// reference decision to every lane.  Must be called by all 32 lanes.
__device__ __forceinline__ bool decide(float s, bool ok, bool leader, int leader_lane,
                                       const TestParams& tp, uint64_t u, uint64_t v,
                                       TestStats& st) {
    const bool need = ok && !(s < tp.lo_thr) && !(s > tp.hi_thr);
    bool acc = ok && (s < tp.lo_thr);
    const unsigned nm = __ballot_sync(kFull, need);
    if (nm) {
        bool ex = false;
        if (need && leader) {
            ex = exact_within(tp, u, v);
            st.band++;
            if (fabsf(s - tp.eps2f) <= 1e-6f * tp.eps2f) st.band6++;
            if ((s <= tp.eps2f) != ex) st.flips++;
        }
        ex = __shfl_sync(kFull, ex, leader_lane);
        if (need) acc = ex;
    }
    return acc;
}

// Same decision when every lane owns one pair (no group broadcast needed).
__device__ __forceinline__ bool decide_lane(float s, bool ok, const TestParams& tp, uint64_t u,
                                            uint64_t v, TestStats& st) {
    const bool need = ok && !(s < tp.lo_thr) && !(s > tp.hi_thr);
    bool acc = ok && (s < tp.lo_thr);
    if (need) {
        acc = exact_within(tp, u, v);
        st.band++;
        if (fabsf(s - tp.eps2f) <= 1e-6f * tp.eps2f) st.band6++;
        if ((s <= tp.eps2f) != acc) st.flips++;
    }
    return acc;
}

__device__ __forceinline__ void flush_stats(const TestStats& st, unsigned long long gpairs,
                                            unsigned long long* counters, int lane) {
    const unsigned long long p = warp_sum(st.pairs), b = warp_sum(st.band),
                             b6 = warp_sum(st.band6), f = warp_sum(st.flips),
                             gp = warp_sum(gpairs);
    if (lane == 0) {
        if (p) atomicAdd(&counters[C_PAIRS], p);
        if (b) atomicAdd(&counters[C_BAND], b);
        if (b6) atomicAdd(&counters[C_BAND6], b6);
        if (f) atomicAdd(&counters[C_FLIPS], f);
        if (gp) atomicAdd(&counters[C_GATHER_PAIRS], gp);
    }
}

}  // namespace sngb
