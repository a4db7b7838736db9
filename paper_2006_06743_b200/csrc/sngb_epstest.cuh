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
// Distance::within for Manhattan / cosine (distance.hpp:55-68, 91-103), fp64 in
// the reference's order.  Zero-norm rows never get here (SNGB_ERR_ZERO_VECTOR).
template <class Row>
__device__ __forceinline__ bool exact_within_metric(int metric, uint32_t d, double eps,
                                                    const Row* a, const Row* b) {
    if (metric == kMetricManhattan) {
        double s = 0.0;
        for (uint32_t k = 0; k < d; ++k) s = __dadd_rn(s, fabs(__dsub_rn(a[k], b[k])));
        return s <= eps;
    }
    double dot = 0.0, na = 0.0, nb = 0.0;
    for (uint32_t k = 0; k < d; ++k) {
        const double x = a[k], y = b[k];
        dot = __dadd_rn(dot, __dmul_rn(x, y));
        na = __dadd_rn(na, __dmul_rn(x, x));
        nb = __dadd_rn(nb, __dmul_rn(y, y));
    }
    double c = __ddiv_rn(dot, __dmul_rn(__dsqrt_rn(na), __dsqrt_rn(nb)));
    if (c > 1.0) c = 1.0;
    if (c < -1.0) c = -1.0;
    return __dsub_rn(1.0, c) <= eps;
}

// The exact decision (rarely taken): scalar arguments, so a caller holding the
// test parameters in its kernel-parameter block does not marshal the struct.
// fp64 input: on the caller's fp64 rows, exactly as the reference does.
static __device__ __noinline__ bool exact_core(const float* pts, uint32_t stride, uint32_t d,
                                               double eps2, double eps, const double* pts64,
                                               int metric, uint64_t u, uint64_t v) {
    if (metric != kMetricEuclid) {
        if (pts64) return exact_within_metric(metric, d, eps, pts64 + u * d, pts64 + v * d);
        return exact_within_metric(metric, d, eps, pts + u * stride, pts + v * stride);
    }
    double s = 0.0;
    if (pts64) {
        const double* a = pts64 + u * d;
        const double* b = pts64 + v * d;
        for (uint32_t k = 0; k < d; ++k) {
            const double t = __dsub_rn(a[k], b[k]);
            s = __dadd_rn(s, __dmul_rn(t, t));
        }
    } else {
        const float* a = pts + u * stride;
        const float* b = pts + v * stride;
        for (uint32_t k = 0; k < d; ++k) {
            const double t = __dsub_rn((double)a[k], (double)b[k]);
            s = __dadd_rn(s, __dmul_rn(t, t));
        }
    }
    return s <= eps2;
}

__device__ __forceinline__ bool exact_within(const TestParams& tp, uint64_t u, uint64_t v) {
    return exact_core(tp.pts, tp.stride, tp.d, tp.eps2, tp.eps, tp.pts64, tp.metric, u, v);
}

struct TestStats {
    unsigned long long pairs = 0, band = 0, band6 = 0, flips = 0;
};

// A pair the filter cannot decide: appended to the band list (k_band decides it
// exactly later and emits the edge if the reference accepts it).
__device__ __forceinline__ void band_push(const TestParams& tp, uint64_t u, uint64_t v, float s) {
    const unsigned long long slot = atomicAdd(tp.band_cursor, 1ull);
    if (slot < tp.band_cap)
        tp.band[slot] = make_uint4((uint32_t)u, (uint32_t)v, __float_as_uint(s), 0u);
}

// Filter decision of one pair per G-lane group (`s` group-uniform): true iff
// the pair is accepted outright; a band pair is handed to k_band and reads as
// not accepted here.
__device__ __forceinline__ bool decide(float s, bool ok, bool leader, int leader_lane,
                                       const TestParams& tp, uint64_t u, uint64_t v,
                                       TestStats& st) {
    (void)leader_lane;
    const bool need = ok && !(s < tp.lo_thr) && !(s > tp.hi_thr);
    if (need && leader) {
        band_push(tp, u, v, s);
        st.band++;
    }
    return ok && (s < tp.lo_thr);
}

// Same when every lane owns one pair.
__device__ __forceinline__ bool decide_lane(float s, bool ok, const TestParams& tp, uint64_t u,
                                            uint64_t v, TestStats& st) {
    const bool need = ok && !(s < tp.lo_thr) && !(s > tp.hi_thr);
    if (need) {
        band_push(tp, u, v, s);
        st.band++;
    }
    return ok && (s < tp.lo_thr);
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
