// sngb_metric.cu -- the Manhattan and cosine metrics of Distance::within, and
// the Euclidean one for rows wider than the specialised gathers (d > 1024)
// (proj/include/sng/distance.hpp:55-68, 75-84, 91-103) on the sampled-graph
// path.  Same structure as k_gather (draws regenerated from their counters,
// live pairs compacted per 32-draw chunk, dynamic row claiming), one G-lane
// group per pair with scalar fp32 loads:
//   Manhattan  s32 = sum |a_k - b_k|              filter value s32
//   cosine     c32 = dot32 / (|a|32 |b|32)         filter value -c32
// against the thresholds of make_test (sngb_api.cu), every pair in the band
// re-evaluated in fp64 in the reference's order (exact_within).  The cosine row
// norms come from k_row_norms, which also counts rows whose fp64 norm is zero
// (the reference throws for them: SNGB_ERR_ZERO_VECTOR).
#include <cuda_runtime.h>

#include <cstdint>

#include "sngb_device.cuh"
#include "sngb_epstest.cuh"
#include "sngb_internal.cuh"
#include "sngb_rng.cuh"

namespace sngb {

namespace {

// warp per row: fp32 |row| for the cosine filter; zero fp64 norm count
__global__ void k_row_norms(const TestParams tp, uint64_t n, float* __restrict__ rnorm,
                            unsigned long long* counters) {
    const int lane = threadIdx.x & 31;
    const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    unsigned zero_rows = 0;
    for (uint64_t r = gw; r < n; r += nw) {
        float acc = 0.f;
        bool nonzero = false;  // some a_k^2 != 0 in fp64 <=> the reference's norm != 0
        for (uint32_t k = lane; k < tp.d; k += 32) {
            const float x = tp.pts[r * tp.stride + k];
            acc = fmaf(x, x, acc);
            const double x64 = tp.pts64 ? tp.pts64[r * tp.d + k] : (double)x;
            nonzero |= __dmul_rn(x64, x64) != 0.0;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
        nonzero = __any_sync(kFull, nonzero);
        if (lane == 0) {
            rnorm[r] = sqrtf(acc);
            zero_rows += nonzero ? 0u : 1u;
        }
    }
    if (lane == 0 && zero_rows) atomicAdd(&counters[C_ZERO_ROWS], (unsigned long long)zero_rows);
}

// the pair's filter value: Manhattan sum, or -cosine similarity
template <int METRIC, int G>
__device__ __forceinline__ float pair_value(const TestParams& tp, uint64_t u, uint64_t v, int q) {
    const float* a = tp.pts + u * tp.stride;
    const float* b = tp.pts + v * tp.stride;
    float acc = 0.f;
    for (uint32_t k = q; k < tp.d; k += G) {
        const float x = __ldg(a + k), y = __ldg(b + k);
        if (METRIC == kMetricEuclid) {
            const float t = x - y;
            acc = fmaf(t, t, acc);
        } else {
            acc = METRIC == kMetricManhattan ? acc + fabsf(x - y) : fmaf(x, y, acc);
        }
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
    if (METRIC != kMetricCosine) return acc;
    return -(acc / (__ldg(tp.rnorm + u) * __ldg(tp.rnorm + v)));  // NaN for a zero fp32 norm
}

template <int METRIC, int G, bool EXH>
__global__ void __launch_bounds__(256) k_gather_metric(const GatherArgs a) {
    constexpr int NG = 32 / G;
    __shared__ unsigned long long s_stage[kWarpsPerBlock][kStage];
    __shared__ uint32_t s_list[kWarpsPerBlock][32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int q = lane % G, g = lane / G;
    const uint64_t gw = (uint64_t)blockIdx.x * kWarpsPerBlock + wib;
    const uint64_t nw = (uint64_t)gridDim.x * kWarpsPerBlock;
    const uint32_t plo = a.part_lo, phi = a.part_hi;
    uint32_t* list = s_list[wib];
    WarpStage<kStage> stage{s_stage[wib], 0};
    TestStats st;
    unsigned long long gpairs = 0;

    uint64_t u = a.row_begin + gw, chunk_end = a.row_end;
    auto grab = [&]() {
        unsigned long long b0 = 0;
        if (lane == 0) b0 = atomicAdd(a.work, (unsigned long long)a.grab);
        b0 = __shfl_sync(kFull, b0, 0);
        u = a.row_begin + b0;
        chunk_end = u + a.grab < a.row_end ? u + a.grab : a.row_end;
    };
    if (a.work) grab();
    for (; u < chunk_end; (a.work && u + 1 >= chunk_end) ? grab() : (void)(u += a.work ? 1 : nw)) {
        uint32_t limit = EXH ? (a.exh_low ? a.exh_low : (uint32_t)(a.n - 1 - u)) : a.draws;
        uint64_t z = EXH ? 0ull : vertex_key(a.seed_mixed, u) + (uint64_t)(lane + 1) * kGamma;
        for (uint32_t i0 = 0; i0 < limit; i0 += 32, z += 32ull * kGamma) {
            const uint32_t i = i0 + lane;
            uint32_t p;
            if (EXH) {
                p = a.exh_low ? i : (uint32_t)u + 1 + i;
            } else {
                const bool valid = i < limit;
                bool fire = false;
                uint32_t t = 0;
                if (valid) {
                    t = lemire32(mix(z), a.base + i + 1, fire);
                    fire |= test_fire(a.force_mod, u, i, a.draws);
                }
                p = t + (t >= (uint32_t)u ? 1u : 0u);
                const unsigned fm = __ballot_sync(kFull, valid && fire);
                if (fm) limit = i0 + __ffs(fm) - 1;  // irregular vertex: cut here
            }
            const bool live = i < limit && p >= plo && p < phi;
            const unsigned m = __ballot_sync(kFull, live);
            if (live) list[__popc(m & lanemask_lt())] = p;
            const uint32_t nlive = __popc(m);
            __syncwarp();
            for (uint32_t j0 = 0; j0 < nlive; j0 += NG) {
                const uint32_t j = j0 + g;
                const bool ok = j < nlive;
                const uint32_t v = list[ok ? j : j0];
                const float val = pair_value<METRIC, G>(a.tp, u, v, q);
                const bool acc = decide(val, ok, q == 0, g * G, a.tp, u, v, st);
                if (ok && q == 0) ++gpairs;
                stage.push(q == 0 && acc, edge_key(u, v, a.sink.nb), a.sink, lane);
            }
            __syncwarp();
        }
    }
    stage.flush(a.sink, lane);
    st.pairs = gpairs;
    flush_stats(st, gpairs, a.counters, lane);
}

// explicit (u, v) pairs (the Floyd replacements), one G-lane group per pair
template <int METRIC, int G>
__global__ void __launch_bounds__(256) k_extras_metric(const ExtrasArgs a) {
    constexpr int NG = 32 / G;
    __shared__ unsigned long long s_stage[kWarpsPerBlock][kStage];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int q = lane % G, g = lane / G;
    const uint64_t gw = (uint64_t)blockIdx.x * kWarpsPerBlock + wib;
    const uint64_t nw = (uint64_t)gridDim.x * kWarpsPerBlock;
    WarpStage<kStage> stage{s_stage[wib], 0};
    TestStats st;
    uint64_t count = *a.count_ptr;
    if (count > a.capacity) count = a.capacity;
    for (uint64_t b = gw * NG; b < count; b += nw * NG) {
        const uint64_t pi = b + g;
        const bool ok = pi < count;
        const unsigned long long rec = a.extras[ok ? pi : b];
        const uint64_t u = rec >> 32, v = rec & 0xffffffffull;
        const float val = pair_value<METRIC, G>(a.tp, u, v, q);
        const bool acc = decide(val, ok, q == 0, g * G, a.tp, u, v, st);
        if (ok && q == 0) st.pairs++;
        stage.push(q == 0 && acc, edge_key(u, v, a.sink.nb), a.sink, lane);
    }
    stage.flush(a.sink, lane);
    flush_stats(st, 0, a.counters, lane);
}

unsigned grid_for_rows(uint64_t rows, int num_sms) {
    uint64_t want = (rows + kWarpsPerBlock - 1) / kWarpsPerBlock;
    const uint64_t cap = (uint64_t)num_sms * 8;
    return (unsigned)(want < cap ? (want ? want : 1) : cap);
}

template <int METRIC, int G>
cudaError_t gather_metric_one(const GatherArgs& a, bool exh, cudaStream_t s, int num_sms) {
    const unsigned grid = grid_for_rows(a.row_end - a.row_begin, num_sms);
    if (exh) k_gather_metric<METRIC, G, true><<<grid, 256, 0, s>>>(a);
    else k_gather_metric<METRIC, G, false><<<grid, 256, 0, s>>>(a);
    note_launch(1);
    return cudaGetLastError();
}

template <int METRIC, int G>
cudaError_t extras_metric_one(const ExtrasArgs& a, cudaStream_t s, int num_sms) {
    const unsigned grid = grid_for_rows((a.capacity + 32 / G - 1) / (32 / G), num_sms);
    k_extras_metric<METRIC, G><<<grid, 256, 0, s>>>(a);
    note_launch(1);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_row_norms(const TestParams& tp, uint64_t n, float* rnorm,
                             unsigned long long* counters, cudaStream_t s, int num_sms) {
    k_row_norms<<<grid_for_rows(n, num_sms), 256, 0, s>>>(tp, n, rnorm, counters);
    note_launch(1);
    return cudaGetLastError();
}

// G = 8 lanes per pair for d <= 64, a warp for wider rows
cudaError_t launch_gather_metric(const GatherArgs& a, bool exhaustive, cudaStream_t s,
                                 int num_sms) {
    if (a.row_end <= a.row_begin) return cudaSuccess;
    const bool wide = a.tp.d > 64;
    if (a.tp.metric == kMetricEuclid)  // d > 1024 (the specialised gathers stop there)
        return gather_metric_one<kMetricEuclid, 32>(a, exhaustive, s, num_sms);
    if (a.tp.metric == kMetricManhattan)
        return wide ? gather_metric_one<kMetricManhattan, 32>(a, exhaustive, s, num_sms)
                    : gather_metric_one<kMetricManhattan, 8>(a, exhaustive, s, num_sms);
    return wide ? gather_metric_one<kMetricCosine, 32>(a, exhaustive, s, num_sms)
                : gather_metric_one<kMetricCosine, 8>(a, exhaustive, s, num_sms);
}

cudaError_t launch_extras_metric(const ExtrasArgs& a, cudaStream_t s, int num_sms) {
    if (a.capacity == 0) return cudaSuccess;
    const bool wide = a.tp.d > 64;
    if (a.tp.metric == kMetricEuclid) return extras_metric_one<kMetricEuclid, 32>(a, s, num_sms);
    if (a.tp.metric == kMetricManhattan)
        return wide ? extras_metric_one<kMetricManhattan, 32>(a, s, num_sms)
                    : extras_metric_one<kMetricManhattan, 8>(a, s, num_sms);
    return wide ? extras_metric_one<kMetricCosine, 32>(a, s, num_sms)
                : extras_metric_one<kMetricCosine, 8>(a, s, num_sms);
}

}  // namespace sngb
