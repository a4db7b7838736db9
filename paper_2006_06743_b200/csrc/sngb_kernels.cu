// sngb_kernels.cu -- sm_100a kernels of the sampled eps-graph build.
//
// Reference being replaced: sng::build_sampled_graph, proj/src/graph.cpp:133-189
// (per-vertex Floyd sampler :161-174, eps-test :152-155 -> distance.hpp:75-83,
// symmetrise :181-187).  Three kernels, one per role:
//
//   k_sampler  Floyd bookkeeping only (no point data): finds, per vertex, the
//              draws whose value t was already chosen and emits their Floyd
//              replacement j as an "extra" pair; vertices whose stream hits
//              the Lemire reject pre-condition are replayed exactly
//              (sequential Stream) and all their partners become extras.
//              Integer / shared-memory bound.
//   k_gather   THE hot kernel: every draw t_i of every vertex is regenerated
//              from its counter (stateless), the partner row is gathered with
//              16-byte vector loads by a G-lane group, the squared distance is
//              accumulated in fp32 and decided against a rigorous guard band;
//              in-band pairs are re-evaluated in the reference's exact fp64
//              order.  Accepted pairs are compacted (ballot + popc) into a
//              per-warp shared-memory stage and flushed with one atomic per
//              ~32 edges.  HBM/L2-gather bound.
//   k_extras   the same eps-test over the sampler's extra pairs.
//
// Why this split reproduces the reference's edge set exactly: for a regular
// vertex the Floyd set is S = {t_i} U {j_i : draw i collided} (SURVEY.md
// Appendix C); k_gather tests every t_i (a duplicated t only re-emits an edge
// that dedup removes), k_extras tests the j_i.  For an irregular vertex
// k_gather stops at the first fired draw (earlier draws used the same
// counters, so their t are members of S) and k_sampler emits all of S.
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "sngb_internal.cuh"
#include "sngb_rng.cuh"

namespace sngb {

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

__device__ __forceinline__ float4 ldg_row(const float4* p) { return __ldg(p); }
__device__ __forceinline__ float2 ldg_row(const float2* p) { return __ldg(p); }
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

// Canonical key of the undirected edge {u, v} (graph.cpp:183-186: min, max).
__device__ __forceinline__ unsigned long long edge_key(uint64_t u, uint64_t v, uint32_t nb) {
    const uint64_t a = u < v ? u : v, b = u < v ? v : u;
    return (a << nb) | b;
}

// distance.hpp:75-83 verbatim in fp64: s += (a_k - b_k)^2 sequentially in k,
// no contraction (explicit _rn intrinsics), then s <= eps*eps.
__device__ __noinline__ bool exact_within(const TestParams tp, uint64_t u, uint64_t v) {
    const float* a = tp.pts + u * tp.stride;
    const float* b = tp.pts + v * tp.stride;
    double s = 0.0;
    for (uint32_t k = 0; k < tp.d; ++k) {
        const double t = __dsub_rn((double)a[k], (double)b[k]);
        s = __dadd_rn(s, __dmul_rn(t, t));
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

// Per-warp shared-memory staging of 64-bit records with batched flushes
// (one global atomic per flush instead of one per record).
template <int STAGE>
struct WarpStage {
    unsigned long long* buf;
    int count;

    __device__ __forceinline__ void flush(const EdgeSink& s, int lane) {
        __syncwarp();
        if (count == 0) return;
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(s.cursor, (unsigned long long)count);
        base = __shfl_sync(kFull, base, 0);
        for (int j = lane; j < count; j += 32)
            if (base + j < s.capacity) s.keys[base + j] = buf[j];
        __syncwarp();
        count = 0;
    }

    __device__ __forceinline__ void push(bool has, unsigned long long rec, const EdgeSink& s,
                                         int lane) {
        const unsigned m = __ballot_sync(kFull, has);
        if (!m) return;
        if (has) buf[count + __popc(m & lanemask_lt())] = rec;
        count += __popc(m);
        if (count > STAGE - 32) flush(s, lane);
    }
};

constexpr int kStage = 128;
constexpr int kWarpsPerBlock = 8;

__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
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

// Pairs per group issued back to back (loads in flight per lane = U * V).
template <int G, int V>
struct Unroll {
    static constexpr int value = G < 32 ? G : (V == 1 ? 8 : (V == 2 ? 4 : 2));
};

// ---------------------------------------------------------------------------
// k_gather: one warp per query vertex (grid-stride), G lanes per partner row,
// each lane holding V vector chunks of the query row in registers.
//   EXH = false: partners are the Floyd draws t_i (graph.cpp:167-174)
//   EXH = true : partners are all v > u (draws >= n-1, graph.cpp:157-159;
//                each unordered pair once -- same edge set)
// ---------------------------------------------------------------------------
template <int G, int V, int R, bool F2, bool EXH>
__global__ void __launch_bounds__(256) k_gather(const GatherArgs a) {
    using Vec = typename std::conditional<F2, float2, float4>::type;
    constexpr int NG = 32 / G;
    constexpr int U = Unroll<G, V>::value;
    __shared__ unsigned long long s_stage[kWarpsPerBlock][kStage];

    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int q = lane % G, g = lane / G;
    const int leader_lane = g * G;
    const bool leader = (q == 0);
    const uint64_t gw = (uint64_t)blockIdx.x * kWarpsPerBlock + wib;
    const uint64_t nw = (uint64_t)gridDim.x * kWarpsPerBlock;
    const Vec* __restrict__ P = reinterpret_cast<const Vec*>(a.tp.pts);
    const uint32_t W = a.tp.stride / (F2 ? 2 : 4);

    WarpStage<kStage> stage{s_stage[wib], 0};
    TestStats st;
    unsigned long long gpairs = 0;

    for (uint64_t u = a.row_begin + gw; u < a.row_end; u += nw) {
        Vec qv[V];
#pragma unroll
        for (int vv = 0; vv < V; ++vv) {
            const uint32_t c = q + G * vv;
            qv[vv] = (c < W) ? ldg_row(P + u * W + c) : vzero<Vec>();
        }
        uint32_t limit = EXH ? (uint32_t)(a.n - 1 - u) : a.draws;
        const uint64_t key = EXH ? 0ull : vertex_key(a.seed_mixed, u);

        for (uint32_t i0 = 0; i0 < limit; i0 += 32 * R) {
            uint32_t pv[R];
            unsigned vm[R];
            if (EXH) {
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    const uint32_t i = i0 + 32 * k + lane;
                    pv[k] = (uint32_t)u + 1 + i;
                    vm[k] = __ballot_sync(kFull, i < limit);
                }
            } else {
                uint32_t first_fire = 0xffffffffu;
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    const uint32_t i = i0 + 32 * k + lane;
                    const bool valid = i < limit;
                    bool fire = false;
                    uint32_t t = 0;
                    if (valid) t = lemire32(stream_at(key, (uint64_t)i + 1), a.base + i + 1, fire);
                    pv[k] = t + (t >= (uint32_t)u ? 1u : 0u);
                    const unsigned fm = __ballot_sync(kFull, valid && fire);
                    if (fm && first_fire == 0xffffffffu) first_fire = i0 + 32 * k + __ffs(fm) - 1;
                }
                if (first_fire != 0xffffffffu) limit = first_fire;  // irregular: cut here
#pragma unroll
                for (int k = 0; k < R; ++k) vm[k] = __ballot_sync(kFull, i0 + 32 * k + lane < limit);
            }

#pragma unroll
            for (int k = 0; k < R; ++k) {
                if (vm[k] == 0) continue;
#pragma unroll 1
                for (int m0 = 0; m0 < G; m0 += U) {
                    Vec rows[U][V];
                    uint32_t pvv[U];
                    bool ok[U];
#pragma unroll
                    for (int uu = 0; uu < U; ++uu) {
                        const int src = (G == 1) ? lane : (g + NG * (m0 + uu));
                        pvv[uu] = (G == 1) ? pv[k] : __shfl_sync(kFull, pv[k], src);
                        ok[uu] = (vm[k] >> src) & 1u;
#pragma unroll
                        for (int vv = 0; vv < V; ++vv) {
                            const uint32_t c = q + G * vv;
                            rows[uu][vv] = (ok[uu] && c < W) ? ldg_row(P + (uint64_t)pvv[uu] * W + c)
                                                             : vzero<Vec>();
                        }
                    }
#pragma unroll
                    for (int uu = 0; uu < U; ++uu) {
                        float s = 0.f;
#pragma unroll
                        for (int vv = 0; vv < V; ++vv) s = diff2(qv[vv], rows[uu][vv], s);
#pragma unroll
                        for (int o = G / 2; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
                        const bool acc = decide(s, ok[uu], leader, leader_lane, a.tp, u, pvv[uu], st);
                        if (ok[uu] && leader) ++gpairs;
                        stage.push(leader && acc, edge_key(u, pvv[uu], a.sink.nb), a.sink, lane);
                    }
                }
            }
        }
    }
    stage.flush(a.sink, lane);
    st.pairs = gpairs;
    flush_stats(st, gpairs, a.counters, lane);
}

// ---------------------------------------------------------------------------
// k_extras: eps-test of explicit (u, v) pairs, one G-lane group per pair.
// ---------------------------------------------------------------------------
template <int G, int V, bool F2>
__global__ void __launch_bounds__(256) k_extras(const ExtrasArgs a) {
    using Vec = typename std::conditional<F2, float2, float4>::type;
    constexpr int NG = 32 / G;
    __shared__ unsigned long long s_stage[kWarpsPerBlock][kStage];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int q = lane % G, g = lane / G;
    const int leader_lane = g * G;
    const bool leader = (q == 0);
    const uint64_t gw = (uint64_t)blockIdx.x * kWarpsPerBlock + wib;
    const uint64_t nw = (uint64_t)gridDim.x * kWarpsPerBlock;
    const Vec* __restrict__ P = reinterpret_cast<const Vec*>(a.tp.pts);
    const uint32_t W = a.tp.stride / (F2 ? 2 : 4);
    WarpStage<kStage> stage{s_stage[wib], 0};
    TestStats st;
    uint64_t count = *a.count_ptr;
    if (count > a.capacity) count = a.capacity;
    for (uint64_t b = gw * NG; b < count; b += nw * NG) {
        const uint64_t p = b + g;
        const bool ok = p < count;
        const unsigned long long rec = ok ? a.extras[p] : 0ull;
        const uint64_t u = rec >> 32, v = rec & 0xffffffffull;
        float s = 0.f;
#pragma unroll
        for (int vv = 0; vv < V; ++vv) {
            const uint32_t c = q + G * vv;
            if (ok && c < W) s = diff2(ldg_row(P + u * W + c), ldg_row(P + v * W + c), s);
        }
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
        const bool acc = decide(s, ok, leader, leader_lane, a.tp, u, v, st);
        if (ok && leader) st.pairs++;
        stage.push(leader && acc, edge_key(u, v, a.sink.nb), a.sink, lane);
    }
    stage.flush(a.sink, lane);
    flush_stats(st, 0, a.counters, lane);
}

// ---------------------------------------------------------------------------
// k_sampler: Floyd bookkeeping (graph.cpp:164-170), one warp per vertex,
// draws processed 32 at a time in order with a per-warp membership table
// (bitmap over [0, n-1) when that is smaller, else an open-addressing hash of
// the chosen values).  Membership is "value already chosen by an earlier
// draw": earlier chunks via the table, earlier lanes of this chunk via
// match.any, and the rare j-chain (t equal to the replacement j of an earlier
// collided lane of the same chunk) by an in-order lane scan.
// ---------------------------------------------------------------------------
template <bool BITMAP>
__device__ __forceinline__ bool table_contains(const uint32_t* tab, uint32_t x,
                                               const SamplerArgs& a) {
    if (BITMAP) return (tab[x >> 5] >> (x & 31)) & 1u;
    uint32_t h = (x * 0x9E3779B1u) >> a.hash_shift;
    for (;;) {
        const uint32_t v = tab[h];
        if (v == x) return true;
        if (v == kEmpty) return false;
        h = (h + 1) & a.hash_mask;
    }
}

// Insert a value known to be absent (concurrent inserts of distinct values).
template <bool BITMAP>
__device__ __forceinline__ void table_insert(uint32_t* tab, uint32_t x, const SamplerArgs& a) {
    if (BITMAP) {
        atomicOr(&tab[x >> 5], 1u << (x & 31));
        return;
    }
    uint32_t h = (x * 0x9E3779B1u) >> a.hash_shift;
    for (;;) {
        if (atomicCAS(&tab[h], kEmpty, x) == kEmpty) return;
        h = (h + 1) & a.hash_mask;
    }
}

// Single-thread insert-if-absent (exact sequential fallback).
template <bool BITMAP>
__device__ bool table_insert_seq(uint32_t* tab, uint32_t x, const SamplerArgs& a) {
    if (BITMAP) {
        const uint32_t bit = 1u << (x & 31);
        if (tab[x >> 5] & bit) return false;
        tab[x >> 5] |= bit;
        return true;
    }
    uint32_t h = (x * 0x9E3779B1u) >> a.hash_shift;
    for (;;) {
        const uint32_t v = tab[h];
        if (v == x) return false;
        if (v == kEmpty) {
            tab[h] = x;
            return true;
        }
        h = (h + 1) & a.hash_mask;
    }
}

template <bool BITMAP>
__device__ __forceinline__ void table_clear(uint32_t* tab, uint32_t words, int lane) {
    const uint32_t fill = BITMAP ? 0u : kEmpty;
    uint4* t4 = reinterpret_cast<uint4*>(tab);
    for (uint32_t w = lane; w < words / 4; w += 32) t4[w] = make_uint4(fill, fill, fill, fill);
    __syncwarp();
}

template <bool BITMAP, bool SHARED>
__global__ void __launch_bounds__(256) k_sampler(const SamplerArgs a) {
    extern __shared__ __align__(16) uint32_t smem[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    const uint64_t gw = (uint64_t)blockIdx.x * wpb + wib;
    const uint64_t nw = (uint64_t)gridDim.x * wpb;
    uint32_t* tab = SHARED ? smem + (size_t)wib * a.table_words
                           : a.scratch + gw * (uint64_t)a.table_words;
    unsigned long long* sbuf =
        reinterpret_cast<unsigned long long*>(smem + (SHARED ? (size_t)wpb * a.table_words : 0)) +
        (size_t)wib * kStage;
    const EdgeSink xs{a.extras, a.extras_capacity, &a.counters[C_EXTRA_CURSOR], 0};
    WarpStage<kStage> stage{sbuf, 0};
    unsigned long long ncol = 0, nirr = 0;
    const uint32_t D = a.draws, base = a.base;

    for (uint64_t u = a.row_begin + gw; u < a.row_end; u += nw) {
        table_clear<BITMAP>(tab, a.table_words, lane);
        const uint64_t key = vertex_key(a.seed_mixed, u);
        bool irregular = false;
        for (uint32_t c0 = 0; c0 < D; c0 += 32) {
            const uint32_t i = c0 + lane;
            const bool valid = i < D;
            bool fire = false;
            uint32_t t = 0;
            if (valid) t = lemire32(stream_at(key, (uint64_t)i + 1), base + i + 1, fire);
            if (__ballot_sync(kFull, valid && fire)) {
                irregular = true;
                break;
            }
            const bool in_prev = valid && table_contains<BITMAP>(tab, t, a);
            const unsigned mm = __match_any_sync(kFull, valid ? t : (0xffffffffu - lane));
            const bool dup = (mm & lanemask_lt()) != 0;
            bool col = valid && (in_prev || dup);
            const uint32_t j = base + i;  // Floyd's replacement value for draw i
            if (__ballot_sync(kFull, valid && !col && t >= base + c0 && t < j)) {
                for (int l = 0; l < 31; ++l) {
                    const bool cl = __shfl_sync(kFull, col, l);
                    if (cl && lane > l && valid && !col && t == base + c0 + l) col = true;
                }
            }
            if (valid) table_insert<BITMAP>(tab, col ? j : t, a);
            __syncwarp();
            const unsigned cm = __ballot_sync(kFull, col);
            ncol += (lane == 0) ? __popc(cm) : 0;
            const uint32_t pj = j + (j >= (uint32_t)u ? 1u : 0u);
            stage.push(col, ((unsigned long long)u << 32) | pj, xs, lane);
        }
        if (irregular) {
            // Exact replay of graph.cpp:163-174 with the true Stream (rejections
            // consume extra counters); every partner of u becomes an extra.
            table_clear<BITMAP>(tab, a.table_words, lane);
            if (lane == 0) {
                ++nirr;
                SeqStream s{key, 0};
                const uint64_t pool = a.n - 1;
                for (uint64_t jj = base; jj < pool; ++jj) {
                    const uint32_t t = (uint32_t)s.next_below(jj + 1);
                    uint32_t e = t;
                    if (!table_insert_seq<BITMAP>(tab, t, a)) {
                        table_insert_seq<BITMAP>(tab, (uint32_t)jj, a);
                        e = (uint32_t)jj;
                    }
                    const uint32_t pe = e + (e >= (uint32_t)u ? 1u : 0u);
                    const unsigned long long slot = atomicAdd(xs.cursor, 1ull);
                    if (slot < xs.capacity) xs.keys[slot] = ((unsigned long long)u << 32) | pe;
                }
            }
            __syncwarp();
        }
    }
    stage.flush(xs, lane);
    if (lane == 0) {
        if (ncol) atomicAdd(&a.counters[C_COLLISIONS], ncol);
        if (nirr) atomicAdd(&a.counters[C_IRREGULAR], nirr);
    }
}

// ---------------------------------------------------------------------------
// k_prepare: copy n x d rows into the padded device layout (stride floats)
// and count non-finite values (dataset.hpp:24-26).  With dst == nullptr the
// kernel only checks.
// ---------------------------------------------------------------------------
__global__ void k_prepare(const float* __restrict__ src, float* __restrict__ dst, uint64_t n,
                          uint32_t d, uint32_t stride, unsigned long long* counters) {
    const uint64_t total = dst ? n * stride : n * d;
    unsigned bad = 0;
    for (uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (uint64_t)gridDim.x * blockDim.x) {
        if (dst) {
            const uint64_t r = idx / stride;
            const uint32_t c = (uint32_t)(idx - r * stride);
            float v = 0.f;
            if (c < d) {
                v = src[r * d + c];
                bad += !isfinite(v);
            }
            dst[idx] = v;
        } else {
            bad += !isfinite(src[idx]);
        }
    }
    bad = __reduce_add_sync(kFull, bad);
    if ((threadIdx.x & 31) == 0 && bad) atomicAdd(&counters[C_NONFINITE], (unsigned long long)bad);
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
cudaError_t launch_prepare_points(const float* src, float* dst, uint64_t n, uint32_t d,
                                  uint32_t stride, unsigned long long* counters, cudaStream_t s) {
    const uint64_t total = dst ? n * stride : n * d;
    uint64_t blocks = (total + 255) / 256;
    if (blocks > 148ull * 16) blocks = 148ull * 16;
    if (blocks == 0) blocks = 1;
    k_prepare<<<(unsigned)blocks, 256, 0, s>>>(src, dst, n, d, stride, counters);
    return cudaGetLastError();
}

namespace {

template <typename K>
unsigned persistent_grid(K kernel, uint64_t rows, int num_sms, size_t smem = 0) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 256, smem);
    if (per_sm < 1) per_sm = 1;
    uint64_t want = (rows + kWarpsPerBlock - 1) / kWarpsPerBlock;
    uint64_t cap = (uint64_t)num_sms * per_sm;
    uint64_t g = want < cap ? want : cap;
    return (unsigned)(g ? g : 1);
}

template <int G, int V, int R, bool F2, bool EXH>
cudaError_t gather_one(const GatherArgs& a, cudaStream_t s, int num_sms) {
    auto k = k_gather<G, V, R, F2, EXH>;
    unsigned grid = persistent_grid(k, a.row_end - a.row_begin, num_sms);
    k<<<grid, 256, 0, s>>>(a);
    return cudaGetLastError();
}

template <bool EXH>
cudaError_t gather_dispatch(const GatherArgs& a, cudaStream_t s, int num_sms) {
    if (a.tp.stride == 2) return gather_one<1, 1, 4, true, EXH>(a, s, num_sms);
    const uint32_t W = a.tp.stride / 4;
    if (W == 1) return gather_one<1, 1, 4, false, EXH>(a, s, num_sms);
    if (W <= 2) return gather_one<2, 1, 2, false, EXH>(a, s, num_sms);
    if (W <= 4) return gather_one<4, 1, 1, false, EXH>(a, s, num_sms);
    if (W <= 8) return gather_one<8, 1, 1, false, EXH>(a, s, num_sms);
    if (W <= 16) return gather_one<16, 1, 1, false, EXH>(a, s, num_sms);
    switch ((W + 31) / 32) {
        case 1: return gather_one<32, 1, 1, false, EXH>(a, s, num_sms);
        case 2: return gather_one<32, 2, 1, false, EXH>(a, s, num_sms);
        case 3: return gather_one<32, 3, 1, false, EXH>(a, s, num_sms);
        case 4: return gather_one<32, 4, 1, false, EXH>(a, s, num_sms);
        case 5: return gather_one<32, 5, 1, false, EXH>(a, s, num_sms);
        case 6: return gather_one<32, 6, 1, false, EXH>(a, s, num_sms);
        case 7: return gather_one<32, 7, 1, false, EXH>(a, s, num_sms);
        case 8: return gather_one<32, 8, 1, false, EXH>(a, s, num_sms);
        default: return cudaErrorInvalidValue;  // d > 1024: not supported yet
    }
}

template <int G, int V, bool F2>
cudaError_t extras_one(const ExtrasArgs& a, cudaStream_t s, int num_sms) {
    auto k = k_extras<G, V, F2>;
    constexpr int NG = 32 / G;
    unsigned grid = persistent_grid(k, (a.capacity + NG - 1) / NG, num_sms);
    k<<<grid, 256, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_gather(const GatherArgs& a, bool exhaustive, cudaStream_t s, int num_sms) {
    if (a.row_end <= a.row_begin) return cudaSuccess;
    return exhaustive ? gather_dispatch<true>(a, s, num_sms) : gather_dispatch<false>(a, s, num_sms);
}

cudaError_t launch_extras(const ExtrasArgs& a, cudaStream_t s, int num_sms) {
    if (a.capacity == 0) return cudaSuccess;
    if (a.tp.stride == 2) return extras_one<1, 1, true>(a, s, num_sms);
    const uint32_t W = a.tp.stride / 4;
    if (W == 1) return extras_one<1, 1, false>(a, s, num_sms);
    if (W <= 2) return extras_one<2, 1, false>(a, s, num_sms);
    if (W <= 4) return extras_one<4, 1, false>(a, s, num_sms);
    if (W <= 8) return extras_one<8, 1, false>(a, s, num_sms);
    if (W <= 16) return extras_one<16, 1, false>(a, s, num_sms);
    switch ((W + 31) / 32) {
        case 1: return extras_one<32, 1, false>(a, s, num_sms);
        case 2: return extras_one<32, 2, false>(a, s, num_sms);
        case 3: return extras_one<32, 3, false>(a, s, num_sms);
        case 4: return extras_one<32, 4, false>(a, s, num_sms);
        case 5: return extras_one<32, 5, false>(a, s, num_sms);
        case 6: return extras_one<32, 6, false>(a, s, num_sms);
        case 7: return extras_one<32, 7, false>(a, s, num_sms);
        case 8: return extras_one<32, 8, false>(a, s, num_sms);
        default: return cudaErrorInvalidValue;
    }
}

// Shared-memory budget for the sampler's per-warp tables.
constexpr size_t kSamplerSmemBudget = 200 * 1024;
constexpr size_t kStageBytes = kStage * sizeof(unsigned long long);

bool sampler_uses_shared(size_t table_bytes) { return table_bytes + kStageBytes <= 96 * 1024; }

static int sampler_warps_per_block(size_t table_bytes) {
    int w = (int)(kSamplerSmemBudget / (table_bytes + kStageBytes));
    if (w > kWarpsPerBlock) w = kWarpsPerBlock;
    if (w < 1) w = 1;
    return w;
}

size_t sampler_scratch_bytes(size_t table_bytes, int num_sms) {
    if (sampler_uses_shared(table_bytes)) return 0;
    return (size_t)num_sms * 4 * kWarpsPerBlock * table_bytes;
}

cudaError_t launch_sampler(const SamplerArgs& a, bool bitmap, size_t table_bytes, cudaStream_t s,
                           int num_sms) {
    const uint64_t rows = a.row_end - a.row_begin;
    if (rows == 0 || a.draws == 0) return cudaSuccess;
    if (sampler_uses_shared(table_bytes)) {
        const int wpb = sampler_warps_per_block(table_bytes);
        const size_t smem = (size_t)wpb * (table_bytes + kStageBytes);
        auto k = bitmap ? k_sampler<true, true> : k_sampler<false, true>;
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, wpb * 32, smem);
        if (per_sm < 1) per_sm = 1;
        uint64_t want = (rows + wpb - 1) / wpb, cap = (uint64_t)num_sms * per_sm;
        unsigned grid = (unsigned)(want < cap ? want : cap);
        k<<<grid, wpb * 32, smem, s>>>(a);
    } else {
        // Tables in global memory (L2-resident scratch), fixed warp count.
        auto k = bitmap ? k_sampler<true, false> : k_sampler<false, false>;
        const size_t smem = (size_t)kWarpsPerBlock * kStageBytes;
        uint64_t want = (rows + kWarpsPerBlock - 1) / kWarpsPerBlock, cap = (uint64_t)num_sms * 4;
        unsigned grid = (unsigned)(want < cap ? want : cap);
        k<<<grid, kWarpsPerBlock * 32, smem, s>>>(a);
    }
    return cudaGetLastError();
}

}  // namespace sngb
