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

#include "sngb_device.cuh"
#include "sngb_epstest.cuh"
#include "sngb_internal.cuh"
#include "sngb_rng.cuh"

namespace sngb {

// Pairs per group issued back to back (loads in flight per lane = U * V).
// G < 32: a group takes R*G pairs of each 32*R-draw chunk in one go.
template <int G, int V, int R>
struct Unroll {
    static constexpr int value = G < 32 ? R * G : (V == 1 ? 8 : (V == 2 ? 4 : 2));
};

// ---------------------------------------------------------------------------
// k_gather: one warp per query vertex (grid-stride), G lanes per partner row,
// each lane holding V vector chunks of the query row in registers.
//   EXH = false: partners are the Floyd draws t_i (graph.cpp:167-174)
//   EXH = true : partners are all v > u (draws >= n-1, graph.cpp:157-159;
//                each unordered pair once -- same edge set)
// Each chunk of 32*R draws is compacted (ballot + popc into a per-warp
// shared list) to the pairs that are live: below the irregular cut and with
// the partner row inside [part_lo, part_hi).  The partner range lets the host
// run the gather as L2-blocked phases (one slice of the rows per launch) when
// the row table is a small multiple of L2; a single phase covers [0, n).
// ---------------------------------------------------------------------------
// Resident blocks per SM that ptxas must leave room for.  Wide rows (G = 32)
// get up to 128 registers for two rows in flight per warp (measured:
// 126 registers and 8.8 ms on cfg2 vs 112 and 9.3 ms under the default
// heuristic); narrow rows keep the occupancy their latency-bound gathers need.
#ifndef SNGB_WIDE_MINB
#define SNGB_WIDE_MINB 1
#endif
// A/B build knobs (python -m paper_2006_06743_b200.build --variant ...): cfg1's
// gather measured 0.191 ms at the defaults, 0.216 / 0.229 with 6 / 8 blocks per
// SM, 0.195 / 0.211 with 2 / 8 draw chunks per step
#ifndef SNGB_NARROW_MINB
#define SNGB_NARROW_MINB 4
#endif
#ifndef SNGB_F2_R
#define SNGB_F2_R 4
#endif
template <int G, int V>
struct MinBlocks {
    static constexpr int value =
        G == 32 ? (V == 8 ? 2 : SNGB_WIDE_MINB) : (G == 16 ? 2 : (G == 8 ? 3 : SNGB_NARROW_MINB));
};

template <int G, int V, int R, bool F2, bool EXH>
__global__ void __launch_bounds__(256, MinBlocks<G, V>::value) k_gather(const GatherArgs a) {
    using Vec = typename std::conditional<F2, float2, float4>::type;
    constexpr int NG = 32 / G;
    constexpr int U = Unroll<G, V, R>::value;
    __shared__ unsigned long long s_stage[kWarpsPerBlock][kStage];
    __shared__ uint32_t s_list[kWarpsPerBlock][32 * R];

    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int q = lane % G, g = lane / G;
    const int leader_lane = g * G;
    const bool leader = (q == 0);
    const uint64_t gw = (uint64_t)blockIdx.x * kWarpsPerBlock + wib;
    const uint64_t nw = (uint64_t)gridDim.x * kWarpsPerBlock;
    const Vec* __restrict__ P = reinterpret_cast<const Vec*>(a.tp.pts);
    const uint32_t W = a.tp.stride / (F2 ? 2 : 4);
    const uint32_t plo = a.part_lo, phi = a.part_hi;
    uint32_t* list = s_list[wib];

    WarpStage<kStage> stage{s_stage[wib], 0};
    TestStats st;
    unsigned long long gpairs = 0;

    // Rows: grid-stride, or (a.work) claimed `grab` consecutive rows at a time
    // from a per-launch counter -- dynamic balancing across SMs, whose
    // memory-bound progress differs (a persistent grid-stride split measured
    // 15 % slower on cfg5).
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
        Vec qv[V];
#pragma unroll
        for (int vv = 0; vv < V; ++vv) {
            const uint32_t c = q + G * vv;
            if constexpr (G == 32)
                qv[vv] = (c < W) ? ldg_stream(P + u * W + c) : vzero<Vec>();
            else  // narrow: past the row end, the last column (partners read it too)
                qv[vv] = ldg_row(P + u * W + (c < W ? c : W - 1));
        }
        using QRow = typename std::conditional<F2, unsigned long long, F4x2>::type;
        QRow q2[G < 32 ? V : 1];
        if constexpr (G < 32) {
#pragma unroll
            for (int vv = 0; vv < V; ++vv) {
                if constexpr (F2) q2[vv] = to_x1(qv[vv]);
                else q2[vv] = to_x2(qv[vv]);
            }
        }
        uint32_t limit = EXH ? (a.exh_low ? a.exh_low : (uint32_t)(a.n - 1 - u)) : a.draws;
        // stream_at(key, i + 1) for i = i0 + 32k + lane, carried incrementally
        // (nothing for ptxas to rematerialise from the vertex key per chunk)
        uint64_t z = EXH ? 0ull : vertex_key(a.seed_mixed, u) + (uint64_t)(lane + 1) * kGamma;

        for (uint32_t i0 = 0; i0 < limit; i0 += 32 * R, z += (uint64_t)(32 * R) * kGamma) {
            uint32_t pv[R];
            if (!EXH) {
                uint32_t first_fire = 0xffffffffu;
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    const uint32_t i = i0 + 32 * k + lane;
                    const bool valid = i < limit;
                    bool fire = false;
                    uint32_t t = 0;
                    if (valid) {
                        t = lemire32(mix(z + (uint64_t)(32 * k) * kGamma), a.base + i + 1, fire);
                        fire |= test_fire(a.force_mod, u, i, a.draws);
                    }
                    pv[k] = t + (t >= (uint32_t)u ? 1u : 0u);
                    const unsigned fm = __ballot_sync(kFull, valid && fire);
                    if (fm && first_fire == 0xffffffffu) first_fire = i0 + 32 * k + __ffs(fm) - 1;
                }
                if (first_fire != 0xffffffffu) limit = first_fire;  // irregular: cut here
            }
            if constexpr (G < 32) {
                // Narrow rows: every lane's draw is one pair; group g takes the
                // pairs of lanes g + NG*m straight from registers (no staging).
                // All R*G rows of the chunk are loaded before any is used (a
                // warp-sync fence keeps ptxas from sinking them), so R*G*V
                // 16-byte loads per lane are in flight together.  A masked pair
                // (tail, other partner slice) reads the query row itself, and a
                // lane past the row end reads the row's last column for both
                // query and partner, so neither needs a zero-fill and both add 0.
                constexpr int UG = G;
                uint32_t pvk[R];
                unsigned vmk[R], any = 0;
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    const uint32_t i = i0 + 32 * k + lane;
                    pvk[k] = EXH ? (a.exh_low ? i : (uint32_t)u + 1 + i) : pv[k];
                    vmk[k] = __ballot_sync(kFull, i < limit && pvk[k] >= plo && pvk[k] < phi);
                    any |= vmk[k];
                }
                if (any == 0) continue;
                using Row = typename std::conditional<F2, unsigned long long, F4x2>::type;
                Row rows[R][UG][V];
#pragma unroll
                for (int k = 0; k < R; ++k)
#pragma unroll
                    for (int uu = 0; uu < UG; ++uu) {
                        const int src = (G == 1) ? lane : (g + NG * uu);
                        const uint32_t pp = (G == 1) ? pvk[k] : __shfl_sync(kFull, pvk[k], src);
                        const bool ok = (vmk[k] >> src) & 1u;
#pragma unroll
                        for (int vv = 0; vv < V; ++vv) {
                            const uint32_t c = q + G * vv;
                            const uint64_t row = (ok && c < W) ? pp : u;
                            const Vec* ptr = P + row * W + (c < W ? c : W - 1);
                            if constexpr (F2) rows[k][uu][vv] = ldg_b64(ptr);
                            else rows[k][uu][vv] = ldg_row2(ptr);
                        }
                    }
                __syncwarp();  // scheduling fence (see the wide-row path)
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    // partial sums of the G pairs of this group, then a
                    // transposed reduce-scatter (G-1 shuffles for G pairs instead
                    // of log2(G) per pair): lane q ends with the total of pair q,
                    // so decision, recheck and emission are one lane per pair.
                    float ps[UG];
#pragma unroll
                    for (int uu = 0; uu < UG; ++uu) {
                        if constexpr (F2) {
                            unsigned long long acc = 0;
#pragma unroll
                            for (int vv = 0; vv < V; ++vv) diff1x2(q2[vv], rows[k][uu][vv], acc);
                            ps[uu] = acc1_sum(acc);
                        } else {
                            Acc2 acc;
#pragma unroll
                            for (int vv = 0; vv < V; ++vv) diff2x2(q2[vv], rows[k][uu][vv], acc);
                            ps[uu] = acc2_sum(acc);
                        }
                    }
#pragma unroll
                    for (int o = UG / 2; o > 0; o >>= 1) {
                        const bool hi = (q & o) != 0;
#pragma unroll
                        for (int j = 0; j < o; ++j) {
                            const float mine = hi ? ps[j + o] : ps[j];
                            const float other = hi ? ps[j] : ps[j + o];
                            ps[j] = mine + __shfl_xor_sync(kFull, other, o);
                        }
                    }
                    const int src = (G == 1) ? lane : (g + NG * q);  // my pair's draw lane
                    const uint32_t pm = (G == 1) ? pvk[k] : __shfl_sync(kFull, pvk[k], src);
                    const bool okm = (vmk[k] >> src) & 1u;
                    const bool acc = decide_lane(ps[0], okm, a.tp, u, pm, st);
                    gpairs += okm ? 1u : 0u;
                    stage.push(acc, edge_key(u, pm, a.sink.nb), a.sink, lane);
                }
                continue;
            }
            // ---- wide rows: compact the live pairs of this chunk ----
            uint32_t nlive = 0;
#pragma unroll
            for (int k = 0; k < R; ++k) {
                const uint32_t i = i0 + 32 * k + lane;
                const uint32_t p = EXH ? (a.exh_low ? i : (uint32_t)u + 1 + i) : pv[k];
                const bool live = i < limit && p >= plo && p < phi;
                const unsigned m = __ballot_sync(kFull, live);
                if (live) list[nlive + __popc(m & lanemask_lt())] = p;
                nlive += __popc(m);
            }
            __syncwarp();
            // ---- eps-test the live pairs, U per step (G = 32: a warp per row) ----
            // Loads are unconditional except the last float4 column (V =
            // ceil(W/32), so columns < V-1 are always inside the row); a tail
            // step re-reads a live partner and ignores the result.  The U
            // partial sums are reduce-scattered (transposed butterfly: U-1 +
            // log2(32/U) shuffles for U pairs), leaving pair k's total in lane
            // k*32/U, which alone decides and emits it.
            if constexpr (G == 32 && !F2) {
            constexpr int SPAN = 32 / U;  // lanes per pair after the scatter
            F4x2 qw[V];
#pragma unroll
            for (int vv = 0; vv < V; ++vv) qw[vv] = to_x2(qv[vv]);
#pragma unroll 1
            for (uint32_t j0 = 0; j0 < nlive; j0 += U) {
                F4x2 rows[U][V];
#pragma unroll
                for (int uu = 0; uu < U; ++uu) {
                    const uint32_t j = j0 + uu;
                    const uint32_t pv = list[j < nlive ? j : j0];
                    const Vec* row = P + (uint64_t)pv * W + lane;
#pragma unroll
                    for (int vv = 0; vv < V; ++vv) {
                        if (vv < V - 1 || lane + 32 * vv < W) rows[uu][vv] = ldg_row2(row + 32 * vv);
                        else rows[uu][vv] = F4x2{0ull, 0ull};  // outside the row (query is 0 too)
                    }
                }
                // scheduling fence: keeps all U*V loads in flight together
                // (ptxas otherwise sinks each next to its use to save registers)
                __syncwarp();
                float ps[U];
#pragma unroll
                for (int uu = 0; uu < U; ++uu) {
                    Acc2 acc;
#pragma unroll
                    for (int vv = 0; vv < V; ++vv) diff2x2(qw[vv], rows[uu][vv], acc);
                    ps[uu] = acc2_sum(acc);
                }
#pragma unroll
                for (int o = 16, m = U; m > 1; o >>= 1, m >>= 1) {
                    const bool hi = (lane & o) != 0;
#pragma unroll
                    for (int k = 0; k < m / 2; ++k) {
                        const float mine = hi ? ps[k + m / 2] : ps[k];
                        const float other = hi ? ps[k] : ps[k + m / 2];
                        ps[k] = mine + __shfl_xor_sync(kFull, other, o);
                    }
                }
#pragma unroll
                for (int o = SPAN / 2; o > 0; o >>= 1) ps[0] += __shfl_xor_sync(kFull, ps[0], o);
                const uint32_t pj = j0 + lane / SPAN;
                const bool okm = (lane % SPAN) == 0 && pj < nlive;
                const uint32_t pm = list[okm ? pj : j0];
                const bool acc = decide_lane(ps[0], okm, a.tp, u, pm, st);
                gpairs += okm ? 1u : 0u;
                stage.push(acc, edge_key(u, pm, a.sink.nb), a.sink, lane);
            }
            }
            __syncwarp();
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
// k_prepare: copy n x d rows into the padded device layout (stride floats)
// and count non-finite values (dataset.hpp:24-26).  With dst == nullptr the
// kernel only checks.
// ---------------------------------------------------------------------------
__global__ void k_prepare(const float* __restrict__ src, float* __restrict__ dst, uint64_t n,
                          uint32_t d, uint32_t stride, unsigned long long* counters, bool minmax) {
    const uint64_t total = dst ? n * stride : n * d;
    unsigned bad = 0;
    uint32_t kmin = 0, kmax = 0;  // kmin = max of ~key (0 = nothing seen)
    auto see = [&](float v) {
        bad += !isfinite(v);
        if (minmax) {
            const uint32_t k = ordered_key(v);
            kmin = max(kmin, ~k);
            kmax = max(kmax, k);
        }
    };
    uint64_t first = 0;
    if (!dst && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
        // check-only pass over an aligned table: 16-byte loads, scalar tail
        const float4* s4 = reinterpret_cast<const float4*>(src);
        const uint64_t n4 = total / 4;
        for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
             i += (uint64_t)gridDim.x * blockDim.x) {
            const float4 v = __ldg(s4 + i);
            see(v.x);
            see(v.y);
            see(v.z);
            see(v.w);
        }
        first = n4 * 4;
    }
    for (uint64_t idx = first + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (uint64_t)gridDim.x * blockDim.x) {
        float v;
        bool real = true;
        if (dst) {
            const uint64_t r = idx / stride;
            const uint32_t c = (uint32_t)(idx - r * stride);
            v = 0.f;
            real = c < d;
            if (real) v = src[r * d + c];
            dst[idx] = v;
        } else {
            v = src[idx];
        }
        if (real) see(v);
    }
    bad = __reduce_add_sync(kFull, bad);
    if ((threadIdx.x & 31) == 0 && bad) atomicAdd(&counters[C_NONFINITE], (unsigned long long)bad);
    if (minmax) {
        kmin = __reduce_max_sync(kFull, kmin);
        kmax = __reduce_max_sync(kFull, kmax);
        if ((threadIdx.x & 31) == 0) {
            atomicMax(&counters[C_QMIN], (unsigned long long)kmin);
            atomicMax(&counters[C_QMAX], (unsigned long long)kmax);
        }
    }
}

// fp64 input: round each value to fp32 (to nearest) into the padded table,
// count non-finite values, reduce the exact fp64 min / max.
__global__ void k_prepare_f64(const double* __restrict__ src, float* __restrict__ dst, uint64_t n,
                              uint32_t d, uint32_t stride, unsigned long long* counters) {
    const uint64_t total = n * stride;
    unsigned bad = 0;
    unsigned long long kmin = 0, kmax = 0;
    for (uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r = idx / stride;
        const uint32_t c = (uint32_t)(idx - r * stride);
        float v = 0.f;
        if (c < d) {
            const double x = src[r * d + c];
            bad += !isfinite(x);
            const unsigned long long k = ordered_key64(x);
            kmin = max(kmin, ~k);
            kmax = max(kmax, k);
            v = __double2float_rn(x);
        }
        dst[idx] = v;
    }
    bad = __reduce_add_sync(kFull, bad);
    if ((threadIdx.x & 31) == 0 && bad) atomicAdd(&counters[C_NONFINITE], (unsigned long long)bad);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        kmin = max(kmin, __shfl_xor_sync(kFull, kmin, o));
        kmax = max(kmax, __shfl_xor_sync(kFull, kmax, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(&counters[C_QMIN], kmin);
        atomicMax(&counters[C_QMAX], kmax);
    }
}

// k_band: the exact decision (distance.hpp, fp64, the reference's order) of
// every pair a filter kernel left in its band; the accepted ones are emitted.
// Also the band statistics: pairs within 1e-6 of eps^2 by the filter value and
// pairs a bare fp32 test would have decided wrongly (fp32 filters only).
__global__ void k_band(const TestParams tp, const EdgeSink sink, unsigned long long* counters) {
    uint64_t count = *tp.band_cursor;
    if (count > tp.band_cap) count = tp.band_cap;
    unsigned b6 = 0, flips = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 r = tp.band[i];
        const bool acc = exact_within(tp, r.x, r.y);
        const float s = __uint_as_float(r.z);
        b6 += fabsf(s - tp.eps2f) <= 1e-6f * fabsf(tp.eps2f) ? 1u : 0u;
        flips += (s == s && (s <= tp.eps2f) != acc) ? 1u : 0u;
        if (acc) {
            const unsigned long long slot = atomicAdd(sink.cursor, 1ull);
            if (slot < sink.capacity) sink.keys[slot] = edge_key(r.x, r.y, sink.nb);
        }
    }
    b6 = __reduce_add_sync(kFull, b6);
    flips = __reduce_add_sync(kFull, flips);
    if ((threadIdx.x & 31) == 0) {
        if (b6) atomicAdd(&counters[C_BAND6], (unsigned long long)b6);
        if (flips) atomicAdd(&counters[C_FLIPS], (unsigned long long)flips);
    }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
cudaError_t launch_band(const TestParams& tp, const EdgeSink& sink, unsigned long long* counters,
                        cudaStream_t s, int num_sms) {
    k_band<<<(unsigned)(num_sms * 4), 256, 0, s>>>(tp, sink, counters);
    note_launch(1);
    return cudaGetLastError();
}
cudaError_t launch_prepare_points_f64(const double* src, float* dst, uint64_t n, uint32_t d,
                                      uint32_t stride, unsigned long long* counters,
                                      cudaStream_t s) {
    uint64_t blocks = (n * stride + 255) / 256;
    if (blocks > 148ull * 16) blocks = 148ull * 16;
    if (blocks == 0) blocks = 1;
    k_prepare_f64<<<(unsigned)blocks, 256, 0, s>>>(src, dst, n, d, stride, counters);
    note_launch(1);
    return cudaGetLastError();
}

cudaError_t launch_prepare_points(const float* src, float* dst, uint64_t n, uint32_t d,
                                  uint32_t stride, unsigned long long* counters, bool minmax,
                                  cudaStream_t s) {
    const uint64_t total = dst ? n * stride : n * d;
    uint64_t blocks = (total + 255) / 256;
    if (blocks > 148ull * 16) blocks = 148ull * 16;
    if (blocks == 0) blocks = 1;
    k_prepare<<<(unsigned)blocks, 256, 0, s>>>(src, dst, n, d, stride, counters, minmax);
    note_launch(1);
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
    const uint64_t rows = a.row_end - a.row_begin;
    // rows_per_block: a non-persistent grid, so the block scheduler can
    // interleave these blocks with a concurrently running sampler
    unsigned grid = a.rows_per_block ? (unsigned)((rows + a.rows_per_block - 1) / a.rows_per_block)
                                     : persistent_grid(k, rows, num_sms);
    k<<<grid, 256, 0, s>>>(a);
    note_launch(1);
    return cudaGetLastError();
}

template <bool EXH>
cudaError_t gather_dispatch(const GatherArgs& a, cudaStream_t s, int num_sms) {
    if (a.tp.stride == 2) return gather_one<1, 1, SNGB_F2_R, true, EXH>(a, s, num_sms);
    const uint32_t W = a.tp.stride / 4;
    // 16-byte rows: 2 chunks of 32 draws per step (R = 4 spilled at 64 registers
    // and measured 37 % slower on cfg4)
    if (W == 1) return gather_one<1, 1, 2, false, EXH>(a, s, num_sms);
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
        default: return cudaErrorInvalidValue;  // d > 1024 runs the generic kernel (sngb_metric.cu)
    }
}

template <int G, int V, bool F2>
cudaError_t extras_one(const ExtrasArgs& a, cudaStream_t s, int num_sms) {
    auto k = k_extras<G, V, F2>;
    constexpr int NG = 32 / G;
    unsigned grid = persistent_grid(k, (a.capacity + NG - 1) / NG, num_sms);
    k<<<grid, 256, 0, s>>>(a);
    note_launch(1);
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

}  // namespace sngb
