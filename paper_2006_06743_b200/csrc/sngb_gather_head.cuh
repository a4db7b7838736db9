// sngb_gather_head.cuh -- the body of k_gather_head (sngb_head.cu), shared with
// the co-scheduled Floyd + gather kernel (sngb_fused.cu, k_duo): a device
// function over caller-provided shared memory (per warp: kStage edge keys and
// gather_head_qcap<G, R>() queued survivors).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "sngb_device.cuh"
#include "sngb_epstest.cuh"
#include "sngb_head.cuh"
#include "sngb_internal.cuh"
#include "sngb_rng.cuh"

#ifndef SNGB_SHARE_DRAWS
#define SNGB_SHARE_DRAWS 0  // see sngb_internal.cuh: the shared-draws experiment (build flag)
#endif
#ifndef SNGB_HEAD_UF
#define SNGB_HEAD_UF 2
#endif
#ifndef SNGB_HEAD_R
#define SNGB_HEAD_R 4
#endif

namespace sngb {

// survivor queue per warp: < STEP left over + one step's worth of draws
template <int G, int R>
__host__ __device__ constexpr int gather_head_qcap() {
    return 32 * R + (32 / G) * SNGB_HEAD_UF;
}

// k_gather_head: one warp per query row (dynamic row claiming, as k_gather).
// Each lane owns one draw per 32-draw chunk (R chunks per step): regenerate t_i
// (counter i+1), read the partner's 4-byte head (L2), reject exactly on the
// head; survivors are queued per warp and, UF per G-lane group at a time, take
// the fp32 test on their full rows (G lanes x V float4 per row, as the narrow
// k_gather path: masked pairs and columns past the row end read the query row).
template <int KIND, int G, int V, int R>
__device__ __forceinline__ void gather_head_body(const GatherArgs& a, const HeadArgs& h,
                                                 unsigned long long* stage_mem,
                                                 uint32_t* queue_mem) {
    constexpr int NG = 32 / G;
    constexpr int UF = SNGB_HEAD_UF;    // fp32 rows per group per step
    constexpr int STEP = NG * UF;       // survivors per fp32 step
    constexpr int QCAP = gather_head_qcap<G, R>();

    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int q = lane % G, g = lane / G;
    const bool leader = (q == 0);
    const uint64_t gw = (uint64_t)blockIdx.x * kWarpsPerBlock + wib;
    const uint64_t nw = (uint64_t)gridDim.x * kWarpsPerBlock;
    const float4* __restrict__ P = reinterpret_cast<const float4*>(a.tp.pts);
    const void* __restrict__ H = h.head;
    const uint32_t W = a.tp.stride / 4;
    const uint32_t plo = a.part_lo, phi = a.part_hi;
    const float reject = h.reject;
    uint32_t* queue = queue_mem + wib * QCAP;
    const uint64_t pol = evict_first_policy();  // survivor rows must not evict the heads

    WarpStage<kStage> stage{stage_mem + wib * kStage, 0};
    TestStats st;
    unsigned long long gpairs = 0, tails = 0;

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
        F4x2 qv[V];
#pragma unroll
        for (int vv = 0; vv < V; ++vv) {
            const uint32_t c = q + G * vv;
            qv[vv] = to_x2(ldg_row(P + u * W + (c < W ? c : W - 1)));
        }
        const uint32_t hq = head_load<KIND>(H, (uint32_t)u);
        // test hook (test_fire) resolved once per vertex: the draw index it fires at
        const uint32_t hook = (a.force_mod != 0 && (u % a.force_mod) == 0) ? a.draws / 2 : 0xffffffffu;
        uint32_t qn = 0;  // queued survivors (warp-uniform)

        // fp32 test of queue entries [e0, e0 + STEP) of which those < qend are real
        auto fp32_step = [&](uint32_t e0, uint32_t qend) {
            F4x2 rows[UF][V];
            uint32_t pe[UF];
            bool oke[UF];
#pragma unroll
            for (int uu = 0; uu < UF; ++uu) {
                const uint32_t e = e0 + g + NG * uu;
                oke[uu] = e < qend;
                pe[uu] = queue[oke[uu] ? e : e0];
#pragma unroll
                for (int vv = 0; vv < V; ++vv) {
                    const uint32_t c = q + G * vv;
                    const uint64_t row = (oke[uu] && c < W) ? pe[uu] : u;
                    rows[uu][vv] = ldg_row2_ef(P + row * W + (c < W ? c : W - 1), pol);
                }
            }
            __syncwarp();  // scheduling fence: all UF*V loads in flight together
#pragma unroll
            for (int uu = 0; uu < UF; ++uu) {
                Acc2 acc;
#pragma unroll
                for (int vv = 0; vv < V; ++vv) diff2x2(qv[vv], rows[uu][vv], acc);
                float s = acc2_sum(acc);
#pragma unroll
                for (int o = G / 2; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
                const bool accd = decide(s, oke[uu], leader, g * G, a.tp, u, pe[uu], st);
                tails += (oke[uu] && leader) ? 1u : 0u;
                stage.push(leader && accd, edge_key(u, pe[uu], a.sink.nb), a.sink, lane);
            }
        };

        uint32_t limit = a.draws;
#if SNGB_SHARE_DRAWS
        // shared draws: this row's slice of the draw buffer (streaming stores)
        uint32_t* tb = a.tbuf ? a.tbuf + (u - a.tbuf_row0) * a.draws : nullptr;
#endif
        uint64_t z = vertex_key(a.seed_mixed, u) + (uint64_t)(lane + 1) * kGamma;
        for (uint32_t i0 = 0; i0 < limit; i0 += 32 * R, z += (uint64_t)(32 * R) * kGamma) {
            // draws of this step, branch-free (the test hook resolved per vertex;
            // lanes past the limit compute a throw-away draw and read row u)
            uint32_t pv[R];
            unsigned fires = 0;
#pragma unroll
            for (int k = 0; k < R; ++k) {
                const uint32_t i = i0 + 32 * k + lane;
                bool fire;
                const uint32_t t = lemire32(mix(z + (uint64_t)(32 * k) * kGamma), a.base + i + 1, fire);
                const bool valid = i < limit;
#if SNGB_SHARE_DRAWS
                if (tb && i < a.draws) __stcs(tb + i, t);
#endif
                fires |= ((fire || i == hook) && valid) ? (1u << k) : 0u;
                const uint32_t p = t + (t >= (uint32_t)u ? 1u : 0u);
                pv[k] = valid ? p : (uint32_t)u;
            }
            if (__any_sync(kFull, fires != 0)) {  // rare: irregular vertex, cut at the first fire
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    const unsigned fm = __ballot_sync(kFull, (fires >> k) & 1u);
                    if (fm) {
                        limit = i0 + 32 * k + __ffs(fm) - 1;
                        break;
                    }
                }
            }
            uint32_t hb[R];
#pragma unroll
            for (int k = 0; k < R; ++k) hb[k] = head_load<KIND>(H, pv[k]);  // pv < n always
#pragma unroll
            for (int k = 0; k < R; ++k) {
                const uint32_t i = i0 + 32 * k + lane;
                const bool live = i < limit && pv[k] >= plo && pv[k] < phi;
                gpairs += live ? 1u : 0u;
                const bool keep = live && !(head_q<KIND>(hq, hb[k]) > reject);
                const unsigned km = __ballot_sync(kFull, keep);
                if (keep) queue[qn + __popc(km & lanemask_lt())] = pv[k];
                qn += __popc(km);
            }
            __syncwarp();
            if (qn >= (uint32_t)STEP) {
                uint32_t e0 = 0;
#pragma unroll 1
                for (; e0 + STEP <= qn; e0 += STEP) fp32_step(e0, qn);
                const uint32_t rem = qn - e0;  // < STEP: move them to the front
                const uint32_t mp = (uint32_t)lane < rem ? queue[e0 + lane] : 0u;
                __syncwarp();
                if ((uint32_t)lane < rem) queue[lane] = mp;
                qn = rem;
                __syncwarp();
            }
        }
        if (qn) fp32_step(0, qn);
#if SNGB_SHARE_DRAWS
        if (a.tflags && lane == 0) a.tflags[u - a.tbuf_row0] = limit < a.draws ? 1 : 0;
#endif
        __syncwarp();
    }
    stage.flush(a.sink, lane);
    st.pairs = gpairs;
    flush_stats(st, gpairs, a.counters, lane);
    const unsigned long long tw = warp_sum(tails);
    if (lane == 0 && tw) atomicAdd(&a.counters[C_TAIL_PAIRS], tw);
}


}  // namespace sngb
