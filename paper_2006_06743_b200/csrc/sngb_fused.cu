// sngb_fused.cu -- k_sample_head: the Floyd bookkeeping (graph.cpp:161-174) and
// the head-filter gather (sngb_head.cu) of large narrow-row problems in ONE
// pass over the draws, one warp per vertex (cfg3, cfg4, cfg5).
//
// Why.  As two kernels (k_floyd_bloom + k_gather_head) every draw
//   t_i = Lemire(mix(key + (i+1) gamma), base + i + 1)   (rng.hpp:26,35-48)
// is generated twice and each kernel spends ~95 SASS instructions per draw
// (ncu, profiles/r02_ncu_floyd_cfg5.md, r01_ncu_head_cfg5.md); the gather
// also waits on one random L2 sector per pair.  Here a warp owns a vertex and
// generates each draw once; the only per-draw work besides the RNG is one
// shared-memory atomic, one coalesced store and the head test.  No block
// barriers: the warps of a block are independent.
//
// Per vertex u (warp-private shared memory, global scratch for the draws):
//   P1  draw i (lane i mod 32, slot-major): t_i; the partner's head load;
//       t_i -> scratch[i]; OR bit h(t_i) into a 2^B-bit filter F -- a draw that
//       finds its bit already set records h in the second-comer list SL;
//       t_i in [base, base + i) (may equal an earlier replacement j_k) goes
//       to the chain list CL; the head test (exact reject, sngb_head.cu) and
//       survivors' fp32 test (sngb_epstest.cuh) as in k_gather_head.
//   P2  F := the bits of SL (every bit hit by >= 2 draws); scan the stored
//       draws, the ones on such a bit -> group list GL (scratch);
//   R   GL in a small hash (F's memory) keyed by t with the minimum index:
//       a draw whose value has a smaller index collides (graph.cpp:168-169:
//       its replacement j_i = base + i is inserted instead); then the chain
//       candidates in index order against the collided set.  Every collided
//       draw's replacement is emitted as an extra pair (tested by k_extras).
// A Lemire reject pre-condition (rng.hpp:43, ~1e-12 per draw) or a list
// overflow sends the vertex to the exact sequential replay (k_replay_list,
// true Stream semantics; every partner becomes an extra); its gather stops at
// the first fired draw, as k_gather_head does.  Every decision is the
// two-kernel path's, so the results are identical (tests/test_gpu_parity.py
// -k fused).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "sngb_device.cuh"
#include "sngb_epstest.cuh"
#include "sngb_head.cuh"
#include "sngb_internal.cuh"
#include "sngb_rng.cuh"

#ifndef SNGB_FUSED_MINB
#define SNGB_FUSED_MINB 4
#endif
#ifndef SNGB_FUSED_R
#define SNGB_FUSED_R 4
#endif

namespace sngb {

namespace {

#include "sngb_floyd_bloom.cuh"

constexpr int kFWarps = 4;       // warps per block (independent vertices)
constexpr int kSLCap = 256;      // second-comer bits per vertex (D^2 / 2^(B+1): 122 at D = 4000)
constexpr int kCLCap = 64;       // chain candidates per vertex (~D^2 / 2n)
constexpr int kFStage = 64;      // edge staging per warp (accepts are rare here)
constexpr int kMaxWarpsPerSM = 32;

// per-warp geometry: filter F of 2^B bits (FW words), its reuse as the
// resolution hash (FW / 2 u64 slots), collided bitmap (CW words)
struct FGeom {
    uint32_t B, FW, CW, gl_cap, dpad;
    __host__ __device__ uint32_t q_cap(int R, int step) const { return ((32 * R + step) + 3) & ~3u; }
    __host__ __device__ uint32_t warp_bytes(int R, int step) const {
        return FW * 4 + kSLCap * 4 + kCLCap * 8 + CW * 4 + q_cap(R, step) * 4 + kFStage * 8;
    }
    __host__ __device__ uint64_t scratch_words() const { return dpad + 2ull * gl_cap; }
};

inline FGeom fgeom(uint32_t draws) {
    const BloomGeom bg = bloom_geometry(draws);
    FGeom g;
    g.B = bg.bits_log2;
    g.FW = bg.words;
    g.CW = bg.col_words;
    g.gl_cap = (g.FW / 2) * 3 / 4;
    g.dpad = (draws + 31) & ~31u;
    return g;
}

__device__ __forceinline__ void red_or_sh(uint32_t addr, uint32_t v) {
    asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

template <int KIND, int G, int V, int R>
__global__ void __launch_bounds__(kFWarps * 32, SNGB_FUSED_MINB)
    k_sample_head(const SamplerArgs a, const GatherArgs g, const HeadArgs h, const FGeom fg) {
    constexpr int NG = 32 / G;
    constexpr int UF = 2;            // fp32 rows per group per step
    constexpr int STEP = NG * UF;    // survivors per fp32 step
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int q = lane % G, grp = lane / G;
    const bool leader = (q == 0);
    const uint32_t D = a.draws, base = a.base;
    const uint32_t shift = 32 - fg.B, FW = fg.FW;
    const uint32_t hs_log = fg.B - 6;  // resolution hash: 2^B / 64 u64 slots
    const uint32_t hs_mask = (1u << hs_log) - 1;

    // warp-private shared memory
    unsigned char* wsm = smem + (size_t)wib * fg.warp_bytes(R, STEP);
    uint32_t* F = reinterpret_cast<uint32_t*>(wsm);
    unsigned long long* HT = reinterpret_cast<unsigned long long*>(wsm);  // F's memory in R
    uint32_t* SL = F + FW;
    unsigned long long* CL = reinterpret_cast<unsigned long long*>(SL + kSLCap);
    uint32_t* colbits = reinterpret_cast<uint32_t*>(CL + kCLCap);
    uint32_t* Q = colbits + fg.CW;
    unsigned long long* stg = reinterpret_cast<unsigned long long*>(Q + fg.q_cap(R, STEP));
    const uint32_t Fa = smem_addr(F);

    // warp-private global scratch: the draws, then the group list
    const uint64_t gw = (uint64_t)blockIdx.x * kFWarps + wib;
    uint32_t* scr = reinterpret_cast<uint32_t*>(a.scratch64) + gw * fg.scratch_words();
    unsigned long long* GL = reinterpret_cast<unsigned long long*>(scr + fg.dpad);
    uint32_t* irr_list = reinterpret_cast<uint32_t*>(a.scratch64) +
                         (uint64_t)gridDim.x * kFWarps * fg.scratch_words();

    const float4* __restrict__ P = reinterpret_cast<const float4*>(g.tp.pts);
    const void* __restrict__ H = h.head;
    const uint32_t W = g.tp.stride / 4;
    const float reject = h.reject;
    const uint64_t pol = evict_first_policy();  // survivor rows must not evict the heads
    const EdgeSink xs{a.extras, a.extras_capacity, &a.counters[C_EXTRA_CURSOR], 0};

    WarpStage<kFStage> stage{stg, 0};
    TestStats st;
    unsigned long long gpairs = 0, tails = 0, ncol = 0;

    for (uint32_t w = lane; w < fg.CW; w += 32) colbits[w] = 0;

    uint64_t u = 0, chunk_end = 0;
    auto grab = [&]() {
        unsigned long long b0 = 0;
        if (lane == 0) b0 = atomicAdd(g.work, (unsigned long long)g.grab);
        b0 = __shfl_sync(kFull, b0, 0);
        u = a.row_begin + b0;
        chunk_end = u + g.grab < a.row_end ? u + g.grab : a.row_end;
    };
    grab();
    for (; u < chunk_end; (u + 1 >= chunk_end) ? grab() : (void)(++u)) {
        F4x2 qv[V];
#pragma unroll
        for (int vv = 0; vv < V; ++vv) {
            const uint32_t c = q + G * vv;
            qv[vv] = to_x2(ldg_row(P + u * W + (c < W ? c : W - 1)));
        }
        const uint32_t hq = head_load<KIND>(H, (uint32_t)u);
        // test hook (test_fire) resolved once per vertex
        const uint32_t hook = (a.force_mod != 0 && (u % a.force_mod) == 0) ? D / 2 : 0xffffffffu;
        {  // F := 0 (the previous vertex left its resolution hash here)
            uint4* f4 = reinterpret_cast<uint4*>(F);
            for (uint32_t w = lane; w < FW / 4; w += 32) f4[w] = make_uint4(0, 0, 0, 0);
        }
        __syncwarp();

        // fp32 test of queue entries [e0, e0 + STEP) of which those < qend are real
        auto fp32_step = [&](uint32_t e0, uint32_t qend) {
            F4x2 rows[UF][V];
            uint32_t pe[UF];
            bool oke[UF];
#pragma unroll
            for (int uu = 0; uu < UF; ++uu) {
                const uint32_t e = e0 + grp + NG * uu;
                oke[uu] = e < qend;
                pe[uu] = Q[oke[uu] ? e : e0];
#pragma unroll
                for (int vv = 0; vv < V; ++vv) {
                    const uint32_t c = q + G * vv;
                    const uint64_t row = (oke[uu] && c < W) ? pe[uu] : u;
                    rows[uu][vv] = ldg_row2_ef(P + row * W + (c < W ? c : W - 1), pol);
                }
            }
            __syncwarp();
#pragma unroll
            for (int uu = 0; uu < UF; ++uu) {
                Acc2 acc;
#pragma unroll
                for (int vv = 0; vv < V; ++vv) diff2x2(qv[vv], rows[uu][vv], acc);
                float s = acc2_sum(acc);
#pragma unroll
                for (int o = G / 2; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
                const bool accd = decide(s, oke[uu], leader, grp * G, g.tp, u, pe[uu], st);
                tails += (oke[uu] && leader) ? 1u : 0u;
                stage.push(leader && accd, edge_key(u, pe[uu], g.sink.nb), g.sink, lane);
            }
        };

        // ---- P1: draws, head tests, filter ----
        uint32_t limit = D, qn = 0, nsl = 0, ncl = 0;
        bool irregular = false;
        uint64_t z = vertex_key(a.seed_mixed, u) + (uint64_t)(lane + 1) * kGamma;
        for (uint32_t i0 = 0; i0 < limit; i0 += 32 * R, z += (uint64_t)(32 * R) * kGamma) {
            uint32_t tv[R], pv[R];
            unsigned fires = 0;
#pragma unroll
            for (int k = 0; k < R; ++k) {
                const uint32_t i = i0 + 32 * k + lane;
                bool fire;
                const uint32_t t = lemire32(mix(z + (uint64_t)(32 * k) * kGamma), base + i + 1, fire);
                const bool valid = i < limit;
                fires |= ((fire || i == hook) && valid) ? (1u << k) : 0u;
                tv[k] = t;
                pv[k] = valid ? t + (t >= (uint32_t)u ? 1u : 0u) : (uint32_t)u;
            }
            uint32_t hb[R];
#pragma unroll
            for (int k = 0; k < R; ++k) hb[k] = head_load<KIND>(H, pv[k]);  // in flight from here
            unsigned sec = 0, chn = 0;
            uint32_t hk[R];
#pragma unroll
            for (int k = 0; k < R; ++k) {
                const uint32_t i = i0 + 32 * k + lane;
                const uint32_t t = tv[k];
                hk[k] = (t * 0x9E3779B1u) >> shift;
                if (i < limit) {
                    scr[i] = t;
                    const uint32_t bit = 1u << (hk[k] & 31);
                    sec |= (atom_or_sh(Fa + (hk[k] >> 5) * 4u, bit) & bit) ? (1u << k) : 0u;
                    chn |= (t - base < i) ? (1u << k) : 0u;  // t <= base + i always
                }
            }
            if (__any_sync(kFull, fires != 0)) {  // rare: irregular vertex, cut at the first fire
                irregular = true;
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    const unsigned fm = __ballot_sync(kFull, (fires >> k) & 1u);
                    if (fm) {
                        limit = i0 + 32 * k + __ffs(fm) - 1;
                        break;
                    }
                }
            }
            if (__any_sync(kFull, sec != 0)) {
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    const bool b = (sec >> k) & 1u;
                    const unsigned m = __ballot_sync(kFull, b);
                    const uint32_t slot = nsl + __popc(m & lanemask_lt());
                    if (b && slot < (uint32_t)kSLCap) SL[slot] = hk[k];
                    nsl += __popc(m);
                }
            }
            if (__any_sync(kFull, chn != 0)) {  // rare (about draws/n per draw)
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    const bool b = (chn >> k) & 1u;
                    const unsigned m = __ballot_sync(kFull, b);
                    const uint32_t slot = ncl + __popc(m & lanemask_lt());
                    if (b && slot < (uint32_t)kCLCap)
                        CL[slot] = ((unsigned long long)tv[k] << 32) | (i0 + 32 * k + lane);
                    ncl += __popc(m);
                }
            }
#pragma unroll
            for (int k = 0; k < R; ++k) {
                const uint32_t i = i0 + 32 * k + lane;
                const bool live = i < limit;
                gpairs += live ? 1u : 0u;
                const bool keep = live && !(head_q<KIND>(hq, hb[k]) > reject);
                const unsigned km = __ballot_sync(kFull, keep);
                if (keep) Q[qn + __popc(km & lanemask_lt())] = pv[k];
                qn += __popc(km);
            }
            __syncwarp();
            if (qn >= (uint32_t)STEP) {
                uint32_t e0 = 0;
#pragma unroll 1
                for (; e0 + STEP <= qn; e0 += STEP) fp32_step(e0, qn);
                const uint32_t rem = qn - e0;  // < STEP: move them to the front
                const uint32_t mp = (uint32_t)lane < rem ? Q[e0 + lane] : 0u;
                __syncwarp();
                if ((uint32_t)lane < rem) Q[lane] = mp;
                qn = rem;
                __syncwarp();
            }
        }
        if (qn) fp32_step(0, qn);
        __syncwarp();

        // ---- P2 + R: the Floyd collisions of this vertex ----
        bool replay = irregular || nsl > (uint32_t)kSLCap || ncl > (uint32_t)kCLCap;
        if (!replay && nsl > 0) {
            {  // F := the shared bits
                uint4* f4 = reinterpret_cast<uint4*>(F);
                for (uint32_t w = lane; w < FW / 4; w += 32) f4[w] = make_uint4(0, 0, 0, 0);
            }
            __syncwarp();
            for (uint32_t e = lane; e < nsl; e += 32) red_or_sh(Fa + (SL[e] >> 5) * 4u, 1u << (SL[e] & 31));
            __syncwarp();
            uint32_t ng = 0;
            for (uint32_t i0 = 0; i0 < D; i0 += 32) {
                const uint32_t i = i0 + lane;
                const uint32_t t = i < D ? scr[i] : 0u;
                const uint32_t hh = (t * 0x9E3779B1u) >> shift;
                const bool hit = i < D && ((ld_sh(Fa + (hh >> 5) * 4u) >> (hh & 31)) & 1u);
                const unsigned m = __ballot_sync(kFull, hit);
                const uint32_t slot = ng + __popc(m & lanemask_lt());
                if (hit && slot < fg.gl_cap) GL[slot] = ((unsigned long long)t << 32) | i;
                ng += __popc(m);
            }
            if (ng > fg.gl_cap) {
                replay = true;
            } else {
                __syncwarp();
                {  // F's memory := an empty (t + 1, min index) hash
                    uint4* f4 = reinterpret_cast<uint4*>(F);
                    for (uint32_t w = lane; w < FW / 4; w += 32) f4[w] = make_uint4(0, 0, 0, 0);
                }
                __syncwarp();
                for (uint32_t e = lane; e < ng; e += 32) {
                    const unsigned long long en = GL[e];
                    const unsigned long long kk = en + (1ull << 32);  // (t + 1) << 32 | i, never 0
                    uint32_t sl = ((uint32_t)(en >> 32) * 0x85EBCA6Bu) >> (32 - hs_log);
                    for (;;) {
                        const unsigned long long old = atomicCAS(&HT[sl], 0ull, kk);
                        if (old == 0ull) break;
                        if ((old >> 32) == (kk >> 32)) {
                            atomicMin(&HT[sl], kk);
                            break;
                        }
                        sl = (sl + 1) & hs_mask;
                    }
                }
                __syncwarp();
                for (uint32_t e = lane; e < ng; e += 32) {
                    const unsigned long long en = GL[e];
                    const uint32_t t1 = (uint32_t)(en >> 32) + 1u, i = (uint32_t)en;
                    uint32_t sl = ((uint32_t)(en >> 32) * 0x85EBCA6Bu) >> (32 - hs_log);
                    while ((uint32_t)(HT[sl] >> 32) != t1) sl = (sl + 1) & hs_mask;
                    if ((uint32_t)HT[sl] != i) {  // an earlier draw has the same value
                        atomicOr(&colbits[i >> 5], 1u << (i & 31));
                        const unsigned long long s2 = atomicAdd(xs.cursor, 1ull);
                        const uint32_t e2 = base + i;
                        if (s2 < xs.capacity)
                            xs.keys[s2] = (u << 32) | (e2 + (e2 >= (uint32_t)u ? 1u : 0u));
                        ++ncol;
                    }
                }
                __syncwarp();
                if (lane == 0 && ncl) {
                    for (uint32_t x = 1; x < ncl; ++x) {  // insertion sort by index (tiny list)
                        const unsigned long long v = CL[x];
                        uint32_t y = x;
                        while (y > 0 && (uint32_t)CL[y - 1] > (uint32_t)v) {
                            CL[y] = CL[y - 1];
                            --y;
                        }
                        CL[y] = v;
                    }
                    for (uint32_t x = 0; x < ncl; ++x) {
                        const uint32_t i = (uint32_t)CL[x];
                        if ((colbits[i >> 5] >> (i & 31)) & 1u) continue;  // already collided
                        const uint32_t kx = (uint32_t)(CL[x] >> 32) - base;
                        if ((colbits[kx >> 5] >> (kx & 31)) & 1u) {  // t_i = j_k, k collided
                            colbits[i >> 5] |= 1u << (i & 31);
                            const unsigned long long s2 = atomicAdd(xs.cursor, 1ull);
                            const uint32_t e2 = base + i;
                            if (s2 < xs.capacity)
                                xs.keys[s2] = (u << 32) | (e2 + (e2 >= (uint32_t)u ? 1u : 0u));
                            ++ncol;
                        }
                    }
                }
                __syncwarp();
                for (uint32_t e = lane; e < ng; e += 32) colbits[(uint32_t)GL[e] >> 5] = 0;
                for (uint32_t e = lane; e < ncl; e += 32) colbits[(uint32_t)CL[e] >> 5] = 0;
                __syncwarp();
            }
        }  // nsl == 0: all values distinct, no replacement exists, no chain can collide
        if (replay && lane == 0) {
            const unsigned long long s2 = atomicAdd(&a.counters[C_IRR_CURSOR], 1ull);
            irr_list[s2] = (uint32_t)u;  // capacity: one slot per row
        }
        __syncwarp();
    }
    stage.flush(g.sink, lane);
    st.pairs = gpairs;
    flush_stats(st, gpairs, g.counters, lane);
    const unsigned long long tw = warp_sum(tails);
    if (lane == 0 && tw) atomicAdd(&g.counters[C_TAIL_PAIRS], tw);
    ncol = warp_sum(ncol);
    if (lane == 0 && ncol) atomicAdd(&a.counters[C_COLLISIONS], ncol);
}

// The exact sequential replay (bloom_replay: graph.cpp:163-174 with true Stream
// semantics) of the vertices k_sample_head listed; every partner is an extra.
__global__ void __launch_bounds__(32) k_replay_list(const SamplerArgs a, const uint32_t* list,
                                                    uint32_t cap) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t* tab = reinterpret_cast<uint32_t*>(smem);
    const EdgeSink xs{a.extras, a.extras_capacity, &a.counters[C_EXTRA_CURSOR], 0};
    const unsigned long long cnt = a.counters[C_IRR_CURSOR];
    unsigned long long nrep = 0;
    for (unsigned long long x = blockIdx.x; x < cnt; x += gridDim.x) {
        if (threadIdx.x == 0) {
            const uint64_t u = list[x];
            bloom_replay(vertex_key(a.seed_mixed, u), u, a.n, a.base, tab, cap, xs);
            ++nrep;
        }
    }
    if (threadIdx.x == 0 && nrep) atomicAdd(&a.counters[C_IRREGULAR], nrep);
}

template <int KIND, int G, int V>
cudaError_t fused_one(SamplerArgs a, GatherArgs ga, const HeadArgs& h, cudaStream_t s,
                      int num_sms) {
    constexpr int R = SNGB_FUSED_R;
    constexpr int STEP = (32 / G) * 2;
    auto k = k_sample_head<KIND, G, V, R>;
    const FGeom fg = fgeom(a.draws);
    const size_t smem = (size_t)kFWarps * fg.warp_bytes(R, STEP);
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kFWarps * 32, smem);
    if (per_sm < 1) per_sm = 1;
    if (per_sm > kMaxWarpsPerSM / kFWarps) per_sm = kMaxWarpsPerSM / kFWarps;
    const uint64_t rows = a.row_end - a.row_begin;
    const uint64_t want = (rows + kFWarps - 1) / kFWarps;
    const uint64_t cap = (uint64_t)num_sms * per_sm;
    const unsigned grid = (unsigned)(want < cap ? want : cap);
    const uint64_t warps = (uint64_t)grid * kFWarps;
    ga.grab = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(32, rows / (warps * 16)));
    k<<<grid, kFWarps * 32, smem, s>>>(a, ga, h, fg);
    note_launch(1);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    // the listed vertices' exact replays (usually none: one small launch)
    uint32_t cap_slots = 1;
    while (cap_slots < 2 * a.draws + 2) cap_slots <<= 1;
    const size_t rsmem = (size_t)cap_slots * 4;
    e = cudaFuncSetAttribute(k_replay_list, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsmem);
    if (e != cudaSuccess) return e;
    const uint32_t* list = reinterpret_cast<const uint32_t*>(a.scratch64) + warps * fg.scratch_words();
    k_replay_list<<<num_sms * 8, 32, rsmem, s>>>(a, list, cap_slots);
    note_launch(1);
    return cudaGetLastError();
}

template <int KIND>
cudaError_t fused_kind(const SamplerArgs& sa, const GatherArgs& ga, const HeadArgs& h,
                       cudaStream_t s, int num_sms) {
    const uint32_t W = ga.tp.stride / 4;
    if (W <= 2) return fused_one<KIND, 2, 1>(sa, ga, h, s, num_sms);
    if (W <= 4) return fused_one<KIND, 4, 1>(sa, ga, h, s, num_sms);
    if (W <= 8) return fused_one<KIND, 8, 1>(sa, ga, h, s, num_sms);
    if (W <= 16) return fused_one<KIND, 16, 1>(sa, ga, h, s, num_sms);
    if (W <= 32) return fused_one<KIND, 32, 1>(sa, ga, h, s, num_sms);
    return cudaErrorInvalidValue;
}

}  // namespace

#ifndef SNGB_FUSED_DEFAULT
#define SNGB_FUSED_DEFAULT 0
#endif
constexpr int kFusedDefault = SNGB_FUSED_DEFAULT;

bool fused_eligible(uint64_t n, uint32_t draws, uint32_t stride) {
    // SNGB_FUSED=0 keeps the two kernels, 1 fuses every eligible shape, 2 (auto)
    // also needs few chain candidates per vertex (about draws^2 / 2n <= 4: they
    // are resolved sequentially by one lane).  Eligible wherever launch_sampler
    // would pick k_floyd_bloom (n beyond the per-warp bitmap kernel's 73 k, or
    // SNGB_FLOYD_NO_BITMAP; draws <= 4096) for rows of <= 32 float4.
    const char* e = std::getenv("SNGB_FUSED");
    const int mode = e ? std::atoi(e) : kFusedDefault;
    if (mode == 0 || draws < 1 || draws > 4096 || n - 2 >= 0xffffffffull || stride / 4 > 32)
        return false;
    if (mode == 2 && (uint64_t)draws * draws > 8 * n) return false;
    const uint64_t bm_words = (((n - 1) + 31) / 32 + 3) & ~3ull;
    return bm_words * 4 > 9216 || std::getenv("SNGB_FLOYD_NO_BITMAP") != nullptr;
}

size_t fused_scratch_bytes(uint32_t draws, uint64_t rows, int num_sms) {
    const FGeom fg = fgeom(draws);
    return ((uint64_t)num_sms * kMaxWarpsPerSM * fg.scratch_words() + rows) * 4;
}

cudaError_t launch_floyd_head(const SamplerArgs& in, const GatherArgs& ga, const HeadArgs& h,
                              cudaStream_t s, int num_sms) {
    const uint64_t rows = in.row_end - in.row_begin;
    if (rows == 0 || in.draws == 0) return cudaSuccess;
    if (!ga.work || !in.scratch64) return cudaErrorInvalidValue;  // zeroed counter, scratch
    switch (h.kind) {
        case kHeadU16x2: return fused_kind<kHeadU16x2>(in, ga, h, s, num_sms);
        case kHeadU8x4: return fused_kind<kHeadU8x4>(in, ga, h, s, num_sms);
        default: return fused_kind<kHeadU8x2>(in, ga, h, s, num_sms);
    }
}

}  // namespace sngb
