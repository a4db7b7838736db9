// sngb_fused.cu -- k_sample_head: the Floyd bookkeeping (graph.cpp:161-174) and
// the head-filter gather (sngb_head.cu) of large narrow-row problems in one
// kernel, one warp per vertex (cfg3, cfg4, cfg5).
//
// Why.  As two kernels (k_floyd_bloom + k_gather_head) each draw
//   t_i = Lemire(mix(key + (i+1) gamma), base + i + 1)   (rng.hpp:26,35-48)
// costs ~100 SASS instructions in each (ncu: profiles/r02_ncu_floyd_cfg5.md,
// r01_ncu_head_cfg5.md), and the Floyd kernel's block barriers and the
// gather's L2 latency each leave the SM a third idle.  A one-pass fusion with
// the draws kept in global scratch (v4, profiles/r02_ncu_fused_v4_cfg5.md) was
// slower: 5.5 warp-instructions per draw and 318 GB of scratch write-back.
// Here every warp owns a vertex and makes TWO lean passes over its draws,
// regenerating them (a draw is ~26 integer instructions; storing it costs
// more in L2/DRAM traffic than it saves):
//
//   P1  filter pass (no memory traffic): t_i, OR bit h(t_i) into a warp-
//       private 2^B-bit filter F; a draw that finds its bit already set
//       records h in its lane's second-comer list SL; the running minimum of
//       Lemire's low word flags a possible reject pre-condition (rng.hpp:43).
//   ->  F := the bits in SL (exactly the bits hit by >= 2 draws).
//   P2  gather pass: t_i again, the partner's head load (exact reject,
//       sngb_head.cu), survivors queued for the fp32 test (sngb_epstest.cuh);
//       draws on a shared bit -> the lane's group list GL (their indices, in
//       SL's slots), t_i in [base, base + i) -> the lane's chain list CL.
//   R   GL's values (regenerated) in a small hash (F's memory) keyed by t with
//       the minimum index: a
//       draw whose value has a smaller index collides (graph.cpp:168-169, its
//       replacement j_i = base + i is inserted instead); then the chain
//       candidates in index order against the collided set.  Every collided
//       draw's replacement is emitted as an extra pair (tested by k_extras).
// A Lemire reject pre-condition (~1e-12 per draw) or a list overflow sends
// the vertex to the exact sequential replay (k_replay_list: true Stream
// semantics, every partner an extra); its gather stops at the first fired
// draw, as k_gather_head's does.  Results are the two-kernel path's bit for
// bit (tests/test_gpu_parity.py -k "fused or head").
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
constexpr int kSLL = 32;         // per lane: second-comer bits (P1; mean D^2/2^(B+1)/32 = 3.8 at D = 4000),
                                 // then group-list draws (P2; mean D^2/2^B/32 = 7.6)
constexpr int kCLL = 4;          // chain candidates per lane (mean D^2 / 2n / 32: 0.01 on cfg5)
constexpr int kFStage = 64;      // edge staging per warp (accepts are rare here)
constexpr int kMaxWarpsPerSM = 32;

// per-warp geometry: filter F of 2^B bits (FW words, reused as the resolution
// hash of FW / 2 u64 slots), collided bitmap (CW words)
struct FGeom {
    uint32_t B, FW, CW;
    __host__ __device__ uint32_t q_cap(int R, int step) const { return ((32 * R + step) + 3) & ~3u; }
    __host__ __device__ uint32_t warp_bytes(int R, int step) const {
        return FW * 4 + 32 * kSLL * 2 + 32 * kCLL * 8 + CW * 4 + q_cap(R, step) * 4 + kFStage * 8;
    }
};

inline FGeom fgeom(uint32_t draws) {
    const BloomGeom bg = bloom_geometry(draws);
    FGeom g;
    g.B = bg.bits_log2;
    g.FW = bg.words;
    g.CW = bg.col_words;
    return g;
}

#ifndef SNGB_FUSED_PF
#define SNGB_FUSED_PF 0  // measured slower on cfg5 (861 vs 845 ms)
#endif
constexpr bool kPrefetch = SNGB_FUSED_PF != 0;
__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

__device__ __forceinline__ void red_or_sh(uint32_t addr, uint32_t v) {
    asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// first draw index < D whose Lemire step meets the reject pre-condition
// (lo < bound, rng.hpp:43), or D: the exact test behind the slo == 0 flag
__device__ __noinline__ uint32_t first_fire(uint64_t key, uint32_t D, uint32_t base, int lane) {
    uint32_t f = D;
    for (uint32_t i = lane; i < D; i += 32) {
        bool fire;
        (void)lemire32(stream_at(key, (uint64_t)i + 1), base + i + 1, fire);
        if (fire) {
            f = i;
            break;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) f = min(f, __shfl_xor_sync(kFull, f, o));
    return f;
}

template <int KIND, int G, int V, int R>
__global__ void __launch_bounds__(kFWarps * 32, SNGB_FUSED_MINB)
    k_sample_head(const SamplerArgs a, const GatherArgs g, const HeadArgs h, const FGeom fg) {
    constexpr int NG = 32 / G;
    constexpr int UF = 2;            // fp32 rows per group per step
    constexpr int STEP = NG * UF;    // survivors per fp32 step
    constexpr uint32_t ITER = 32 * R;
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
    uint16_t* SL = reinterpret_cast<uint16_t*>(F + FW);       // [32][kSLL], lane-major (B <= 16)
    unsigned long long* CL = reinterpret_cast<unsigned long long*>(SL + 32 * kSLL);  // [32][kCLL]
    uint32_t* colbits = reinterpret_cast<uint32_t*>(CL + 32 * kCLL);
    uint32_t* Q = colbits + fg.CW;
    unsigned long long* stg = reinterpret_cast<unsigned long long*>(Q + fg.q_cap(R, STEP));
    const uint32_t Fa = smem_addr(F);
    uint16_t* mySL = SL + lane * kSLL;
    unsigned long long* myCL = CL + lane * kCLL;

    // the lane's group list (draw indices) reuses its SL slots: SL is consumed
    // (F rebuilt) before P2 pushes the first group entry
    uint16_t* myGL = mySL;
    uint32_t* irr_list = reinterpret_cast<uint32_t*>(a.scratch64);  // the replay list

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
    for (int j = 0; j < kCLL; ++j) myCL[j] = 0ull;  // chain lists start empty (0 = no entry)

    uint64_t u = 0, chunk_end = 0;
    auto grab = [&]() {
        unsigned long long b0 = 0;
        if (lane == 0) b0 = atomicAdd(g.work, (unsigned long long)g.grab);
        b0 = __shfl_sync(kFull, b0, 0);
        u = a.row_begin + b0;
        chunk_end = u + g.grab < a.row_end ? u + g.grab : a.row_end;
    };
    auto zeroF = [&]() {
        uint4* f4 = reinterpret_cast<uint4*>(F);
        for (uint32_t w = lane; w < FW / 4; w += 32) f4[w] = make_uint4(0, 0, 0, 0);
    };
    auto emit_extra = [&](uint32_t i) {  // collided draw i: its replacement j_i = base + i
        const unsigned long long s2 = atomicAdd(xs.cursor, 1ull);
        const uint32_t e2 = base + i;
        if (s2 < xs.capacity) xs.keys[s2] = (u << 32) | (e2 + (e2 >= (uint32_t)u ? 1u : 0u));
        ++ncol;
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
        const uint64_t key = vertex_key(a.seed_mixed, u);
        const uint64_t z0 = key + (uint64_t)(lane + 1) * kGamma;
        zeroF();
        __syncwarp();

        // ---- P1: the filter pass ----
        uint32_t nsl = 0, mn = 0xffffffffu;
        auto p1 = [&](uint32_t i0, uint64_t z, bool tail) {
            uint32_t hk[R], old[R];
#pragma unroll
            for (int k = 0; k < R; ++k) {
                const uint32_t i = i0 + 32 * k + lane;
                uint32_t slo;
                const uint32_t t = lemire32_slo(mix(z + (uint64_t)(32 * k) * kGamma), base + i + 1, slo);
                hk[k] = (t * 0x9E3779B1u) >> shift;
                if (!tail || i < D) mn = min(mn, slo);
            }
            // all R atomics in flight before any result is used
#pragma unroll
            for (int k = 0; k < R; ++k) {
                const uint32_t i = i0 + 32 * k + lane;
                old[k] = (!tail || i < D) ? atom_or_sh(Fa + (hk[k] >> 5) * 4u, 1u << (hk[k] & 31)) : 0u;
            }
#pragma unroll
            for (int k = 0; k < R; ++k) {
                if ((old[k] >> (hk[k] & 31)) & 1u) {  // a second comer
                    if (nsl < (uint32_t)kSLL) mySL[nsl] = (uint16_t)hk[k];
                    ++nsl;
                }
            }
        };
        {
            const uint32_t nfull = D / ITER;
            uint64_t z = z0;
            for (uint32_t it = 0; it < nfull; ++it, z += (uint64_t)ITER * kGamma) p1(it * ITER, z, false);
            if (nfull * ITER < D) p1(nfull * ITER, z, true);
        }
        // a possible reject pre-condition (or the test hook): the exact first fire
        uint32_t limit = D;
        const bool hooked = a.force_mod != 0 && (u % a.force_mod) == 0;
        if (__any_sync(kFull, mn == 0u) || hooked) {
            limit = first_fire(key, D, base, lane);
            if (hooked) limit = min(limit, D / 2);
        }
        const bool irregular = limit < D;
        bool replay = irregular || __any_sync(kFull, nsl > (uint32_t)kSLL);
        // F := the shared bits
        __syncwarp();
        zeroF();
        __syncwarp();
        {
            const uint32_t ns = min(nsl, (uint32_t)kSLL);
            for (uint32_t j = 0; j < ns; ++j) red_or_sh(Fa + (mySL[j] >> 5) * 4u, 1u << (mySL[j] & 31));
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

        // ---- P2: the gather pass (draws below limit) ----
        uint32_t qn = 0, ngl = 0, ncl = 0;
        auto p2 = [&](uint32_t i0, uint64_t z, bool tail) {
            uint32_t tv[R], pv[R];
#pragma unroll
            for (int k = 0; k < R; ++k) {
                const uint32_t i = i0 + 32 * k + lane;
                uint32_t slo;
                tv[k] = lemire32_slo(mix(z + (uint64_t)(32 * k) * kGamma), base + i + 1, slo);
                const uint32_t p = tv[k] + (tv[k] >= (uint32_t)u ? 1u : 0u);
                pv[k] = (!tail || i < limit) ? p : (uint32_t)u;
            }
            uint32_t hb[R];
#pragma unroll
            for (int k = 0; k < R; ++k) hb[k] = head_load<KIND>(H, pv[k]);  // in flight from here
            uint32_t fw[R];
#pragma unroll
            for (int k = 0; k < R; ++k) fw[k] = ld_sh(Fa + ((tv[k] * 0x9E3779B1u) >> shift >> 5) * 4u);
#pragma unroll
            for (int k = 0; k < R; ++k) {
                const uint32_t i = i0 + 32 * k + lane;
                const uint32_t t = tv[k];
                const bool ok = !tail || i < limit;
                if (ok && ((fw[k] >> (((t * 0x9E3779B1u) >> shift) & 31)) & 1u)) {  // on a shared bit
                    if (ngl < (uint32_t)kSLL) myGL[ngl] = (uint16_t)i;
                    ++ngl;
                }
                if (ok && t - base < i) {  // may equal an earlier replacement (t <= base + i)
                    if (ncl < (uint32_t)kCLL) myCL[ncl] = ((unsigned long long)t << 32) | i;
                    ++ncl;
                }
            }
#pragma unroll
            for (int k = 0; k < R; ++k) {
                const uint32_t i = i0 + 32 * k + lane;
                const bool keep = (!tail || i < limit) && !(head_q<KIND>(hq, hb[k]) > reject);
                const unsigned km = __ballot_sync(kFull, keep);
                if (keep) {
                    Q[qn + __popc(km & lanemask_lt())] = pv[k];
                    // wide rows come from HBM: start the fetch into L2 now, the
                    // fp32 test reads it a queue-fill later (SNGB_FUSED_PF)
                    if (kPrefetch && G >= 8) prefetch_l2(P + (uint64_t)pv[k] * W);
                }
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
        };
        {
            const uint32_t nfull = limit / ITER;
            uint64_t z = z0;
            for (uint32_t it = 0; it < nfull; ++it, z += (uint64_t)ITER * kGamma) p2(it * ITER, z, false);
            if (nfull * ITER < limit) p2(nfull * ITER, z, true);
        }
        if (qn) fp32_step(0, qn);
        if (lane == 0) gpairs += limit;
        __syncwarp();

        // ---- R: the collided draws of this vertex ----
        replay = replay || __any_sync(kFull, ngl > (uint32_t)kSLL || ncl > (uint32_t)kCLL) ||
                 (__any_sync(kFull, ncl != 0) && warp_sum(ncl) > FW / 2);  // chain sort room
        if (!replay && __any_sync(kFull, ngl != 0)) {
            zeroF();  // F's memory := an empty (t + 1, min index) hash
            __syncwarp();
            // the group draws' values are regenerated (cheaper than keeping them)
            auto draw_t = [&](uint32_t i) {
                bool f;
                return lemire32(stream_at(key, (uint64_t)i + 1), base + i + 1, f);
            };
            for (uint32_t e = 0; e < ngl; ++e) {
                const uint32_t i = myGL[e], t = draw_t(i);
                const unsigned long long kk = ((unsigned long long)(t + 1u) << 32) | i;  // never 0
                uint32_t sl = (t * 0x85EBCA6Bu) >> (32 - hs_log);
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
            for (uint32_t e = 0; e < ngl; ++e) {
                const uint32_t i = myGL[e], t = draw_t(i);
                uint32_t sl = (t * 0x85EBCA6Bu) >> (32 - hs_log);
                while ((uint32_t)(HT[sl] >> 32) != t + 1u) sl = (sl + 1) & hs_mask;
                if ((uint32_t)HT[sl] != i) {  // an earlier draw has the same value
                    atomicOr(&colbits[i >> 5], 1u << (i & 31));
                    emit_extra(i);
                }
            }
            __syncwarp();
        }
        if (!replay && __any_sync(kFull, ncl != 0)) {
            // chain candidates of all lanes in index order (tiny), against the
            // collided set; a collision makes its replacement visible to later ones
            const unsigned cm = __ballot_sync(kFull, ncl != 0);
            if (lane == 0) {
                unsigned long long* cl = HT;  // F's memory is free now
                uint32_t nc = 0;
                for (unsigned m = cm; m; m &= m - 1) {
                    const int l = __ffs(m) - 1;
                    for (int j = 0; j < kCLL; ++j) {
                        const unsigned long long v = CL[l * kCLL + j];
                        if (v == 0ull) break;  // empty slot (a chain entry has i > 0)
                        uint32_t y = nc++;
                        while (y > 0 && (uint32_t)cl[y - 1] > (uint32_t)v) {
                            cl[y] = cl[y - 1];
                            --y;
                        }
                        cl[y] = v;
                    }
                }
                for (uint32_t x = 0; x < nc; ++x) {
                    const uint32_t i = (uint32_t)cl[x];
                    if ((colbits[i >> 5] >> (i & 31)) & 1u) continue;  // already collided
                    const uint32_t kx = (uint32_t)(cl[x] >> 32) - base;
                    if ((colbits[kx >> 5] >> (kx & 31)) & 1u) {  // t_i = j_k, draw k collided
                        colbits[i >> 5] |= 1u << (i & 31);
                        emit_extra(i);
                    }
                }
            }
            __syncwarp();
        }
        if (!replay) {  // clear the touched collided-bitmap words
            for (uint32_t e = 0; e < ngl; ++e) colbits[(uint32_t)myGL[e] >> 5] = 0;
            for (uint32_t e = 0; e < ncl; ++e) colbits[(uint32_t)myCL[e] >> 5] = 0;
        }
        for (int j = 0; j < kCLL; ++j) myCL[j] = 0ull;  // chain lists start empty
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
    const uint32_t* list = reinterpret_cast<const uint32_t*>(a.scratch64);
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
    (void)draws;
    (void)num_sms;
    return rows * 4;  // the replay list: at most one entry per row
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
