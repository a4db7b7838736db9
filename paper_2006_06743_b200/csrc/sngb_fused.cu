// sngb_fused.cu -- k_floyd_head: the Floyd bookkeeping (k_floyd_bloom) and the
// head-filter gather (k_gather_head) of large narrow-row problems in ONE pass
// over the draws (cfg3, cfg4, cfg5).
//
// Why.  Run as two kernels, every draw t_i = Lemire(mix(key + (i+1) gamma))
// (rng.hpp:26,35-48; graph.cpp:161-174) is generated twice -- once for the
// collision filter, once for the partner gather -- and the two halves of the
// step sit on different limits: the filter kernel is issue-bound (shared-memory
// atomics, ~100 instructions per draw) while the gather waits on one random L2
// sector per pair.  Here each draw is generated once, ORed into the collision
// filter, and its partner's head load is issued in the same slot; the head
// tests run while the block's resolver warp settles the previous vertex, so
// the SM's issue slots and its L1/L2 request pipe work at the same time.
//
// Per vertex u (one block, 8 worker warps + 1 resolver warp, draws in
// registers; the structure of k_floyd_bloom, sngb_floyd_bloom.cuh):
//   P1  draw i: t_i, filter bit (atomicOr; a second hit marks the shared-bit
//       filter), chain candidate t_i in [base, base + i), partner
//       p = t_i + (t_i >= u), head load of p (in flight from here on);
//   B   vertex-wide OR of the Lemire pre-condition: an irregular vertex is
//       replayed exactly and sequentially (all partners become extras) and
//       its head tests are skipped;
//   P2  draws whose bit is shared go to the group list (the draw values wait
//       in shared memory, slot-major: conflict-free);
//   ->  resolver warp (one vertex behind): exact first occurrences, chain
//       candidates in index order, collided draws' replacements -> extras;
//   H   the head test of every draw (exact reject, sngb_head.cu); survivors
//       queue per warp and take the fp32 test on their rows,
//       G lanes per row (sngb_epstest.cuh: guard band, exact fp64 band list).
// Vertices are claimed dynamically (one atomic per vertex, handed to the
// resolver through a 3-slot ring).  Every decision, list and counter is the
// two-kernel path's, so results are identical (tests/test_gpu_parity.py -k fused).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "sngb_device.cuh"
#include "sngb_epstest.cuh"
#include "sngb_head.cuh"
#include "sngb_internal.cuh"
#include "sngb_rng.cuh"

#ifndef SNGB_FUSED_MINB
#define SNGB_FUSED_MINB 3
#endif
#ifndef SNGB_FUSED_UF
#define SNGB_FUSED_UF 2
#endif

namespace sngb {

namespace {

#include "sngb_floyd_bloom.cuh"

constexpr int kFusedStage = 64;     // edge staging per warp (accepts are rare here)
constexpr int kFusedHash = 1024;    // resolver hash slots (group lists: <= kGroupCap)
constexpr int kFusedHashLog2 = 10;
constexpr int kDefCap = 128;        // survivors per warp a vertex may defer to the next

__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.wait_all;" ::: "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

template <int KIND, int G, int V, int MAXR>
__global__ void __launch_bounds__(kBloomBlock, SNGB_FUSED_MINB)
    k_floyd_head(const SamplerArgs a, const GatherArgs g, const HeadArgs h) {
    constexpr int kT = kBloomThreads;
    constexpr int NG = 32 / G;
    constexpr int UF = SNGB_FUSED_UF;
    constexpr int STEP = NG * UF;
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t WB = a.hash_mask;  // filter words (2^B / 32)
    const uint32_t shift = 32 - a.key_bits;
    const uint32_t W = a.col_words;
    uint32_t* filt = reinterpret_cast<uint32_t*>(smem);          // [2][WB]
    uint32_t* shared_bits = filt + 2 * WB;                         // [2][WB]
    uint32_t* colbits = shared_bits + 2 * WB;                      // [W]
    unsigned long long* glist =
        reinterpret_cast<unsigned long long*>(colbits + W);       // [2][kGroupCap]
    uint32_t* clist = reinterpret_cast<uint32_t*>(glist + 2 * kGroupCap);  // [2][kChainCap]
    unsigned long long* htab =
        reinterpret_cast<unsigned long long*>(clist + 2 * kChainCap);  // [kFusedHash]
    __shared__ uint32_t s_cnt[2][2];  // [parity][group, chain]
    __shared__ unsigned long long s_u[3];  // claimed vertices: ring of the last three
    __shared__ unsigned long long s_stage[kBloomThreads / 32][kFusedStage];
    __shared__ uint32_t s_t[MAXR * kBloomThreads];  // this vertex's draws, slot-major
    __shared__ uint32_t s_h[MAXR * kBloomThreads];  // their partners' head words (cp.async)
    __shared__ uint32_t s_defq[kBloomThreads / 32][2][kDefCap];  // deferred survivors per warp

    const int tid = threadIdx.x, lane = tid & 31, wib = tid >> 5;
    const bool resolver = tid >= kT;
    const EdgeSink xs{a.extras, a.extras_capacity, &a.counters[C_EXTRA_CURSOR], 0};
    const uint32_t D = a.draws, base = a.base;
    unsigned long long ncol = 0, nrep = 0;

    for (uint32_t s = tid; s < 4 * WB + W; s += kBloomBlock) filt[s] = 0;
    for (uint32_t s = tid; s < kFusedHash; s += kBloomBlock) htab[s] = ~0ull;
    if (tid < 4) (&s_cnt[0][0])[tid] = 0;
    if (tid == 0) s_u[0] = a.row_begin + atomicAdd(g.work, 1ull);
    __syncthreads();

    auto emit = [&](uint64_t u, uint32_t e) {  // extra pair (u, partner of value e)
        const unsigned long long s2 = atomicAdd(xs.cursor, 1ull);
        if (s2 < xs.capacity)
            xs.keys[s2] = ((unsigned long long)u << 32) | (e + (e >= (uint32_t)u ? 1u : 0u));
    };

    if (resolver) {
        // ---- the resolver warp, one vertex behind the workers (k_floyd_bloom P3) ----
        uint32_t par = 0;
        for (uint32_t k = 0;; ++k) {
            par ^= 1u;
            bar_sync(kBarReady + par, kBloomBlock);
            const uint64_t u = s_u[k % 3];
            if (u >= a.row_end) break;  // the workers' end-of-rows sentinel
            unsigned long long* gl = glist + par * kGroupCap;
            uint32_t* cl = clist + par * kChainCap;
            uint32_t* cnt = s_cnt[par];
            const uint32_t ng = cnt[0], nc = cnt[1];
            if (ng || nc) {
                for (uint32_t p = lane; p < ng; p += 32) {
                    const unsigned long long e = gl[p];
                    const uint32_t t = (uint32_t)(e >> 32);
                    uint32_t hh = (t * 0x85EBCA6Bu) >> (32 - kFusedHashLog2);
                    for (;;) {
                        const unsigned long long old = atomicCAS(&htab[hh], ~0ull, e);
                        if (old == ~0ull) break;
                        if ((uint32_t)(old >> 32) == t) {
                            atomicMin(&htab[hh], e);
                            break;
                        }
                        hh = (hh + 1) & (kFusedHash - 1);
                    }
                }
                __syncwarp();
                for (uint32_t p = lane; p < ng; p += 32) {
                    const unsigned long long e = gl[p];
                    const uint32_t t = (uint32_t)(e >> 32), i = (uint32_t)e;
                    uint32_t hh = (t * 0x85EBCA6Bu) >> (32 - kFusedHashLog2);
                    while ((uint32_t)(htab[hh] >> 32) != t) hh = (hh + 1) & (kFusedHash - 1);
                    if ((uint32_t)htab[hh] != i) {  // an earlier draw has the same value
                        atomicOr(&colbits[i >> 5], 1u << (i & 31));
                        emit(u, base + i);
                        ++ncol;
                    }
                }
                __syncwarp();
                for (uint32_t s2 = lane; s2 < kFusedHash; s2 += 32) htab[s2] = ~0ull;
                __syncwarp();
                if (lane == 0 && nc) {
                    const uint64_t key = vertex_key(a.seed_mixed, u);
                    for (uint32_t x = 1; x < nc; ++x) {  // insertion sort (tiny list)
                        const uint32_t v = cl[x];
                        uint32_t y = x;
                        while (y > 0 && cl[y - 1] > v) {
                            cl[y] = cl[y - 1];
                            --y;
                        }
                        cl[y] = v;
                    }
                    for (uint32_t x = 0; x < nc; ++x) {
                        const uint32_t i = cl[x];
                        if ((colbits[i >> 5] >> (i & 31)) & 1u) continue;  // already collided
                        bool fi;
                        const uint32_t kk =
                            lemire32(stream_at(key, (uint64_t)i + 1), base + i + 1, fi) - base;
                        if ((colbits[kk >> 5] >> (kk & 31)) & 1u) {
                            colbits[i >> 5] |= 1u << (i & 31);
                            emit(u, base + i);
                            ++ncol;
                        }
                    }
                }
                __syncwarp();
                for (uint32_t p = lane; p < ng + nc; p += 32) {  // clear the touched words
                    const uint32_t i = p < ng ? (uint32_t)gl[p] : cl[p - ng];
                    colbits[i >> 5] = 0;
                }
                __syncwarp();
                if (lane == 0) cnt[0] = cnt[1] = 0;
            }
            __syncwarp();
            bar_arrive(kBarFree + par, kBloomBlock);
        }
    } else {
        const float4* __restrict__ P = reinterpret_cast<const float4*>(g.tp.pts);
        const char* __restrict__ H = static_cast<const char*>(h.head);
        const uint32_t Wr = g.tp.stride / 4;
        const float reject = h.reject;
        const int q = lane % G, grp = lane / G;
        const bool leader = (q == 0);
        const uint64_t pol = evict_first_policy();  // survivor rows must not evict the heads
        WarpStage<kFusedStage> stage{s_stage[wib], 0};
        TestStats st;
        uint32_t gpairs = 0, tails = 0;
        // this thread's draw slot r lives at +4 kT r from these (slot-major: conflict-free)
        const uint32_t ta = smem_addr(s_t) + 4u * tid, ha = smem_addr(s_h) + 4u * tid;
        // the warp's slots, numbered j = 32 r + lane, double as its survivor queue in H
        const uint32_t qa = smem_addr(s_t) + 4u * (wib * 32);
        auto qaddr = [&](uint32_t j) { return qa + 4u * ((j >> 5) * kT + (j & 31)); };
        // deferred survivors: vertex k's are tested during vertex k + 1's draws, their
        // rows prefetched to L2 in between (HBM latency off the vertex's critical path)
        uint32_t dn = 0, dcur = 0;
        uint64_t u_prev = 0;
        F4x2 qv_prev[V];
#pragma unroll
        for (int vv = 0; vv < V; ++vv) qv_prev[vv] = F4x2{0, 0};

        // fp32 test of survivors [e0, e0 + STEP) of `qend` (entry e read by ld(e))
        // against query row qvx of vertex ux: G lanes per row, UF rows per group
        auto fp32_step = [&](auto ld, uint32_t e0, uint32_t qend, const F4x2* qvx, uint64_t ux) {
            F4x2 rows[UF][V];
            uint32_t pe[UF];
            bool oke[UF];
#pragma unroll
            for (int uu = 0; uu < UF; ++uu) {
                const uint32_t e = e0 + grp + NG * uu;
                oke[uu] = e < qend;
                pe[uu] = ld(oke[uu] ? e : e0);
#pragma unroll
                for (int vv = 0; vv < V; ++vv) {
                    const uint32_t c = q + G * vv;
                    const uint64_t row = (oke[uu] && c < Wr) ? pe[uu] : ux;
                    rows[uu][vv] = ldg_row2_ef(P + row * Wr + (c < Wr ? c : Wr - 1), pol);
                }
            }
            __syncwarp();
#pragma unroll
            for (int uu = 0; uu < UF; ++uu) {
                Acc2 acc;
#pragma unroll
                for (int vv = 0; vv < V; ++vv) diff2x2(qvx[vv], rows[uu][vv], acc);
                float sum = acc2_sum(acc);
#pragma unroll
                for (int o = G / 2; o > 0; o >>= 1) sum += __shfl_xor_sync(kFull, sum, o);
                const bool accd = decide(sum, oke[uu], leader, grp * G, g.tp, ux, pe[uu], st);
                tails += (oke[uu] && leader) ? 1u : 0u;
                stage.push(leader && accd, edge_key(ux, pe[uu], g.sink.nb), g.sink, lane);
            }
        };
        auto run_deferred = [&]() {
            const uint32_t* dq = s_defq[wib][dcur];
#pragma unroll 1
            for (uint32_t e0 = 0; e0 < dn; e0 += STEP)
                fp32_step([&](uint32_t e) { return dq[e]; }, e0, dn, qv_prev, u_prev);
            dn = 0;
        };

        uint32_t par = 0;
        const uint64_t dz = (uint64_t)kT * kGamma;  // counter step between a thread's draws
        for (uint32_t k = 0;; ++k) {
            par ^= 1u;
            if (k >= 2) bar_sync(kBarFree + par, kBloomBlock);  // parity par reusable
            const uint64_t u = s_u[k % 3];
            if (u >= a.row_end) {
                bar_arrive(kBarReady + par, kBloomBlock);  // tell the resolver to stop
                break;
            }
            uint32_t* f = filt + par * WB;
            uint32_t* sb = shared_bits + par * WB;
            unsigned long long* gl = glist + par * kGroupCap;
            uint32_t* cl = clist + par * kChainCap;
            uint32_t* cnt = s_cnt[par];
            {  // clear the other parity's filters (last used by vertex k - 1)
                uint4* fo = reinterpret_cast<uint4*>(filt + (par ^ 1u) * WB);
                uint4* so = reinterpret_cast<uint4*>(shared_bits + (par ^ 1u) * WB);
                const uint4 z4 = make_uint4(0, 0, 0, 0);
                for (uint32_t w = tid; w < WB / 4; w += kT) {
                    fo[w] = z4;
                    so[w] = z4;
                }
            }
            if (tid == 0) s_u[(k + 1) % 3] = a.row_begin + atomicAdd(g.work, 1ull);  // next vertex
            // the query's head and fp32 row (G lanes x V float4), loaded early
            const uint32_t hq = head_load<KIND>(H, (uint32_t)u);
            F4x2 qv[V];
#pragma unroll
            for (int vv = 0; vv < V; ++vv) {
                const uint32_t c = q + G * vv;
                qv[vv] = to_x2(ldg_row(P + u * Wr + (c < Wr ? c : Wr - 1)));
            }
            const uint64_t key = vertex_key(a.seed_mixed, u);
            uint64_t z = key + (uint64_t)(tid + 1) * kGamma;  // stream_at(key, i + 1), i = tid
            const uint32_t fa = smem_addr(f), sa = smem_addr(sb);
            const uint32_t nfull = D / kT;  // slots in which every thread has a draw
            const uint32_t forced_i =
                (a.force_mod != 0 && (u % a.force_mod) == 0) ? D / 2 : 0xffffffffu;

            // ---- P1: draw, filter bit, chain candidate, async head copy ----
            uint32_t chain = 0;
            bool fired = false;
#pragma unroll
            for (int r = 0; r < MAXR; ++r, z += dz) {
                const uint32_t i = tid + kT * r;
                if ((uint32_t)r < nfull || i < D) {
                    bool fi;
                    const uint32_t t = lemire32(mix(z), base + i + 1, fi);
                    fired |= fi | (i == forced_i);
                    const uint32_t hh = (t * 0x9E3779B1u) >> shift;
                    const uint32_t off = (hh >> 5) * 4u, bit = 1u << (hh & 31);
                    red_or_sh_if(sa + off, bit, atom_or_sh(fa + off, bit) & bit);
                    chain |= (t - base < i ? 1u : 0u) << r;
                    st_sh(ta + 4u * kT * r, t);
                    const uint32_t p = t + (t >= (uint32_t)u ? 1u : 0u);
                    // the 4-byte word holding p's head (2-byte heads: the aligned pair)
                    const uint64_t hoff = KIND == kHeadU8x2 ? (uint64_t)(p & ~1u) * 2u
                                                            : (uint64_t)p * 4u;
                    cp_async4(ha + 4u * kT * r, H + hoff);
                }
            }
            cp_async_commit();
            if (chain) {  // rare (about draws/n per draw)
#pragma unroll
                for (int r = 0; r < MAXR; ++r)
                    if ((chain >> r) & 1u) {
                        const uint32_t p = atomicAdd(&cnt[1], 1u);
                        if (p < kChainCap) cl[p] = tid + kT * r;
                    }
            }
            // the previous vertex's survivors, while this vertex's heads arrive
            if (dn) run_deferred();
            auto replay = [&]() {  // exact sequential replay (k_floyd_bloom), rare
                cp_async_wait_all();  // no copy of this vertex may land after the next one's
                bar_sync(kBarWorkers, kT);
                if (tid == 0) {
                    ++nrep;
                    bloom_replay(key, u, a.n, base, filt, 4 * WB, xs);
                    cnt[0] = cnt[1] = 0;
                }
                bar_sync(kBarWorkers, kT);
                for (uint32_t s = tid; s < 4 * WB; s += kT) filt[s] = 0;
                bar_sync(kBarWorkers, kT);
                bar_arrive(kBarReady + par, kBloomBlock);
            };
            if (bar_or(kBarWorkers, kT, fired)) {  // irregular vertex: all partners are extras
                replay();
                continue;
            }
            // ---- P2: draws on a shared filter bit -> the group list ----
#pragma unroll 4
            for (int r = 0; r < MAXR; ++r) {
                const uint32_t i = tid + kT * r;
                if ((uint32_t)r * kT >= D) break;
                if ((uint32_t)r < nfull || i < D) {
                    const uint32_t t = ld_sh(ta + 4u * kT * r);
                    const uint32_t hh = (t * 0x9E3779B1u) >> shift;
                    if ((ld_sh(sa + (hh >> 5) * 4u) >> (hh & 31)) & 1u) {
                        const uint32_t p = atomicAdd(&cnt[0], 1u);
                        if (p < kGroupCap) gl[p] = ((unsigned long long)t << 32) | i;
                    }
                }
            }
            bar_sync(kBarWorkers, kT);
            if (cnt[0] > kGroupCap || cnt[1] > kChainCap) {  // list overflow: exact replay
                replay();
                continue;
            }
            bar_arrive(kBarReady + par, kBloomBlock);

            // ---- H: head tests (the resolver runs meanwhile) ----
            cp_async_wait_all();
            __syncwarp();
            uint32_t qn = 0;
#pragma unroll 2
            for (int r = 0; r < MAXR; ++r) {
                if ((uint32_t)r * kT >= D) break;  // uniform
                const uint32_t i = tid + kT * r;
                const bool valid = (uint32_t)r < nfull || i < D;
                gpairs += valid ? 1u : 0u;
                const uint32_t t = ld_sh(ta + 4u * kT * r);
                const uint32_t p = t + (t >= (uint32_t)u ? 1u : 0u);
                const uint32_t w = ld_sh(ha + 4u * kT * r);
                const uint32_t hv = KIND == kHeadU8x2 ? ((p & 1u) ? (w >> 16) : (w & 0xffffu)) : w;
                const bool keep = valid && !(head_q<KIND>(hq, hv) > reject);
                const unsigned km = __ballot_sync(kFull, keep);
                __syncwarp();  // every lane read slot r before the queue overwrites it
                if (keep) st_sh(qaddr(qn + __popc(km & lanemask_lt())), p);
                qn += __popc(km);
            }
            __syncwarp();
            if (qn <= (uint32_t)kDefCap) {
                // defer: copy to the idle deferred queue, prefetch the rows into L2
                uint32_t* dq = s_defq[wib][dcur ^ 1u];
                for (uint32_t e = lane; e < qn; e += 32) {
                    const uint32_t p = ld_sh(qaddr(e));
                    dq[e] = p;
                    const char* row = reinterpret_cast<const char*>(P + (uint64_t)p * Wr);
                    for (uint32_t b = 0; b < Wr * 16; b += 128) prefetch_l2(row + b);
                }
                __syncwarp();
                dcur ^= 1u;
                dn = qn;
                u_prev = u;
#pragma unroll
                for (int vv = 0; vv < V; ++vv) qv_prev[vv] = qv[vv];
            } else {  // a dense vertex: test its survivors now
#pragma unroll 1
                for (uint32_t e0 = 0; e0 < qn; e0 += STEP)
                    fp32_step([&](uint32_t e) { return ld_sh(qaddr(e)); }, e0, qn, qv, u);
            }
            __syncwarp();
        }
        if (dn) run_deferred();
        stage.flush(g.sink, lane);
        st.pairs = gpairs;
        flush_stats(st, gpairs, g.counters, lane);
        const unsigned long long tw = warp_sum((unsigned long long)tails);
        if (lane == 0 && tw) atomicAdd(&g.counters[C_TAIL_PAIRS], tw);
    }
    ncol = warp_sum(ncol);
    if (lane == 0) {
        if (ncol) atomicAdd(&a.counters[C_COLLISIONS], ncol);
        if (nrep) atomicAdd(&a.counters[C_IRREGULAR], nrep);
    }
}

size_t fused_smem_bytes(const BloomGeom& bg) {
    return 4ull * bg.words * 4 + (size_t)bg.col_words * 4 + 2ull * kGroupCap * 8 +
           2ull * kChainCap * 4 + (size_t)kFusedHash * 8;
}

template <int KIND, int G, int V, int MAXR>
cudaError_t fused_one(const SamplerArgs& sa, const GatherArgs& ga, const HeadArgs& h,
                      cudaStream_t s, int num_sms, size_t smem) {
    auto k = k_floyd_head<KIND, G, V, MAXR>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kBloomBlock, smem);
    if (per_sm < 1) per_sm = 1;
    const uint64_t rows = sa.row_end - sa.row_begin;
    const uint64_t cap = (uint64_t)num_sms * per_sm;
    k<<<(unsigned)(rows < cap ? rows : cap), kBloomBlock, smem, s>>>(sa, ga, h);
    note_launch(1);
    return cudaGetLastError();
}

template <int KIND, int MAXR>
cudaError_t fused_rows(const SamplerArgs& sa, const GatherArgs& ga, const HeadArgs& h,
                       cudaStream_t s, int num_sms, size_t smem) {
    const uint32_t W = ga.tp.stride / 4;
    if (W <= 2) return fused_one<KIND, 2, 1, MAXR>(sa, ga, h, s, num_sms, smem);
    if (W <= 4) return fused_one<KIND, 4, 1, MAXR>(sa, ga, h, s, num_sms, smem);
    if (W <= 8) return fused_one<KIND, 8, 1, MAXR>(sa, ga, h, s, num_sms, smem);
    if (W <= 16) return fused_one<KIND, 16, 1, MAXR>(sa, ga, h, s, num_sms, smem);
    if (W <= 32) return fused_one<KIND, 32, 1, MAXR>(sa, ga, h, s, num_sms, smem);
    return cudaErrorInvalidValue;
}

template <int KIND>
cudaError_t fused_kind(const SamplerArgs& sa, const GatherArgs& ga, const HeadArgs& h,
                       cudaStream_t s, int num_sms, size_t smem) {
    const uint32_t D = sa.draws;
    if (D <= 1024) return fused_rows<KIND, 4>(sa, ga, h, s, num_sms, smem);
    if (D <= 2560) return fused_rows<KIND, 10>(sa, ga, h, s, num_sms, smem);
    return fused_rows<KIND, 16>(sa, ga, h, s, num_sms, smem);
}

}  // namespace

#ifndef SNGB_FUSED_DEFAULT
#define SNGB_FUSED_DEFAULT 0
#endif
constexpr int kFusedDefault = SNGB_FUSED_DEFAULT;

bool fused_eligible(uint64_t n, uint32_t draws, uint32_t stride) {
    // SNGB_FUSED=0 keeps the two kernels, 1 fuses (default: SNGB_FUSED_DEFAULT).  Fused wherever launch_sampler would
    // pick k_floyd_bloom (n beyond the per-warp bitmap kernel's 73 k, or
    // SNGB_FLOYD_NO_BITMAP; draws <= 4096) for rows of <= 32 float4
    const char* e = std::getenv("SNGB_FUSED");
    const int mode = e ? std::atoi(e) : kFusedDefault;
    if (mode == 0 || draws < 1 || draws > 4096 || n - 2 >= 0xffffffffull ||
        stride / 4 > 32)
        return false;
    const uint64_t bm_words = (((n - 1) + 31) / 32 + 3) & ~3ull;
    return bm_words * 4 > 9216 || std::getenv("SNGB_FLOYD_NO_BITMAP") != nullptr;
}

cudaError_t launch_floyd_head(const SamplerArgs& in, const GatherArgs& ga, const HeadArgs& h,
                              cudaStream_t s, int num_sms) {
    const uint64_t rows = in.row_end - in.row_begin;
    if (rows == 0 || in.draws == 0) return cudaSuccess;
    if (!ga.work) return cudaErrorInvalidValue;  // dynamic claiming needs a zeroed counter
    SamplerArgs a = in;
    const BloomGeom bg = bloom_geometry(a.draws);
    a.hash_mask = bg.words;
    a.key_bits = bg.bits_log2;
    a.col_words = bg.col_words;
    const size_t smem = fused_smem_bytes(bg);
    switch (h.kind) {
        case kHeadU16x2: return fused_kind<kHeadU16x2>(a, ga, h, s, num_sms, smem);
        case kHeadU8x4: return fused_kind<kHeadU8x4>(a, ga, h, s, num_sms, smem);
        default: return fused_kind<kHeadU8x2>(a, ga, h, s, num_sms, smem);
    }
}

}  // namespace sngb
