// sngb_floyd_head.cuh -- k_floyd_head: k_floyd_lean's Floyd bookkeeping and the
// head-filter gather (sngb_head.cu) in one block-per-vertex kernel, each draw
// generated once, the survivors' fp32 rows tested off the workers' path
// (large n, 1024 < draws <= 4096, narrow rows: cfg4, cfg5).  Included by
// sngb_fused.cu after sngb_floyd_bloom.cuh and sngb_floyd_lean.cuh.
//
// Why.  As two kernels, k_floyd_lean (2.64 warp-instructions per draw) and
// k_gather_head (2.92) each regenerate every draw
//   t_i = Lemire(mix(key + (i+1) gamma), base + i + 1)   (rng.hpp:26,35-48)
// and, sharing the SMs, they are issue-bound together (cfg5: 629 ms for 8e10
// draws, ncu profiles/r02_ncu_floyd_lean_cfg5.md, r01_ncu_head_cfg5.md).  The
// warp-per-vertex fusions (k_sample_head) tested each vertex's survivors inline
// and stalled on their HBM rows (99 registers, long-scoreboard bound).  Here a
// block owns one vertex at a time and splits the work by warp role:
//
//   workers (8 warps, 16 draws per thread for D = 4000), per vertex:
//     P1  t_i, k_floyd_lean's filter bit and running tests; the partner's head
//         load (partner p = t + (t >= u), graph.cpp:172-173) is issued here and
//         consumed in P2, so its L2 latency hides behind the rest of P1;
//     P2  the group list (k_floyd_lean) and the exact head reject
//         (sngb_head.cu): survivors' partners -> the vertex's survivor queue;
//   resolver (1 warp), one vertex behind: P3 (bloom_resolve_vertex: collided
//     draws -> extras);
//   testers (SNGB_FH_TESTERS warps), one vertex behind: the survivors' fp32
//     test on their full rows (UF rows per G-lane group in flight), edges to
//     the sink, guard-band pairs to k_band -- the same decision code as
//     k_gather_head (sngb_epstest.cuh).
// Lists and the survivor queue are double-buffered by vertex parity; the
// consumers (resolver + testers) release a parity with one named barrier.  A
// vertex whose stream meets the Lemire reject pre-condition (or the test hook)
// is replayed exactly by one worker (bloom_replay: every partner an extra) and
// skips its head tests; its gather-pair count is the draws before the first
// fired one, as k_gather_head counts them.  Results equal the two-kernel path
// bit for bit (tests/test_gpu_parity.py -k floyd_head).
#pragma once

#ifndef SNGB_FH_TESTERS
#define SNGB_FH_TESTERS 4
#endif
constexpr int kFhTesters = SNGB_FH_TESTERS;
constexpr int kFhConsumers = 32 * (1 + kFhTesters);
constexpr int kFhBlock = kBloomThreads + kFhConsumers;
constexpr int kFhStage = 64;  // edge staging per tester warp

// dynamic shared memory: k_floyd_bloom's tables, then the survivor queues
// [2][scap] and the testers' edge stages
inline size_t fh_smem_bytes(const BloomGeom& g, uint32_t scap) {
    return bloom_smem_bytes(g) + 2ull * scap * 4 + (size_t)kFhTesters * kFhStage * 8;
}

// testers: G lanes per survivor row, V 16-byte chunks per lane, UF rows per
// group in flight (G * V * 16 bytes >= the row; G * V * UF <= 8 chunks of
// registers per lane)
template <int KIND, int G, int V>
__global__ void __launch_bounds__(kFhBlock, 2)
    k_floyd_head(const SamplerArgs a, const GatherArgs g, const HeadArgs h, uint32_t scap) {
    constexpr int kT = kBloomThreads;
    constexpr int MAXR = 16;  // draws <= 4096: at most 16 slots per worker thread
    constexpr int NG = 32 / G;
    constexpr int UF = V >= 4 ? 2 : 4;  // fp32 rows per group per tester step
    constexpr int STEP = NG * UF;   // survivors per tester step
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t WB = a.hash_mask;  // filter words (2^B / 32)
    const uint32_t W = a.col_words;
    uint32_t* filt = reinterpret_cast<uint32_t*>(smem);          // [2][WB]
    uint32_t* shared_bits = filt + 2 * WB;                         // [2][WB]
    uint32_t* colbits = shared_bits + 2 * WB;                      // [W]
    unsigned long long* glist =
        reinterpret_cast<unsigned long long*>(colbits + W);       // [2][kGroupCap]
    uint32_t* clist = reinterpret_cast<uint32_t*>(glist + 2 * kGroupCap);  // [2][kChainCap]
    unsigned long long* htab =
        reinterpret_cast<unsigned long long*>(clist + 2 * kChainCap);  // [kHashSlots]
    uint32_t* squeue = reinterpret_cast<uint32_t*>(htab + kHashSlots);   // [2][scap]
    unsigned long long* stages =
        reinterpret_cast<unsigned long long*>(squeue + 2 * scap);      // [kFhTesters][kFhStage]
    __shared__ uint32_t s_cnt[2][2];  // [parity][group, chain]
    __shared__ uint32_t s_scnt[2];    // [parity] survivors
    __shared__ uint32_t s_lim;        // first fired draw of the vertex being replayed

    const int tid = threadIdx.x, lane = tid & 31;
    const EdgeSink xs{a.extras, a.extras_capacity, &a.counters[C_EXTRA_CURSOR], 0};
    const uint32_t D = a.draws, base = a.base;
    const void* __restrict__ H = h.head;
    const float reject = h.reject;
    unsigned long long ncol = 0, nrep = 0, gpairs = 0;

    for (uint32_t s = tid; s < 4 * WB + W; s += kFhBlock) filt[s] = 0;
    for (uint32_t s = tid; s < kHashSlots; s += kFhBlock) htab[s] = ~0ull;
    if (tid < 4) (&s_cnt[0][0])[tid] = 0;
    if (tid < 2) s_scnt[tid] = 0;
    if (tid == 0) s_lim = D;
    __syncthreads();

    if (tid >= kT) {
        // ---------------- consumers, one vertex behind the workers ----------------
        const int cw = (tid - kT) >> 5;  // 0: resolver, 1..: testers
        const int tw = cw - 1;
        const int q = lane % G, grp = lane / G;
        const bool leader = q == 0;
        const float4* __restrict__ P = reinterpret_cast<const float4*>(g.tp.pts);
        const uint32_t RW = g.tp.stride / 4;
        const uint64_t pol = evict_first_policy();  // survivor rows must not evict the heads
        WarpStage<kFhStage> stage{stages + (tw > 0 ? tw : 0) * kFhStage, 0};
        TestStats st;
        unsigned long long tails = 0;
        uint32_t par = 0;
        for (uint64_t u = a.row_begin + blockIdx.x; u < a.row_end; u += gridDim.x) {
            par ^= 1u;
            bar_sync(kBarReady + par, kFhBlock);
            if (cw == 0) {
                bloom_resolve_vertex(a, u, par, glist, clist, s_cnt, colbits, htab, xs, lane, ncol);
            } else {
                const uint32_t ns = s_scnt[par];
                const uint32_t* sq = squeue + par * scap;
                if (ns > (uint32_t)(tw * STEP)) {
                    F4x2 qv[V];
#pragma unroll
                    for (int vv = 0; vv < V; ++vv) {
                        const uint32_t c = q + G * vv;
                        qv[vv] = to_x2(ldg_row(P + u * RW + (c < RW ? c : RW - 1)));
                    }
                    for (uint32_t e0 = tw * STEP; e0 < ns; e0 += kFhTesters * STEP) {
                        F4x2 rows[UF][V];
                        uint32_t pe[UF];
                        bool oke[UF];
#pragma unroll
                        for (int uu = 0; uu < UF; ++uu) {
                            const uint32_t e = e0 + grp + NG * uu;
                            oke[uu] = e < ns;
                            pe[uu] = sq[oke[uu] ? e : e0];
#pragma unroll
                            for (int vv = 0; vv < V; ++vv) {
                                const uint32_t c = q + G * vv;
                                const uint64_t row = (oke[uu] && c < RW) ? pe[uu] : u;
                                rows[uu][vv] = ldg_row2_ef(P + row * RW + (c < RW ? c : RW - 1), pol);
                            }
                        }
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
                    }
                }
                __syncwarp();
            }
            bar_arrive(kBarFree + par, kFhBlock);
        }
        if (cw > 0) {
            stage.flush(g.sink, lane);
            flush_stats(st, 0, g.counters, lane);
            const unsigned long long t2 = warp_sum(tails);
            if (lane == 0 && t2) atomicAdd(&g.counters[C_TAIL_PAIRS], t2);
        }
    } else {
        // ---------------- workers ----------------
        uint32_t par = 0, vcount = 0;
        const uint64_t dz = (uint64_t)kT * kGamma;  // counter step between a thread's draws
        const uint32_t nslots = (D + kT - 1) / kT;  // block-uniform; the last slot is partial
        const bool in_tail = (uint32_t)tid < D - kT * (nslots - 1);
        const uint32_t wmask = (WB - 1) << 2;
        const uint32_t b0 = base + (uint32_t)tid + 1;  // Lemire bound of slot 0
        const bool hook_thread = a.force_mod != 0 && (D / 2) % kT == (uint32_t)tid;
        for (uint64_t u = a.row_begin + blockIdx.x; u < a.row_end; u += gridDim.x) {
            par ^= 1u;
            if (++vcount > 2) bar_sync(kBarFree + par, kFhBlock);  // parity par reusable
            unsigned long long* gl = glist + par * kGroupCap;
            uint32_t* cl = clist + par * kChainCap;
            uint32_t* cnt = s_cnt[par];
            uint32_t* sq = squeue + par * scap;
            if (tid == 0) s_scnt[par] = 0;  // ordered before P2's pushes by bar_or
            {  // clear the other parity's filters (last used by vertex u - 1)
                uint4* fo = reinterpret_cast<uint4*>(filt + (par ^ 1u) * WB);
                uint4* so = reinterpret_cast<uint4*>(shared_bits + (par ^ 1u) * WB);
                const uint4 z4 = make_uint4(0, 0, 0, 0);
                for (uint32_t w = tid; w < WB / 4; w += kT) {
                    fo[w] = z4;
                    so[w] = z4;
                }
            }
            const uint64_t key = vertex_key(a.seed_mixed, u);
            const uint64_t z0 = key + (uint64_t)(tid + 1) * kGamma;
            const uint32_t fa = smem_addr(filt + par * WB), sa = smem_addr(shared_bits + par * WB);
            const uint32_t u32 = (uint32_t)u;
            const uint32_t hq = head_load<KIND>(H, u32);

            // ---- P1 ----
            uint32_t tr[MAXR], hb[MAXR];
            uint32_t smin = 0xffffffffu, tmax = 0;
#pragma unroll
            for (int r = 0; r < MAXR; ++r) {
                if ((uint32_t)r >= nslots) break;
                uint32_t slo;
                const uint32_t t = lemire32_slo(mix(z0 + (uint64_t)r * dz), b0 + kT * r, slo);
                tr[r] = t;
                const bool valid = (uint32_t)r + 1 < nslots || in_tail;
                const uint32_t p = t + (t >= u32 ? 1u : 0u);
                hb[r] = head_load32<KIND>(H, valid ? p : u32);  // consumed in P2
                if (valid) {
                    smin = min(smin, slo);
                    tmax = max(tmax, t);
                    const uint32_t off = (t >> 3) & wmask, bit = 1u << (t & 31);
                    red_or_sh(sa + off, atom_or_sh(fa + off, bit) & bit);
                }
            }
            // exact tests for the rare flagged threads
            uint32_t first_fire = hook_thread && (u % a.force_mod) == 0 ? D / 2 : D;
            if (smin == 0u) {  // the exact pre-condition, lo < bound
#pragma unroll 1
                for (uint32_t r = 0; r < nslots; ++r) {
                    bool fi;
                    lemire32(mix(z0 + (uint64_t)r * dz), b0 + kT * r, fi);
                    const uint32_t i = (uint32_t)tid + kT * r;
                    if (fi && (r + 1 < nslots || in_tail) && i < first_fire) first_fire = i;
                }
            }
            const bool fired = first_fire < D;
            if (fired) atomicMin(&s_lim, first_fire);
            if (tmax >= base) {  // chain candidates: t - base < i
#pragma unroll
                for (int r = 0; r < MAXR; ++r) {
                    if ((uint32_t)r >= nslots) break;
                    const uint32_t i = (uint32_t)tid + kT * r;
                    if (((uint32_t)r + 1 < nslots || in_tail) && tr[r] - base < i) {
                        const uint32_t pp = atomicAdd(&cnt[1], 1u);
                        if (pp < kChainCap) cl[pp] = i;
                    }
                }
            }
            // exact sequential replay of the vertex (rare), as k_floyd_lean
            auto replay = [&]() {
                bar_sync(kBarWorkers, kT);
                if (tid == 0) {
                    ++nrep;
                    ncol += bloom_replay(key, u, a.n, base, filt, 4 * WB, xs);
                    cnt[0] = cnt[1] = 0;
                }
                bar_sync(kBarWorkers, kT);
                for (uint32_t s = tid; s < 4 * WB; s += kT) filt[s] = 0;
                bar_sync(kBarWorkers, kT);
                bar_arrive(kBarReady + par, kFhBlock);
            };
            if (bar_or(kBarWorkers, kT, fired)) {
                // the head tests stop at the first fired draw (k_gather_head's
                // limit); the replay emits every partner as an extra
                if (tid == 0) {
                    gpairs += s_lim;
                    s_lim = D;
                }
                replay();
                continue;
            }
            // ---- P2: group list + head reject ----
#pragma unroll
            for (int r = 0; r < MAXR; ++r) {
                if ((uint32_t)r >= nslots) break;
                const uint32_t t = tr[r];
                const bool valid = (uint32_t)r + 1 < nslots || in_tail;
                const uint32_t off = (t >> 3) & wmask, bit = 1u << (t & 31);
                if ((ld_sh(sa + off) & bit) && valid) {
                    const uint32_t pp = atomicAdd(&cnt[0], 1u);
                    if (pp < kGroupCap) gl[pp] = ((unsigned long long)t << 32) | ((uint32_t)tid + kT * r);
                }
                if (valid && !(head_q<KIND>(hq, hb[r]) > reject)) {
                    const uint32_t pp = atomicAdd(&s_scnt[par], 1u);  // < D <= scap
                    sq[pp] = t + (t >= u32 ? 1u : 0u);
                }
            }
            if (tid == 0) gpairs += D;
            bar_sync(kBarWorkers, kT);
            if (cnt[0] > kGroupCap || cnt[1] > kChainCap) {  // list overflow: exact replay
                replay();  // the survivors stay queued: every draw was head-tested
                continue;
            }
            bar_arrive(kBarReady + par, kFhBlock);
        }
        if (tid < 32) {
            TestStats st;
            st.pairs = gpairs;
            flush_stats(st, gpairs, g.counters, lane);
        }
    }
    ncol = warp_sum(ncol);
    nrep = warp_sum(nrep);
    if (lane == 0) {
        if (ncol) atomicAdd(&a.counters[C_COLLISIONS], ncol);
        if (nrep) atomicAdd(&a.counters[C_IRREGULAR], nrep);
    }
}
