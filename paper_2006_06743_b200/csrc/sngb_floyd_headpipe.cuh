// sngb_floyd_headpipe.cuh -- k_floyd_headpipe: k_floyd_pipe's Floyd bookkeeping and
// the head-filter gather (sngb_head.cu) in one block-per-vertex kernel, each draw
// generated once (large n, 1024 < draws <= 4096, rows of <= 8 float4: cfg4, cfg5).
// Included by sngb_fused.cu after sngb_floyd_pipe.cuh.
//
// Why.  As two kernels, k_floyd_pipe (2.8 warp-instructions per draw) and
// k_gather_head (2.9) each regenerate every draw
//   t_i = Lemire(mix(key + (i+1) gamma), base + i + 1)   (rng.hpp:26,35-48)
// and, run side by side (k_duo), they queue on the same in-order L1TEX pipe and
// lose.  k_floyd_head fused them around a resolver warp and tester warps and was
// bound by those consumers' serial latency (46 % issue).  Here the eight worker
// warps of k_floyd_pipe do everything themselves:
//
//   P1(s)  as k_floyd_pipe, plus the partner's head load (p = t + (t >= u),
//          graph.cpp:172-173), issued here and consumed in P2 so its L2 latency
//          hides behind the rest of P1;
//   P2(s)  as k_floyd_pipe, plus the exact head reject (sngb_head.cu): survivors'
//          partners -> the warp's own queue (ballot + popc);
//   T(s)   each warp tests the survivors it found on their fp32 rows (G lanes per
//          row, UF rows per group in flight, evict-first loads): the same
//          decision code as k_gather_head (sngb_epstest.cuh: accept, reject, or
//          the band list for k_band), edges through the warp's stage;
//   A/B/C  the group entries' exact resolution, pipelined as in k_floyd_pipe.
//
// A vertex whose stream meets the Lemire reject pre-condition (or the test hook)
// is replayed exactly by one thread (bloom_replay: every partner an extra) and
// skips its head tests; its gather-pair count is the draws before the first
// fired one, as k_gather_head counts them.  Results equal the two-kernel path
// bit for bit (tests/test_gpu_parity.py -k headpipe).
#pragma once

#ifndef SNGB_FHP_UF
#define SNGB_FHP_UF 4
#endif
constexpr int kFhpQueue = 32 * 16;  // survivors per warp and vertex: every draw may survive
constexpr int kFhpStage = 64;       // edge staging per warp

inline size_t fhp_smem_bytes(const BloomGeom& g) {
    return pipe_smem_bytes(g) + (size_t)(kBloomThreads / 32) * (kFhpQueue * 4 + kFhpStage * 8);
}

template <int KIND, int G, int MAXR>
__device__ __forceinline__ void floyd_headpipe_run(const SamplerArgs& a, const GatherArgs& g,
                                                   const HeadArgs& hd, unsigned char* smem,
                                                   const uint64_t first, const uint64_t stride,
                                                   const uint32_t nv) {
    constexpr int kT = kBloomThreads;
    constexpr int kW = kT / 32;
    constexpr int NG = 32 / G;
    constexpr int UF = SNGB_FHP_UF;  // fp32 rows per G-lane group per survivor step
    constexpr int STEP = NG * UF;
    const uint32_t WB = a.hash_mask;  // filter words (2^B / 32)
    const uint32_t W = a.col_words;
    uint32_t* filt = reinterpret_cast<uint32_t*>(smem);          // [2][WB]
    uint32_t* shared_bits = filt + 2 * WB;                         // [2][WB]
    uint32_t* colbits = shared_bits + 2 * WB;                      // [2][W]
    unsigned long long* glist =
        reinterpret_cast<unsigned long long*>(colbits + 2 * W);   // [2][kW][kPipeSeg]
    uint32_t* clist = reinterpret_cast<uint32_t*>(glist + 2 * kW * kPipeSeg);  // [2][kChainCap]
    unsigned long long* htab =
        reinterpret_cast<unsigned long long*>(clist + 2 * kChainCap);  // [2][kPipeSlots]
    uint32_t* squeue = reinterpret_cast<uint32_t*>(htab + 2 * kPipeSlots);  // [kW][kFhpQueue]
    unsigned long long* stages =
        reinterpret_cast<unsigned long long*>(squeue + kW * kFhpQueue);  // [kW][kFhpStage]
    __shared__ uint32_t s_lim;  // first fired draw of a vertex being replayed
    __shared__ uint32_t s_wc[2][kW];  // [parity][warp] group entries
    __shared__ uint32_t s_ng[2];      // [parity] group entries of the vertex
    __shared__ uint32_t s_cc[2];      // [parity] chain candidates
    __shared__ uint32_t s_ovf[2];     // [parity] a list overflowed

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const EdgeSink xs{a.extras, a.extras_capacity, &a.counters[C_EXTRA_CURSOR], 0};
    const uint32_t D = a.draws, base = a.base;
    unsigned long long ncol = 0, nrep = 0, gpairs = 0, tails = 0;
    const void* __restrict__ H = hd.head;
    const float reject = hd.reject;
    const float4* __restrict__ P = reinterpret_cast<const float4*>(g.tp.pts);
    const uint32_t RW = g.tp.stride / 4;
    const int q = lane % G, grp = lane / G;
    const bool leader = q == 0;
    const uint64_t pol = evict_first_policy();  // survivor rows must not evict the heads
    uint32_t* myq = squeue + warp * kFhpQueue;
    WarpStage<kFhpStage> stage{stages + warp * kFhpStage, 0};
    TestStats st;
    auto emit = [&](uint64_t u, uint32_t e) {  // extra pair (u, partner of value e)
        const unsigned long long s2 = atomicAdd(xs.cursor, 1ull);
        if (s2 < xs.capacity)
            xs.keys[s2] = ((unsigned long long)u << 32) | (e + (e >= (uint32_t)u ? 1u : 0u));
    };

    for (uint32_t s = tid; s < 4 * WB + 2 * W; s += kT) filt[s] = 0;
    for (uint32_t s = tid; s < 2 * kPipeSlots; s += kT) htab[s] = ~0ull;
    if (tid < 2 * kW) (&s_wc[0][0])[tid] = 0;
    if (tid < 2) s_ng[tid] = s_cc[tid] = s_ovf[tid] = 0;
    if (tid == 0) s_lim = D;
    __syncthreads();

    const uint64_t dz = (uint64_t)kT * kGamma;  // counter step between a thread's draws
    // MAXR = ceil(D / kT): slots r < MAXR - 1 are full, the last one holds D - kT (MAXR - 1) draws
    const bool in_tail = (uint32_t)tid < D - kT * (MAXR - 1);
    const uint32_t wmask = (WB - 1) << 2;          // byte offset of t's filter word
    const uint32_t b0 = base + (uint32_t)tid + 1;  // Lemire bound of slot 0: j + 1
    const bool hook_thread = a.force_mod != 0 && (D / 2) % kT == (uint32_t)tid;
    const uint32_t lt = (1u << lane) - 1u;
    uint32_t h0 = kPipeNone, h1 = kPipeNone;  // hash slots of my entries (vertex s - 1)

    for (uint32_t s = 0; s < nv + 2; ++s) {
        const uint32_t par = s & 1u;
        const uint64_t u = first + (uint64_t)s * stride;  // vertex s (s < nv)
        const bool has_v = s < nv, has_prev = s >= 1 && s <= nv;
        unsigned long long* Hprev = htab + (par ^ 1u) * kPipeSlots;
        const unsigned long long* seg = glist + ((par ^ 1u) * kW + warp) * kPipeSeg;

        // ---- C: vertex s - 2 (parity par) ----
        if (s >= 2) {
            unsigned long long* H = htab + par * kPipeSlots;
            if (h0 != kPipeNone) H[h0] = ~0ull;
            if (h1 != kPipeNone) H[h1] = ~0ull;
            if (tid == 0) {
                const uint32_t nc = s_cc[par];
                if (nc) {
                    const uint64_t u2 = u - 2ull * stride;
                    uint32_t* cl = clist + par * kChainCap;
                    uint32_t* cb = colbits + par * W;
                    const uint64_t key = vertex_key(a.seed_mixed, u2);
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
                        if ((cb[i >> 5] >> (i & 31)) & 1u) continue;  // already collided
                        bool fi;
                        const uint32_t k =
                            lemire32(stream_at(key, (uint64_t)i + 1), base + i + 1, fi) - base;
                        if ((cb[k >> 5] >> (k & 31)) & 1u) {
                            cb[i >> 5] |= 1u << (i & 31);
                            emit(u2, base + i);
                            ++ncol;
                        }
                    }
                    s_cc[par] = 0;
                }
                s_ng[par] = 0;
            }
        }
        h0 = h1 = kPipeNone;

        // ---- A: vertex s - 1 (parity par ^ 1): first occurrence per value ----
        if (has_prev) {
            const uint32_t wc = s_wc[par ^ 1u][warp];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const uint32_t k = lane + 32 * q;
                if (k < wc) {
                    const unsigned long long e = seg[k];
                    const uint32_t t = (uint32_t)(e >> 32);
                    uint32_t h = (t * 0x85EBCA6Bu) >> (32 - kPipeHashLog2);
                    for (;;) {
                        const unsigned long long old = atomicCAS(&Hprev[h], ~0ull, e);
                        if (old == ~0ull) break;
                        if ((uint32_t)(old >> 32) == t) {
                            atomicMin(&Hprev[h], e);
                            break;
                        }
                        h = (h + 1) & (kPipeSlots - 1);
                    }
                }
            }
        }

        __syncwarp();  // reconverge after the divergent probe loops (else P1 runs per fragment)

        // ---- P1: vertex s ----
        uint32_t tr[MAXR], hb[MAXR];
        uint32_t tmax = 0;
        bool fired = false;
        uint64_t key = 0;
        uint32_t sa = 0, hq = 0;
        const uint32_t u32 = (uint32_t)u;
        if (has_v) {
            {  // clear the other parity's filters (last used by vertex s - 1)
                uint4* fo = reinterpret_cast<uint4*>(filt + (par ^ 1u) * WB);
                uint4* so = reinterpret_cast<uint4*>(shared_bits + (par ^ 1u) * WB);
                const uint4 z4 = make_uint4(0, 0, 0, 0);
                for (uint32_t w = tid; w < WB / 4; w += kT) {
                    fo[w] = z4;
                    so[w] = z4;
                }
            }
            key = vertex_key(a.seed_mixed, u);
            const uint64_t z0 = key + (uint64_t)(tid + 1) * kGamma;  // stream_at(key, i + 1)
            const uint32_t fa = smem_addr(filt + par * WB);
            sa = smem_addr(shared_bits + par * WB);
            uint32_t smin = 0xffffffffu;
            hq = head_load<KIND>(H, u32);
#pragma unroll
            for (int r = 0; r < MAXR; ++r) {
                uint32_t slo;
                const uint32_t t = lemire32_slo(mix(z0 + (uint64_t)r * dz), b0 + kT * r, slo);
                tr[r] = t;
                // the partner's head (partner p = t + (t >= u), graph.cpp:172-173): issued
                // here, consumed in P2, so its L2 latency hides behind the rest of P1
                hb[r] = head_load32<KIND>(H, (r < MAXR - 1 || in_tail) ? t + (t >= u32 ? 1u : 0u) : u32);
                if (r < MAXR - 1 || in_tail) {
                    smin = min(smin, slo);
                    tmax = max(tmax, t);
                    const uint32_t off = (t >> 3) & wmask, bit = 1u << (t & 31);
                    red_or_sh(sa + off, atom_or_sh(fa + off, bit) & bit);
                }
            }
            uint32_t first_fire = hook_thread && (u % a.force_mod) == 0 ? D / 2 : D;
            if (smin == 0u) {  // rare (2^-32 per draw): the exact pre-condition, lo < bound
#pragma unroll 1
                for (int r = 0; r < MAXR; ++r) {
                    bool fi;
                    lemire32(mix(z0 + (uint64_t)r * dz), b0 + kT * r, fi);
                    const uint32_t i = (uint32_t)tid + kT * r;
                    if (fi && (r < MAXR - 1 || in_tail) && i < first_fire) first_fire = i;
                }
            }
            fired = first_fire < D;
            if (fired) atomicMin(&s_lim, first_fire);
        }
        const bool any_fired = __syncthreads_or(fired);

        // ---- B: vertex s - 1: collided entries ----
        if (has_prev) {
            const uint32_t wc = s_wc[par ^ 1u][warp];
            const uint64_t u1 = u - stride;
            uint32_t* cb = colbits + (par ^ 1u) * W;
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const uint32_t k = lane + 32 * q;
                if (k < wc) {
                    const unsigned long long e = seg[k];
                    const uint32_t t = (uint32_t)(e >> 32), i = (uint32_t)e;
                    uint32_t h = (t * 0x85EBCA6Bu) >> (32 - kPipeHashLog2);
                    unsigned long long f;
                    while ((uint32_t)((f = *(volatile unsigned long long*)&Hprev[h]) >> 32) != t)
                        h = (h + 1) & (kPipeSlots - 1);
                    if ((uint32_t)f != i) {  // an earlier draw has the same value
                        atomicOr(&cb[i >> 5], 1u << (i & 31));
                        emit(u1, base + i);
                        ++ncol;
                    }
                    if (q == 0) h0 = h; else h1 = h;
                }
            }
        }
        __syncwarp();
        // vertex s - 2's collided bitmap (parity par): its chain was settled in C
        if ((uint32_t)tid < W) colbits[par * W + tid] = 0;

        // exact sequential replay of vertex s (rare); the filter memory (4 * WB >=
        // 4 * draws words) serves as its hash set, then is re-zeroed; its lists stay empty
        auto replay = [&](bool fired_vertex) {
            __syncthreads();
            if (tid == 0) {
                ++nrep;
                ncol += bloom_replay(key, u, a.n, base, filt, 4 * WB, xs);
                s_cc[par] = s_ovf[par] = 0;
                if (fired_vertex) {  // the head tests stop at the first fired draw
                    gpairs += s_lim;  // (k_gather_head's limit); every partner is an extra
                    s_lim = D;
                }
            }
            if (tid < kW) s_wc[par][tid] = 0;
            __syncthreads();
            for (uint32_t x = tid; x < 4 * WB; x += kT) filt[x] = 0;
        };

        if (has_v) {
            if (any_fired) {
                replay(true);
            } else {
                // ---- P2: vertex s ----
                unsigned long long* wl = glist + (par * kW + warp) * kPipeSeg;
                uint32_t wpos = 0, qn = 0;
#pragma unroll
                for (int r = 0; r < MAXR; ++r) {
                    const uint32_t t = tr[r];
                    const bool valid = r < MAXR - 1 || in_tail;
                    const uint32_t off = (t >> 3) & wmask, bit = 1u << (t & 31);
                    const bool hit = (ld_sh(sa + off) & bit) && valid;
                    const uint32_t m = __ballot_sync(kFull, hit);
                    const uint32_t pos = wpos + __popc(m & lt);
                    if (hit && pos < kPipeSeg)
                        wl[pos] = ((unsigned long long)t << 32) | ((uint32_t)tid + kT * r);
                    wpos += __popc(m);
                    // the exact head reject (sngb_head.cu); survivors -> my warp's queue
                    const bool keep = valid && !(head_q<KIND>(hq, hb[r]) > reject);
                    const uint32_t km = __ballot_sync(kFull, keep);
                    if (keep) myq[qn + __popc(km & lt)] = t + (t >= u32 ? 1u : 0u);
                    qn += __popc(km);
                }
                if (tid == 0) gpairs += D;
                if (lane == 0) {
                    s_wc[par][warp] = wpos < kPipeSeg ? wpos : kPipeSeg;
                    if (wpos > kPipeSeg) s_ovf[par] = 1;
                    if (atomicAdd(&s_ng[par], wpos) + wpos > kPipeMaxGroup) s_ovf[par] = 1;
                }
                if (tmax >= base) {  // a draw may be a chain candidate: t - base < i
                    uint32_t* cl = clist + par * kChainCap;
#pragma unroll
                    for (int r = 0; r < MAXR; ++r) {
                        const uint32_t i = (uint32_t)tid + kT * r;
                        if ((r < MAXR - 1 || in_tail) && tr[r] - base < i) {
                            const uint32_t p = atomicAdd(&s_cc[par], 1u);
                            if (p < kChainCap) cl[p] = i;
                            else s_ovf[par] = 1;
                        }
                    }
                }
                // ---- T: vertex s: my warp's survivors take the fp32 test on their rows
                // (G lanes per row, UF rows per group in flight; sngb_epstest.cuh decides) ----
                __syncwarp();
                if (qn) {
                    const uint32_t c = (uint32_t)q < RW ? (uint32_t)q : RW - 1;
                    const F4x2 qv = to_x2(ldg_row(P + u * RW + c));
                    for (uint32_t e0 = 0; e0 < qn; e0 += STEP) {
                        F4x2 rows[UF];
                        uint32_t pe[UF];
                        bool oke[UF];
#pragma unroll
                        for (int uu = 0; uu < UF; ++uu) {
                            const uint32_t e = e0 + grp + NG * uu;
                            oke[uu] = e < qn;
                            pe[uu] = myq[oke[uu] ? e : e0];
                            const uint64_t row = (oke[uu] && (uint32_t)q < RW) ? pe[uu] : u;
                            rows[uu] = ldg_row2_ef(P + row * RW + c, pol);
                        }
                        __syncwarp();  // scheduling fence: all UF loads in flight together
#pragma unroll
                        for (int uu = 0; uu < UF; ++uu) {
                            Acc2 acc;
                            diff2x2(qv, rows[uu], acc);
                            float sum = acc2_sum(acc);
#pragma unroll
                            for (int o = G / 2; o > 0; o >>= 1) sum += __shfl_xor_sync(kFull, sum, o);
                            const bool accd = decide(sum, oke[uu], leader, grp * G, g.tp, u, pe[uu], st);
                            tails += (oke[uu] && leader) ? 1u : 0u;
                            stage.push(leader && accd, edge_key(u, pe[uu], g.sink.nb), g.sink, lane);
                        }
                    }
                    __syncwarp();
                }
            }
        }
        __syncthreads();
        if (has_v && !any_fired && s_ovf[par]) {  // list overflow: exact replay
            replay(false);  // the survivors were tested: every draw took the head test
            __syncthreads();
        }
    }
    stage.flush(g.sink, lane);
    st.pairs = gpairs;
    flush_stats(st, gpairs, g.counters, lane);
    tails = warp_sum(tails);
    if (lane == 0 && tails) atomicAdd(&g.counters[C_TAIL_PAIRS], tails);
    ncol = warp_sum(ncol);
    nrep = warp_sum(nrep);
    if (lane == 0) {
        if (ncol) atomicAdd(&a.counters[C_COLLISIONS], ncol);
        if (nrep) atomicAdd(&a.counters[C_IRREGULAR], nrep);
    }
}


template <int KIND, int G, int MAXR>
__global__ void __launch_bounds__(kBloomThreads, 3)
    k_floyd_headpipe(const SamplerArgs a, const GatherArgs g, const HeadArgs hd, uint32_t grab) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ unsigned long long s_c0;
    const uint64_t rows = a.row_end - a.row_begin;
    for (;;) {  // chunks of `grab` consecutive vertices, claimed from g.work (zeroed)
        if (threadIdx.x == 0) s_c0 = atomicAdd(g.work, (unsigned long long)grab);
        __syncthreads();
        const unsigned long long c0 = s_c0;
        __syncthreads();
        if (c0 >= rows) break;
        const uint32_t nv = (uint32_t)(rows - c0 < grab ? rows - c0 : grab);
        floyd_headpipe_run<KIND, G, MAXR>(a, g, hd, smem, a.row_begin + c0, 1, nv);
    }
}
