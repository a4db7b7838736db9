// sngb_floyd_lean.cuh -- k_floyd_lean, the Floyd bookkeeping of k_floyd_bloom
// with an instruction diet on the workers (large n, 1024 < draws <= 4096: cfg4,
// cfg5).  Included by sngb_sampler.cu after sngb_floyd_bloom.cuh, whose shared-
// memory layout, barriers, resolver warp (bloom_resolver) and exact replay it
// reuses unchanged.
//
// k_floyd_bloom spends ~100 SASS instructions per draw (ncu,
// profiles/r02_ncu_floyd_cfg5.md: 3.14 warp-instructions per draw) where the
// draw itself (rng.hpp:26 mix + rng.hpp:35-48 Lemire) is ~25: every draw slot
// carried its own validity test (BSSY/BSYNC/BRA), a multiplicative hash, an
// exact Lemire pre-condition and chain test with their selects, and the test
// hook's compare.  Here, per draw:
//
//   * the launch picks MAXR = ceil(draws / 256), so slots r < MAXR - 1 are full
//     for every thread at compile time: no per-draw validity test; only the
//     last slot is predicated;
//   * the filter bit is t's own low B bits (t is uniform on [0, j+1), so its
//     low bits are as good a hash as a multiply);
//   * the Lemire reject pre-condition (rng.hpp:43, lo < bound) needs the low
//     word of x*b's high half to be 0: a running minimum of that word (one
//     instruction) flags the rare thread that must redo the exact test;
//   * chain candidates (t_i in [base, base + i), graph.cpp:168 can then meet an
//     earlier replacement j_k) need t >= base: a running maximum of t flags the
//     rare thread that must look, and only it re-tests its draws exactly;
//   * the test hook is resolved once per vertex and thread.
// P2 (the group list) and P3 (the resolver warp) are k_floyd_bloom's.
#pragma once

__device__ __forceinline__ void red_or_sh(uint32_t addr, uint32_t v) {
    asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

template <int MAXR>
__global__ void __launch_bounds__(kBloomBlock, SNGB_BLOOM_MINB) k_floyd_lean(const SamplerArgs a) {
    constexpr int kT = kBloomThreads;
    extern __shared__ __align__(16) unsigned char smem[];
    // filter words (2^B / 32): bloom_geometry gives B = 15 up to 2048 draws (MAXR <= 8) and
    // B = 16 above -- a compile-time constant, so a draw's shared-bit word is its filter
    // word plus an immediate offset (as k_floyd_pipe)
    constexpr uint32_t WB = MAXR >= 9 ? 2048u : 1024u;
    constexpr uint32_t kShOff = 2 * WB * 4;  // bytes from filt[par] to shared_bits[par]
    const uint32_t W = a.col_words;
    uint32_t* filt = reinterpret_cast<uint32_t*>(smem);          // [2][WB]
    uint32_t* shared_bits = filt + 2 * WB;                         // [2][WB]
    uint32_t* colbits = shared_bits + 2 * WB;                      // [W]
    unsigned long long* glist =
        reinterpret_cast<unsigned long long*>(colbits + W);       // [2][kGroupCap]
    uint32_t* clist = reinterpret_cast<uint32_t*>(glist + 2 * kGroupCap);  // [2][kChainCap]
    unsigned long long* htab =
        reinterpret_cast<unsigned long long*>(clist + 2 * kChainCap);  // [kHashSlots]
    __shared__ uint32_t s_cnt[2][2];  // [parity][group, chain]
    __shared__ unsigned long long s_key;  // the next vertex's stream key (worker thread 0 computes it)

    const int tid = threadIdx.x, lane = tid & 31;
    const bool resolver = tid >= kT;
    const EdgeSink xs{a.extras, a.extras_capacity, &a.counters[C_EXTRA_CURSOR], 0};
    const uint32_t D = a.draws, base = a.base;
    unsigned long long ncol = 0, nrep = 0;

    for (uint32_t s = tid; s < 4 * WB + W; s += kBloomBlock) filt[s] = 0;
    for (uint32_t s = tid; s < kHashSlots; s += kBloomBlock) htab[s] = ~0ull;
    if (tid < 4) (&s_cnt[0][0])[tid] = 0;
    if (tid == 0) s_key = vertex_key(a.seed_mixed, a.row_begin + blockIdx.x);
    __syncthreads();

    if (resolver) {
        bloom_resolver(a, glist, clist, s_cnt, colbits, htab, xs, lane, ncol);
    } else {
        uint32_t par = 0, vcount = 0;
        const uint64_t dz = (uint64_t)kT * kGamma;  // counter step between a thread's draws
        // MAXR = ceil(D / kT): slots r < MAXR - 1 are full, the last one holds
        // D - kT (MAXR - 1) draws
        const bool in_tail = (uint32_t)tid < D - kT * (MAXR - 1);
        constexpr uint32_t wmask = (WB - 1) << 2;   // byte offset of t's filter word
        const uint32_t b0 = base + (uint32_t)tid + 1;  // Lemire bound of slot 0: j + 1
        // test hook (see test_fire): the thread and slot of draw D / 2
        const bool hook_thread = a.force_mod != 0 && (D / 2) % kT == (uint32_t)tid;
        for (uint64_t u = a.row_begin + blockIdx.x; u < a.row_end; u += gridDim.x) {
            par ^= 1u;
            if (++vcount > 2) bar_sync(kBarFree + par, kBloomBlock);  // parity par reusable
            unsigned long long* gl = glist + par * kGroupCap;
            uint32_t* cl = clist + par * kChainCap;
            uint32_t* cnt = s_cnt[par];
            {  // clear the other parity's filters (last used by vertex u - 1)
                uint4* fo = reinterpret_cast<uint4*>(filt + (par ^ 1u) * WB);
                uint4* so = reinterpret_cast<uint4*>(shared_bits + (par ^ 1u) * WB);
                const uint4 z4 = make_uint4(0, 0, 0, 0);
                for (uint32_t w = tid; w < WB / 4; w += kT) {
                    fo[w] = z4;
                    so[w] = z4;
                }
            }
            const uint64_t key = s_key;  // vertex_key(a.seed_mixed, u), written one vertex ahead
            const uint64_t z0 = key + (uint64_t)(tid + 1) * kGamma;  // stream_at(key, i + 1)
            const uint32_t fa = smem_addr(filt + par * WB);

            uint32_t tr[MAXR];
            uint32_t smin = 0xffffffffu, tmax = 0;
            auto filter = [&](uint32_t t) {
                const uint32_t off = (t >> 3) & wmask, bit = 1u << (t & 31);
                // the shared-bit mark is an unconditional OR of (old & bit): a
                // predicated red compiles to a branch + reconvergence (3 issue slots)
                pipe_red_or_off<kShOff>(fa + off, atom_or_sh(fa + off, bit) & bit);
            };
#pragma unroll
            for (int r = 0; r < MAXR; ++r) {
                uint32_t slo;
                const uint32_t t = lemire32_slo(mix(z0 + (uint64_t)r * dz), b0 + kT * r, slo);
                tr[r] = t;
                if (r < MAXR - 1 || in_tail) {
                    smin = min(smin, slo);
                    tmax = max(tmax, t);
                    filter(t);
                }
            }
            // exact tests for the rare flagged threads
            bool fired = hook_thread && (u % a.force_mod) == 0;
            if (smin == 0u) {  // rare (2^-32 per draw): the exact pre-condition, lo < bound
#pragma unroll 1
                for (int r = 0; r < MAXR; ++r) {
                    bool fi;
                    lemire32(mix(z0 + (uint64_t)r * dz), b0 + kT * r, fi);
                    fired |= fi && (r < MAXR - 1 || in_tail);
                }
            }
            if (tmax >= base) {  // a draw may be a chain candidate: t - base < i
#pragma unroll
                for (int r = 0; r < MAXR; ++r) {
                    const uint32_t i = (uint32_t)tid + kT * r;
                    if ((r < MAXR - 1 || in_tail) && tr[r] - base < i) {
                        const uint32_t p = atomicAdd(&cnt[1], 1u);
                        if (p < kChainCap) cl[p] = i;
                    }
                }
            }
            // exact sequential replay of one vertex (rare); the filter memory
            // (4 * WB >= 4 * draws words) serves as its hash set, then is re-zeroed;
            // the resolver then sees empty lists for this vertex
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
                bar_arrive(kBarReady + par, kBloomBlock);
            };
            const bool any_fired = bar_or(kBarWorkers, kT, fired);
            // every worker has read s_key: the next vertex's key (read after this vertex's
            // last worker barrier)
            if (tid == 0) s_key = vertex_key(a.seed_mixed, u + gridDim.x);
            if (any_fired) {
                replay();
                continue;
            }
            // P2: draws whose bit is shared go to the group list
#pragma unroll
            for (int r = 0; r < MAXR; ++r) {
                const uint32_t t = tr[r];
                const uint32_t off = (t >> 3) & wmask, bit = 1u << (t & 31);
                const bool hit = (pipe_ld_off<kShOff>(fa + off) & bit) && (r < MAXR - 1 || in_tail);
                if (hit) {
                    const uint32_t p = atomicAdd(&cnt[0], 1u);
                    if (p < kGroupCap) gl[p] = ((unsigned long long)t << 32) | ((uint32_t)tid + kT * r);
                }
            }
            bar_sync(kBarWorkers, kT);
            if (cnt[0] > kGroupCap || cnt[1] > kChainCap) {  // list overflow: exact replay
                replay();
                continue;
            }
            bar_arrive(kBarReady + par, kBloomBlock);
        }
    }
    ncol = warp_sum(ncol);
    if (lane == 0) {
        if (ncol) atomicAdd(&a.counters[C_COLLISIONS], ncol);
        if (nrep) atomicAdd(&a.counters[C_IRREGULAR], nrep);
    }
}
