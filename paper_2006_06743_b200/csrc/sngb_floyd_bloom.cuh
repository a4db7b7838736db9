// sngb_floyd_bloom.cuh -- k_floyd_bloom, Floyd bookkeeping for large n and
// draws <= 4096 (cfg2-cfg5).  Included by sngb_sampler.cu.
//
// k_floyd_fast claims every draw value in a CAS-built key set; profiling
// showed it issue/latency bound on divergent claim loops (CAS races, probes)
// and barrier waits.  For large n a vertex's draws are almost all distinct
// (about D^2/2n duplicates), so exact membership is only needed for the few
// draws that can collide.  Per vertex (one block, draws in registers):
//
//   P1  every draw ORs bit h(t) into a 2^B-bit filter (atomicOr never fails,
//       no loops); a draw that finds its bit already set also marks it in a
//       second "shared bit" filter.  Draws with t in [base, base + i) (may
//       equal an earlier replacement j_k) go to a small chain list.
//   P2  every draw whose bit is shared (true duplicates + ~D/2^B false
//       positives) appends (t, i) to a small group list.
//   P3  warp 0: a group-list draw collides iff another entry has the same t and
//       a smaller index (first occurrence = minimum index); chain candidates
//       are then resolved in index order against the collided bitmap.  Every
//       collided draw emits its replacement j_i as an extra.
//
// Filters and lists are double-buffered by vertex parity: while a vertex runs
// on parity p, the workers clear parity p^1's filters with 16-byte stores (the
// barriers of vertex u separate that clear from its reuse by vertex u+1), so
// there are two barriers per vertex.  A list overflow or a Lemire reject
// pre-condition replays the vertex exactly and sequentially.
#pragma once


constexpr int kBloomThreads = 256;
constexpr int kGroupCap = 512;
constexpr int kHashLog2 = 10;
constexpr int kHashSlots = 1 << kHashLog2;
constexpr int kChainCap = 256;

struct BloomGeom {
    uint32_t bits_log2;   // B
    uint32_t words;       // 2^B / 32
    uint32_t col_words;   // draws-bit bitmap words
};

inline BloomGeom bloom_geometry(uint32_t draws) {
    uint32_t lg = 0;
    while ((1u << lg) < draws) ++lg;
    BloomGeom g;
    g.bits_log2 = lg + 4 < 12 ? 12 : lg + 4;  // false-positive rate ~ draws / 2^B <= 1/16
    if (g.bits_log2 > 17) g.bits_log2 = 17;
    g.words = (1u << g.bits_log2) / 32;
    g.col_words = ((draws + 31) / 32 + 3) & ~3u;
    return g;
}

inline size_t bloom_smem_bytes(const BloomGeom& g) {
    return 4ull * g.words * 4                    // filter + shared-bit filter, x2 parity
           + (size_t)g.col_words * 4             // collided bitmap
           + 2ull * kGroupCap * 8                // group lists (t << 32 | i), x2 parity
           + 2ull * kChainCap * 4                // chain lists, x2 parity
           + (size_t)kHashSlots * 8;             // warp 0's first-occurrence hash
}

// Exact sequential replay (graph.cpp:163-174) with a u32 open-addressing set
// in `tab` (cap slots, power of two); every partner becomes an extra.  Returns
// the vertex's Floyd collisions (draws replaced by j), so the collision count
// does not depend on which vertices a kernel replays.
__device__ unsigned long long bloom_replay(uint64_t key, uint64_t u, uint64_t n, uint32_t base,
                                           uint32_t* tab, uint32_t cap, const EdgeSink& xs) {
    unsigned long long ncol = 0;
    for (uint32_t s = 0; s < cap; ++s) tab[s] = kEmpty;
    const uint32_t mask = cap - 1;
    auto insert = [&](uint32_t t) -> bool {
        uint32_t h = (t * 0x9E3779B1u) & mask;
        for (;;) {
            if (tab[h] == kEmpty) {
                tab[h] = t;
                return true;
            }
            if (tab[h] == t) return false;
            h = (h + 1) & mask;
        }
    };
    SeqStream st{key, 0};
    for (uint64_t jj = base; jj < n - 1; ++jj) {
        const uint32_t t = (uint32_t)st.next_below(jj + 1);
        uint32_t e = t;
        if (!insert(t)) {
            insert((uint32_t)jj);
            e = (uint32_t)jj;
            ++ncol;
        }
        const unsigned long long s2 = atomicAdd(xs.cursor, 1ull);
        if (s2 < xs.capacity)
            xs.keys[s2] = ((unsigned long long)u << 32) | (e + (e >= (uint32_t)u ? 1u : 0u));
    }
    return ncol;
}

// Named barriers (bar.sync/arrive with a thread count): the 8 worker warps
// synchronise among themselves and hand each vertex's lists to a resolver warp
// producer/consumer style, so the resolver's work never stalls the workers.
__device__ __forceinline__ void bar_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int count) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ bool bar_or(int id, int count, bool pred) {
    unsigned r;
    asm volatile(
        "{\n\t.reg .pred p, q;\n\tsetp.ne.u32 p, %1, 0;\n\t"
        "bar.red.or.pred q, %2, %3, p;\n\tselp.u32 %0, 1, 0, q;\n\t}"
        : "=r"(r)
        : "r"((unsigned)pred), "r"(id), "r"(count)
        : "memory");
    return r != 0;
}

// Shared-memory access by 32-bit address: the base is converted once per
// vertex instead of per draw (ptxas otherwise re-derives it under register
// pressure), and the shared-bit mark is a predicated reduction (no branch).
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t atom_or_sh(uint32_t addr, uint32_t v) {
    uint32_t old;
    asm volatile("atom.shared.or.b32 %0, [%1], %2;" : "=r"(old) : "r"(addr), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ void red_or_sh_if(uint32_t addr, uint32_t v, uint32_t pred) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p red.shared.or.b32 [%0], %1;\n\t}"
        ::"r"(addr), "r"(v), "r"(pred) : "memory");
}
__device__ __forceinline__ void st_sh(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_sh(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}

// shared-memory access at a compile-time byte offset from a 32-bit shared address
template <uint32_t OFF>
__device__ __forceinline__ void pipe_red_or_off(uint32_t addr, uint32_t v) {
    asm volatile("red.shared.or.b32 [%0+%2], %1;" ::"r"(addr), "r"(v), "n"(OFF) : "memory");
}
template <uint32_t OFF>
__device__ __forceinline__ uint32_t pipe_ld_off(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1+%2];" : "=r"(v) : "r"(addr), "n"(OFF) : "memory");
    return v;
}

constexpr int kBarWorkers = 1;  // 256 worker threads
constexpr int kBarReady = 2;    // + parity: lists of a vertex are complete (288)
constexpr int kBarFree = 4;     // + parity: resolver is done with that parity (288)
constexpr int kBloomBlock = kBloomThreads + 32;

// P3 of one vertex (the resolver warp of k_floyd_bloom / k_floyd_lean /
// k_floyd_head): the vertex's group list (every draw on a bloom bit hit by >= 2
// draws) and chain list (parity `par`) become collided draws, whose
// replacements are emitted as extras; the lists are left empty.
__device__ __forceinline__ void bloom_resolve_vertex(const SamplerArgs& a, uint64_t u, uint32_t par,
                                                     unsigned long long* glist, uint32_t* clist,
                                                     uint32_t (*s_cnt)[2], uint32_t* colbits,
                                                     unsigned long long* htab, const EdgeSink& xs,
                                                     int lane, unsigned long long& ncol) {
    const uint32_t base = a.base;
    auto emit = [&](uint64_t u, uint32_t e) {  // extra pair (u, partner of value e)
        const unsigned long long s2 = atomicAdd(xs.cursor, 1ull);
        if (s2 < xs.capacity)
            xs.keys[s2] = ((unsigned long long)u << 32) | (e + (e >= (uint32_t)u ? 1u : 0u));
    };
    unsigned long long* gl = glist + par * kGroupCap;
    uint32_t* cl = clist + par * kChainCap;
    uint32_t* cnt = s_cnt[par];
    const uint32_t ng = cnt[0], nc = cnt[1];
    if (ng || nc) {
        // first occurrence per value: (t, min index) in a small hash
        for (uint32_t p = lane; p < ng; p += 32) {
            const unsigned long long e = gl[p];
            const uint32_t t = (uint32_t)(e >> 32);
            uint32_t h = (t * 0x85EBCA6Bu) >> (32 - kHashLog2);
            for (;;) {
                const unsigned long long old = atomicCAS(&htab[h], ~0ull, e);
                if (old == ~0ull) break;
                if ((uint32_t)(old >> 32) == t) {
                    atomicMin(&htab[h], e);
                    break;
                }
                h = (h + 1) & (kHashSlots - 1);
            }
        }
        __syncwarp();
        for (uint32_t p = lane; p < ng; p += 32) {
            const unsigned long long e = gl[p];
            const uint32_t t = (uint32_t)(e >> 32), i = (uint32_t)e;
            uint32_t h = (t * 0x85EBCA6Bu) >> (32 - kHashLog2);
            while ((uint32_t)(htab[h] >> 32) != t) h = (h + 1) & (kHashSlots - 1);
            if ((uint32_t)htab[h] != i) {  // an earlier draw has the same value
                atomicOr(&colbits[i >> 5], 1u << (i & 31));
                emit(u, base + i);
                ++ncol;
            }
        }
        __syncwarp();  // all lookups done: reset the whole (8 KB) hash
        for (uint32_t s2 = lane; s2 < kHashSlots; s2 += 32) htab[s2] = ~0ull;
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
                const uint32_t k =
                    lemire32(stream_at(key, (uint64_t)i + 1), base + i + 1, fi) - base;
                if ((colbits[k >> 5] >> (k & 31)) & 1u) {
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
}

// P3 loop of the resolver warp, one vertex behind the workers.
__device__ __forceinline__ void bloom_resolver(const SamplerArgs& a, unsigned long long* glist,
                                               uint32_t* clist, uint32_t (*s_cnt)[2],
                                               uint32_t* colbits, unsigned long long* htab,
                                               const EdgeSink& xs, int lane,
                                               unsigned long long& ncol) {
    uint32_t par = 0;
    for (uint64_t u = a.row_begin + blockIdx.x; u < a.row_end; u += gridDim.x) {
        par ^= 1u;
        bar_sync(kBarReady + par, kBloomBlock);
        bloom_resolve_vertex(a, u, par, glist, clist, s_cnt, colbits, htab, xs, lane, ncol);
        bar_arrive(kBarFree + par, kBloomBlock);
    }
}


template <int MAXR>
// Four resident blocks per SM (<= 56 registers, no spills): the kernel is
// latency-bound on its shared-memory filter and barriers, and the fourth block
// beats the heuristic's 72 registers / 3 blocks (cfg5 352 -> 321 ms, cfg4
// 53.4 -> 51.4 ms, cfg3 5.26 -> 5.19 ms; 3 blocks measured no better).
#ifndef SNGB_BLOOM_MINB
#define SNGB_BLOOM_MINB 4
#endif
__global__ void __launch_bounds__(kBloomBlock, SNGB_BLOOM_MINB) k_floyd_bloom(const SamplerArgs a) {
    constexpr int kT = kBloomThreads;
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
        reinterpret_cast<unsigned long long*>(clist + 2 * kChainCap);  // [kHashSlots]
    __shared__ uint32_t s_cnt[2][2];  // [parity][group, chain]

    const int tid = threadIdx.x, lane = tid & 31;
    const bool resolver = tid >= kT;
    const EdgeSink xs{a.extras, a.extras_capacity, &a.counters[C_EXTRA_CURSOR], 0};
    const uint32_t D = a.draws, base = a.base;
    unsigned long long ncol = 0, nrep = 0;

    for (uint32_t s = tid; s < 4 * WB + W; s += kBloomBlock) filt[s] = 0;
    for (uint32_t s = tid; s < kHashSlots; s += kBloomBlock) htab[s] = ~0ull;
    if (tid < 4) (&s_cnt[0][0])[tid] = 0;
    __syncthreads();

    if (resolver) {
        bloom_resolver(a, glist, clist, s_cnt, colbits, htab, xs, lane, ncol);
    } else {
        // ---- workers: P1 filter bits + chain candidates, P2 group list ----
        uint32_t par = 0, vcount = 0;
        const uint64_t dz = (uint64_t)kT * kGamma;  // counter step between a thread's draws
        for (uint64_t u = a.row_begin + blockIdx.x; u < a.row_end; u += gridDim.x) {
            par ^= 1u;
            if (++vcount > 2) bar_sync(kBarFree + par, kBloomBlock);  // parity par reusable
            uint32_t* f = filt + par * WB;
            uint32_t* sb = shared_bits + par * WB;
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
            const uint64_t key = vertex_key(a.seed_mixed, u);
            uint64_t z = key + (uint64_t)(tid + 1) * kGamma;  // stream_at(key, i + 1), i = tid
            const uint32_t fa = smem_addr(f), sa = smem_addr(sb);
            const uint32_t nfull = D / kT;  // slots in which every thread has a draw
            // test hook (see test_fire): resolved once per vertex
            const uint32_t forced_i =
                (a.force_mod != 0 && (u % a.force_mod) == 0) ? D / 2 : 0xffffffffu;

            uint32_t tr[MAXR];
            uint32_t chain = 0;  // bit r: draw r may equal an earlier replacement j_k
            bool fired = false;
            auto p1 = [&](int r, uint32_t i, uint64_t zz) {
                bool fi;
                const uint32_t t = lemire32(mix(zz), base + i + 1, fi);
                fired |= fi | (i == forced_i);
                tr[r] = t;
                const uint32_t h = (t * 0x9E3779B1u) >> shift;
                const uint32_t off = (h >> 5) * 4u, bit = 1u << (h & 31);
                red_or_sh_if(sa + off, bit, atom_or_sh(fa + off, bit) & bit);
                // t in [base, base + i): t <= base + i always, so one unsigned compare
                chain |= (t - base < i ? 1u : 0u) << r;
            };
#pragma unroll
            for (int r = 0; r < MAXR; ++r, z += dz) {
                const uint32_t i = tid + kT * r;
                if ((uint32_t)r < nfull || i < D) p1(r, i, z);
            }
            if (chain) {  // rare (about draws/n per draw)
#pragma unroll
                for (int r = 0; r < MAXR; ++r)
                    if ((chain >> r) & 1u) {
                        const uint32_t p = atomicAdd(&cnt[1], 1u);
                        if (p < kChainCap) cl[p] = tid + kT * r;
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
            if (bar_or(kBarWorkers, kT, fired)) {
                replay();
                continue;
            }
            // P2: draws whose bit is shared go to the group list (per-lane pushes:
            // a warp-aggregated ballot variant measured 11 % slower on cfg4)
#pragma unroll
            for (int r = 0; r < MAXR; ++r) {
                const uint32_t i = tid + kT * r;
                if ((uint32_t)r * kT >= D) break;  // uniform: no thread has slot r
                bool hit = false;
                if ((uint32_t)r < nfull || i < D) {
                    const uint32_t h = (tr[r] * 0x9E3779B1u) >> shift;
                    hit = (ld_sh(sa + (h >> 5) * 4u) >> (h & 31)) & 1u;
                }
                if (hit) {
                    const uint32_t p = atomicAdd(&cnt[0], 1u);
                    if (p < kGroupCap) gl[p] = ((unsigned long long)tr[r] << 32) | i;
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

// The exact sequential replay (bloom_replay: graph.cpp:163-174 with true Stream
// semantics) of the vertices k_floyd_warp / k_sample_head listed; every partner is an extra.
__global__ void __launch_bounds__(32) k_replay_list(const SamplerArgs a, const uint32_t* list,
                                                    uint32_t cap) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t* tab = reinterpret_cast<uint32_t*>(smem);
    const EdgeSink xs{a.extras, a.extras_capacity, &a.counters[C_EXTRA_CURSOR], 0};
    const unsigned long long cnt = a.counters[C_IRR_CURSOR];
    unsigned long long nrep = 0, ncol = 0;
    for (unsigned long long x = blockIdx.x; x < cnt; x += gridDim.x) {
        if (threadIdx.x == 0) {
            const uint64_t u = list[x];
            ncol += bloom_replay(vertex_key(a.seed_mixed, u), u, a.n, a.base, tab, cap, xs);
            ++nrep;
        }
    }
    if (threadIdx.x == 0 && nrep) atomicAdd(&a.counters[C_IRREGULAR], nrep);
    if (threadIdx.x == 0 && ncol) atomicAdd(&a.counters[C_COLLISIONS], ncol);
}
