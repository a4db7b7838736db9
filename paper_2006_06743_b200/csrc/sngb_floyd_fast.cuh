// sngb_floyd_fast.cuh -- k_floyd_fast, the Floyd bookkeeping kernel for
// draws <= 4096 (every BASELINE config).  Included by sngb_sampler.cu.
//
// Same decomposition as k_floyd (see sngb_sampler.cu), restructured after
// profiling showed k_floyd issue-bound (~340 instructions per draw: divergent
// probe loops, a block-wide classify pass over every draw, 4 barriers per
// vertex):
//
//   phase 1 (all threads, draws in registers): each draw claims its value t
//     in a shared-memory set of u32 keys (16-byte buckets, one CAS32); the
//     winner writes its index beside the key.  A draw that finds t already
//     claimed goes to a small "dup" list; a draw whose t lies in
//     [base, base + i) may equal an earlier replacement j_k and goes to a
//     small "chain" list.  Both lists are rare (about D^2/2n entries per
//     vertex).  The common path is branch-free: one 16-byte bucket load, four
//     compares, one CAS.
//   phase 2 (warp 0, only when a list is non-empty): per duplicated value the
//     minimum index is the first occurrence and every other member collides;
//     chain candidates are resolved in index order against the collided
//     bitmap; every collided draw emits its replacement j_i as an extra.
//
// Keys carry a vertex epoch in their spare high bits ((epoch << tbits) | t),
// so the set is cleared only once per 2^(32-tbits) - 2 vertices; lists and
// counters are double-buffered by vertex parity.  One barrier per vertex in
// the common case.  A list overflow or a Lemire reject pre-condition replays
// the vertex exactly and sequentially, emitting all of its partners.
#pragma once

constexpr int kFastThreads = 256;
constexpr int kListCap = 256;

// Single-thread insert-if-absent on the u32 key set (replay only; the keys
// were cleared, so every live key is a plain t).
__device__ bool set_insert_seq(uint32_t* keys, uint32_t t, uint32_t mask, uint32_t shift) {
    uint32_t b = hslot(t, shift);
    for (;;) {
        for (int k = 0; k < 4; ++k) {
            uint32_t& cur = keys[4 * b + k];
            if (cur == kEmpty) {
                cur = t;
                return true;
            }
            if (cur == t) return false;
        }
        b = (b + 1) & mask;
    }
}

size_t floyd_fast_smem_bytes(uint32_t buckets, uint32_t col_words) {
    // keys (u32) + first index (u16) per slot, collided bitmap, 2 x 3 lists
    return (size_t)buckets * 4 * (4 + 2) + (size_t)col_words * 4 + 6ull * kListCap * 4;
}

__device__ __forceinline__ void ld_bucket(const uint32_t* p, uint32_t (&e)[4]) {
    asm volatile("ld.volatile.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(e[0]), "=r"(e[1]), "=r"(e[2]), "=r"(e[3])
                 : "r"((uint32_t)__cvta_generic_to_shared(p)));
}

template <int MAXR>
__global__ void __launch_bounds__(kFastThreads) k_floyd_fast(const SamplerArgs a) {
    constexpr int kT = kFastThreads;
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t NB = a.hash_mask + 1;  // buckets of 4 keys
    const uint32_t W = a.col_words;       // words of a draws-bit bitmap
    uint32_t* keys = reinterpret_cast<uint32_t*>(smem);              // 4 NB
    uint16_t* idxs = reinterpret_cast<uint16_t*>(keys + 4 * NB);     // 4 NB
    uint32_t* colbits = reinterpret_cast<uint32_t*>(idxs + 4 * NB);  // W
    uint32_t* lists = colbits + W;  // [parity][dup_slot | dup_idx | chain_idx][kListCap]
    __shared__ uint32_t s_cnt[2][2];  // [parity][dup, chain]

    const int tid = threadIdx.x, lane = tid & 31, wib = tid >> 5;
    const EdgeSink xs{a.extras, a.extras_capacity, &a.counters[C_EXTRA_CURSOR], 0};
    const uint32_t D = a.draws, base = a.base, mask = a.hash_mask, shift = a.hash_shift;
    const uint32_t tbits = a.key_bits;  // < 30 (launcher)
    const uint32_t hi_mask = ~((1u << tbits) - 1u);
    const uint32_t ep_max = (0xffffffffu >> tbits) - 1u;
    unsigned long long ncol = 0, nrep = 0;
    uint32_t ep = ep_max;  // forces a clear before the first vertex
    uint32_t par = 0;

    for (uint32_t s = tid; s < W; s += kT) colbits[s] = 0;
    if (tid < 4) (&s_cnt[0][0])[tid] = 0;

    auto emit = [&](uint64_t u, uint32_t e) {  // extra pair (u, partner of value e)
        const unsigned long long s2 = atomicAdd(xs.cursor, 1ull);
        if (s2 < xs.capacity)
            xs.keys[s2] = ((unsigned long long)u << 32) | (e + (e >= (uint32_t)u ? 1u : 0u));
    };

    for (uint64_t u = a.row_begin + blockIdx.x; u < a.row_end; u += gridDim.x) {
        if (ep == ep_max) {  // (re)initialise the key set
            ep = 0;
            for (uint32_t s = tid; s < 4 * NB; s += kT) keys[s] = kEmpty;
            __syncthreads();
        } else {
            ++ep;
        }
        par ^= 1u;
        uint32_t* cnt = s_cnt[par];
        uint32_t* dup_slot = lists + par * 3 * kListCap;
        uint32_t* dup_idx = dup_slot + kListCap;
        uint32_t* chain_idx = dup_idx + kListCap;
        const uint32_t epk = ep << tbits;
        const uint64_t key = vertex_key(a.seed_mixed, u);

        // ---- phase 1 ----
        uint32_t tr[MAXR];
        bool fired = false;
#pragma unroll
        for (int r = 0; r < MAXR; ++r) {
            const uint32_t i = tid + kT * r;
            bool f = false;
            tr[r] = (i < D) ? lemire32(stream_at(key, (uint64_t)i + 1), base + i + 1, f) : 0u;
            fired |= (i < D) && (f || test_fire(a.force_mod, u, i, D));
        }
#pragma unroll
        for (int r = 0; r < MAXR; ++r) {
            const uint32_t i = tid + kT * r;
            if (i < D) {
                const uint32_t t = tr[r];
                const uint32_t want = epk | t;
                uint32_t b = hslot(t, shift);
                // in-bucket start slot from a second hash: different values of one
                // bucket race for different slots (same value -> same slot order)
                const int k0 = (int)((t * 0x85EBCA6Bu) >> 30);
                for (;;) {
                    uint32_t e[4];
                    ld_bucket(keys + 4 * b, e);
                    uint32_t eq = 0, fr = 0;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        eq |= (e[k] == want ? 1u : 0u) << k;
                        fr |= ((e[k] & hi_mask) != epk ? 1u : 0u) << k;  // stale or empty
                    }
                    if (eq) {  // t already claimed by another draw of this vertex
                        const uint32_t p = atomicAdd(&cnt[0], 1u);
                        if (p < kListCap) {
                            dup_slot[p] = 4 * b + (__ffs(eq) - 1);
                            dup_idx[p] = i;
                        }
                        break;
                    }
                    if (fr) {
                        const uint32_t rot = ((fr >> k0) | (fr << (4 - k0))) & 0xfu;
                        const int k = (__ffs(rot) - 1 + k0) & 3;
                        const uint32_t ek = k == 0 ? e[0] : k == 1 ? e[1] : k == 2 ? e[2] : e[3];
                        if (atomicCAS(&keys[4 * b + k], ek, want) == ek) {
                            idxs[4 * b + k] = (uint16_t)i;
                            break;
                        }
                        continue;  // lost a race: re-read the same bucket
                    }
                    b = (b + 1) & mask;  // bucket full of other live values
                }
                if (t >= base && t - base < i) {
                    const uint32_t p = atomicAdd(&cnt[1], 1u);
                    if (p < kListCap) chain_idx[p] = i;
                }
            }
        }
        const bool anyfire = __syncthreads_or(fired);
        const uint32_t ndup = cnt[0], nchain = cnt[1];
        if (anyfire || ndup > kListCap || nchain > kListCap) {
            // exact sequential replay of graph.cpp:163-174; all partners -> extras
            for (uint32_t s = tid; s < 4 * NB; s += kT) keys[s] = kEmpty;
            __syncthreads();
            if (tid == 0) {
                ++nrep;
                SeqStream st{key, 0};
                const uint64_t pool = a.n - 1;
                for (uint64_t jj = base; jj < pool; ++jj) {
                    const uint32_t t = (uint32_t)st.next_below(jj + 1);
                    uint32_t e = t;
                    if (!set_insert_seq(keys, t, mask, shift)) {
                        set_insert_seq(keys, (uint32_t)jj, mask, shift);
                        e = (uint32_t)jj;
                    }
                    emit(u, e);
                }
                cnt[0] = cnt[1] = 0;
            }
            ep = ep_max;  // the replay left plain keys: clear before the next vertex
            __syncthreads();
            continue;
        }
        if (ndup == 0 && nchain == 0) continue;  // (block-uniform)

        // ---- phase 2 (warp 0) ----
        if (wib == 0) {
            // (a) duplicate groups: first = min(claimant, finders); the others
            //     collide.  The finder holding `first` reports the claimant.
            for (uint32_t p = lane; p < ndup; p += 32) {
                const uint32_t s = dup_slot[p], i = dup_idx[p];
                uint32_t first = idxs[s];
                for (uint32_t q = 0; q < ndup; ++q)
                    if (dup_slot[q] == s && dup_idx[q] < first) first = dup_idx[q];
                const uint32_t c = (i == first) ? (uint32_t)idxs[s] : i;
                atomicOr(&colbits[c >> 5], 1u << (c & 31));
                emit(u, base + c);
                ++ncol;
            }
            __syncwarp();
            // (b) chains, in index order (lane 0; the list is tiny)
            if (lane == 0 && nchain) {
                for (uint32_t x = 1; x < nchain; ++x) {  // insertion sort
                    const uint32_t v = chain_idx[x];
                    uint32_t y = x;
                    while (y > 0 && chain_idx[y - 1] > v) {
                        chain_idx[y] = chain_idx[y - 1];
                        --y;
                    }
                    chain_idx[y] = v;
                }
                for (uint32_t x = 0; x < nchain; ++x) {
                    const uint32_t i = chain_idx[x];
                    if ((colbits[i >> 5] >> (i & 31)) & 1u) continue;  // already collided
                    bool f;
                    const uint32_t k =
                        lemire32(stream_at(key, (uint64_t)i + 1), base + i + 1, f) - base;
                    if ((colbits[k >> 5] >> (k & 31)) & 1u) {
                        colbits[i >> 5] |= 1u << (i & 31);
                        emit(u, base + i);
                        ++ncol;
                    }
                }
            }
            __syncwarp();
            // (c) clear exactly the words that may hold set bits
            for (uint32_t p = lane; p < ndup + nchain; p += 32) {
                const uint32_t i = p < ndup ? dup_idx[p] : chain_idx[p - ndup];
                colbits[i >> 5] = 0;
                if (p < ndup) colbits[idxs[dup_slot[p]] >> 5] = 0;
            }
            __syncwarp();
            if (lane == 0) cnt[0] = cnt[1] = 0;
        }
        __syncthreads();
    }
    ncol = warp_sum(ncol);  // phase 2 counts on every lane of warp 0
    if (lane == 0) {
        if (ncol) atomicAdd(&a.counters[C_COLLISIONS], ncol);
        if (nrep && wib == 0) atomicAdd(&a.counters[C_IRREGULAR], nrep);
    }
}
