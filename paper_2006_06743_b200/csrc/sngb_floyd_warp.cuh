// sngb_floyd_warp.cuh -- k_floyd_warp: the Floyd bookkeeping for large n and
// draws <= 4096 (cfg3-cfg5), one warp per vertex.  Included by sngb_sampler.cu
// after sngb_floyd_bloom.cuh (shared-memory helpers, bloom_geometry, replay).
//
// k_floyd_bloom (a block of 8 workers + a resolver warp per vertex) spends
// ~100 SASS instructions per draw and stalls on its per-vertex barriers
// (ncu: profiles/r02_ncu_floyd_cfg5.md: 3.14 warp-instructions per draw, 68 %
// issue, barrier 1.8 stalls per instruction).  Here each warp owns a vertex,
// keeps the draws' 16-bit filter hashes in its shared memory and never waits
// for another warp:
//
//   P1  draw i (lane i mod 32, R slots per step, full steps branch-free):
//       t_i = Lemire(mix(key + (i+1) gamma)) (rng.hpp:26,35-48); the running
//       minimum of Lemire's low word flags a possible reject pre-condition
//       (rng.hpp:43) -- the exact test then finds the first fired draw and the
//       vertex goes to the sequential replay; h_i = hash(t_i) -> HS[i]; OR bit
//       h_i into a 2^B-bit filter F: a draw finding its bit set appends h_i to
//       its lane's second-comer list SL; t_i in [base, base + i) (it may equal
//       an earlier replacement j_k) appends i to its lane's chain list.
//   P2  F := the bits in SL, exactly the bits hit by >= 2 draws; scan HS: the
//       draws on such a bit -> the lane's group list (SL's slots).
//   R   the group draws' values (regenerated, ~6 % of the draws) in a small
//       hash in F's memory keyed by t with the minimum index: a draw whose
//       value has a smaller index collides (graph.cpp:168-169), its
//       replacement j_i = base + i is emitted as an extra pair; then the chain
//       candidates in index order against the collided bitmap (HS's memory).
// A fired draw or a list overflow lists the vertex for k_replay_list (exact
// sequential Stream semantics, every partner an extra).  Same extras and
// counters as k_floyd_bloom (tests/test_gpu_parity.py -k "floyd or head").
#pragma once

#ifdef SNGB_FW_DEBUG
#define FW_CHECK(cond, what)                                                               \
    do {                                                                                   \
        if (!(cond)) {                                                                     \
            printf("k_floyd_warp check failed: %s (block %d lane %d)\n", what, blockIdx.x, \
                   (int)(threadIdx.x & 31));                                               \
            __trap();                                                                      \
        }                                                                                  \
    } while (0)
#else
#define FW_CHECK(cond, what) \
    do {                     \
    } while (0)
#endif

constexpr int kFwSLL = 32;  // per lane: second comers (P1, mean D^2/2^(B+1)/32 = 3.8 at D = 4000),
                            // then group draws (P2, mean D^2/2^B/32 = 7.6)
constexpr int kFwCLL = 16;  // chain candidates per lane (mean D^2/2n/32: 0.02 on cfg4 / cfg5)

struct FwGeom {
    uint32_t B, FW, CW, hs_words;
    __host__ __device__ uint32_t warp_bytes() const {
        return FW * 4 + hs_words * 4 + 32 * kFwSLL * 2 + 32 * kFwCLL * 2;
    }
};

inline FwGeom fw_geometry(uint32_t draws) {
    const BloomGeom bg = bloom_geometry(draws);
    FwGeom g;
    g.B = bg.bits_log2;  // <= 16 for draws <= 4096: hashes fit 16 bits
    g.FW = bg.words;
    g.CW = bg.col_words;
    g.hs_words = ((draws + 255) / 256) * 128;  // 16-byte rows of 8 hashes
    if (g.hs_words < g.CW) g.hs_words = (g.CW + 3) & ~3u;
    return g;
}

__device__ __forceinline__ void st_sh_u16(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"((unsigned short)v) : "memory");
}
__device__ __forceinline__ void st_sh_u16_if(uint32_t addr, uint32_t v, bool p) {
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.shared.u16 [%0], %1;\n\t}" ::"r"(addr),
        "h"((unsigned short)v), "r"((uint32_t)p)
        : "memory");
}
__device__ __forceinline__ uint32_t atom_or_sh_if(uint32_t addr, uint32_t v, bool p) {
    uint32_t old = 0;
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\t@q atom.shared.or.b32 %0, [%1], %2;\n\t}"
        : "+r"(old)
        : "r"(addr), "r"(v), "r"((uint32_t)p)
        : "memory");
    return old;
}
__device__ __forceinline__ uint4 ld_sh_v4(uint32_t addr) {
    uint4 r;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "r"(addr)
                 : "memory");
    return r;
}
__device__ __forceinline__ void st_sh_zero16(uint32_t addr) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(addr), "r"(0u) : "memory");
}
__device__ __forceinline__ void red_or_sh2(uint32_t addr, uint32_t v) {
    asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// P2 + R of one vertex (k_floyd_warp, k_sample_head): from the second-comer
// lists (nsl per lane in SL) and chain lists (ncl per lane in CLs) of a full P1
// over HS, the collided draws' replacements as extras.  May set replay.
// F, HS, SL are warp-private shared memory (FW words, hs_words words, 32 lists).
__device__ __forceinline__ void fw_resolve(const SamplerArgs& a, const FwGeom& fg, uint64_t u,
                                           uint64_t key, uint32_t* F, uint16_t* HS, uint16_t* SL,
                                           const uint16_t* CLs, uint32_t nsl, uint32_t ncl,
                                           bool& replay, unsigned long long& ncol) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t D = a.draws, base = a.base, FW = fg.FW;
    const uint32_t hs_log = fg.B - 6;  // resolution hash: 2^B / 64 u64 slots
    const uint32_t hs_mask = (1u << hs_log) - 1;
    unsigned long long* HT = reinterpret_cast<unsigned long long*>(F);  // F's memory in R
    uint32_t* colbits = reinterpret_cast<uint32_t*>(HS);                // HS's memory in R
    const uint32_t Fa = smem_addr(F), HSa = smem_addr(HS);
    const uint16_t* mySL = SL + lane * kFwSLL;
    const EdgeSink xs{a.extras, a.extras_capacity, &a.counters[C_EXTRA_CURSOR], 0};
    auto zero_words = [&](uint32_t addr, uint32_t words) {  // words: a multiple of 4
        for (uint32_t w = lane; w < words / 4; w += 32) st_sh_zero16(addr + 16 * w);
    };
        // ---- P2: the group list, compacted warp-wide into SL's memory ----
    uint32_t ngl = 0;  // warp-uniform
    uint16_t* GLw = SL;  // [32 * kFwSLL] (SL is consumed when F is rebuilt)
    const uint32_t SLw = smem_addr(SL);
    constexpr uint32_t kGLCap = 32 * kFwSLL;
    if (!replay && __any_sync(kFull, nsl != 0)) {
        __syncwarp();
        zero_words(Fa, FW);  // F := the shared bits
        __syncwarp();
        for (uint32_t j = 0; j < nsl; ++j) red_or_sh2(Fa + ((mySL[j] >> 5) << 2), 1u << (mySL[j] & 31));
        __syncwarp();
        // (the last row's slots past D hold stale bits: keep them inside F)
        const uint32_t hmask = FW * 32 - 1;
        for (uint32_t c0 = 0; c0 * 8 < D; c0 += 32) {  // 8 hashes (16 bytes) per lane per step
            const uint32_t c = c0 + lane;
            uint32_t hits = 0;
            if (c * 8 < D) {
                const uint4 w4 = ld_sh_v4(HSa + 16 * c);
                const uint32_t ws[4] = {w4.x, w4.y, w4.z, w4.w};
                uint32_t fw[8];
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    fw[j] = ld_sh(Fa + ((((ws[j >> 1] >> ((j & 1) * 16)) & hmask) >> 5) << 2));
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    hits |= ((fw[j] >> ((ws[j >> 1] >> ((j & 1) * 16)) & 31)) & 1u) << j;
                if (c * 8 + 8 > D) hits &= (1u << (D - c * 8)) - 1u;
            }
            while (__any_sync(kFull, hits != 0)) {  // ~0.5 hits per lane per step
                const bool has = hits != 0;
                const unsigned m = __ballot_sync(kFull, has);
                const uint32_t slot = ngl + __popc(m & lanemask_lt());
                st_sh_u16_if(SLw + 2 * min(slot, kGLCap - 1), c * 8 + __ffs(hits) - 1, has);
                hits &= hits - 1;
                ngl += __popc(m);
            }
        }
        replay = ngl > kGLCap || ngl > FW / 2 * 3 / 4;  // list room, hash load <= 3/4
    }
    // ---- R: collided draws ----
    const bool chains = !replay && __any_sync(kFull, ncl != 0);
    if (chains && warp_sum(ncl) > FW / 2) replay = true;  // chain sort room (F's memory)
    const bool groups = !replay && ngl != 0;
    if (groups || (chains && !replay)) {
        __syncwarp();
        zero_words(HSa, fg.CW);  // HS is consumed: its memory holds the collided bitmap
        auto draw_t = [&](uint32_t i) {
            bool f;
            return lemire32(stream_at(key, (uint64_t)i + 1), base + i + 1, f);
        };
        auto emit = [&](uint32_t i) {  // collided draw i: its replacement j_i = base + i
            const unsigned long long s2 = atomicAdd(xs.cursor, 1ull);
            const uint32_t e2 = base + i;
            if (s2 < xs.capacity) xs.keys[s2] = (u << 32) | (e2 + (e2 >= (uint32_t)u ? 1u : 0u));
            ++ncol;
        };
        if (groups) {
            zero_words(Fa, FW);  // F's memory := an empty (t + 1, min index) hash
            __syncwarp();
            uint32_t gt[4];  // the values of this lane's first entries (<= 128 total: kept)
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const uint32_t e = lane + 32 * r;
                gt[r] = e < ngl ? draw_t(GLw[e]) : 0u;
            }
            auto t_of = [&](uint32_t e, int r) { return r < 4 ? gt[r] : draw_t(GLw[e]); };
            for (uint32_t e0 = 0, r = 0; e0 < ngl; e0 += 32, ++r) {
                const uint32_t e = e0 + lane;
                if (e < ngl) {
                    const uint32_t i = GLw[e], t = t_of(e, r);
                    FW_CHECK(i < D, "group index");
                    const unsigned long long kk = ((unsigned long long)(t + 1u) << 32) | i;  // never 0
                    uint32_t sl = (t * 0x85EBCA6Bu) >> (32 - hs_log);
                    for (;;) {
                        const unsigned long long o2 = atomicCAS(&HT[sl], 0ull, kk);
                        if (o2 == 0ull) break;
                        if ((o2 >> 32) == (kk >> 32)) {
                            atomicMin(&HT[sl], kk);
                            break;
                        }
                        sl = (sl + 1) & hs_mask;
                    }
                }
            }
            __syncwarp();
            for (uint32_t e0 = 0, r = 0; e0 < ngl; e0 += 32, ++r) {
                const uint32_t e = e0 + lane;
                if (e < ngl) {
                    const uint32_t i = GLw[e], t = t_of(e, r);
                    uint32_t sl = (t * 0x85EBCA6Bu) >> (32 - hs_log);
                    while ((uint32_t)(HT[sl] >> 32) != t + 1u) sl = (sl + 1) & hs_mask;
                    if ((uint32_t)HT[sl] != i) {  // an earlier draw has the same value
                        FW_CHECK((i >> 5) < fg.CW, "colbits (group)");
                        atomicOr(&colbits[i >> 5], 1u << (i & 31));
                        emit(i);
                    }
                }
            }
            __syncwarp();
        }
        if (chains) {
            // chain candidates of all lanes in index order (tiny), against the
            // collided set; a collision makes its replacement visible to later ones
            const unsigned cm = __ballot_sync(kFull, ncl != 0);
            if (lane == 0) {
                uint32_t* cl = F;  // F's memory is free now (FW >= 2 x the entries)
                uint32_t nc = 0;
                for (unsigned m = cm; m; m &= m - 1) {
                    const int l = __ffs(m) - 1;
                    for (int j = 0; j < kFwCLL; ++j) {
                        const uint32_t v = CLs[l * kFwCLL + j];
                        if (v == 0u) break;  // empty slot (a chain entry has i > 0)
                        FW_CHECK(v < D && nc < FW, "chain entry");
                        uint32_t y = nc++;
                        while (y > 0 && cl[y - 1] > v) {
                            cl[y] = cl[y - 1];
                            --y;
                        }
                        cl[y] = v;
                    }
                }
                for (uint32_t x = 0; x < nc; ++x) {
                    const uint32_t i = cl[x];
                    if ((colbits[i >> 5] >> (i & 31)) & 1u) continue;  // already collided
                    const uint32_t kx = draw_t(i) - base;
                    FW_CHECK(kx < i, "chain target");
                    if ((colbits[kx >> 5] >> (kx & 31)) & 1u) {  // t_i = j_k, draw k collided
                        colbits[i >> 5] |= 1u << (i & 31);
                        emit(i);
                    }
                }
            }
            __syncwarp();
        }
    }
}

template <int R>
__global__ void __launch_bounds__(32, 8) k_floyd_warp(const SamplerArgs a, const FwGeom fg) {
    constexpr uint32_t ITER = 32 * R;
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t D = a.draws, base = a.base;
    const uint32_t shift = 32 - fg.B, FW = fg.FW;
    const uint32_t hs_log = fg.B - 6;  // resolution hash: 2^B / 64 u64 slots
    const uint32_t hs_mask = (1u << hs_log) - 1;

    uint32_t* F = reinterpret_cast<uint32_t*>(smem);
    unsigned long long* HT = reinterpret_cast<unsigned long long*>(smem);  // F's memory in R
    uint16_t* HS = reinterpret_cast<uint16_t*>(F + FW);
    uint32_t* colbits = F + FW;  // HS's memory in R
    uint16_t* SL = HS + 2 * fg.hs_words;  // [32][kFwSLL]
    uint16_t* CLs = SL + 32 * kFwSLL;     // [32][kFwCLL]
    const uint32_t Fa = smem_addr(F), HSa = smem_addr(HS);
    const uint32_t SLa = smem_addr(SL + lane * kFwSLL), CLa = smem_addr(CLs + lane * kFwCLL);
    uint16_t* mySL = SL + lane * kFwSLL;
    uint16_t* myCL = CLs + lane * kFwCLL;
    uint32_t* irr_list = reinterpret_cast<uint32_t*>(a.scratch64);
    const EdgeSink xs{a.extras, a.extras_capacity, &a.counters[C_EXTRA_CURSOR], 0};
    unsigned long long ncol = 0;

    auto zero_words = [&](uint32_t addr, uint32_t words) {  // words: a multiple of 4
        for (uint32_t w = lane; w < words / 4; w += 32) st_sh_zero16(addr + 16 * w);
    };
    for (int j = 0; j < kFwCLL; ++j) myCL[j] = 0;  // chain lists start empty (0 = no entry)

    uint64_t u, uend, ustep;
    if (a.rows_per_block) {
        u = a.row_begin + (uint64_t)blockIdx.x * a.rows_per_block;
        uend = min(u + a.rows_per_block, a.row_end);
        ustep = 1;
    } else {
        u = a.row_begin + blockIdx.x;
        uend = a.row_end;
        ustep = gridDim.x;
    }
    for (; u < uend; u += ustep) {
        const uint64_t key = vertex_key(a.seed_mixed, u);
        zero_words(Fa, FW);
        __syncwarp();
        // test hook: a hooked vertex is replayed (its pre-condition "fires" at D/2)
        bool replay = a.force_mod != 0 && (u % a.force_mod) == 0;
        uint32_t nsl = 0, ncl = 0;

        // ---- P1 ----
        // one step of R slots; TAIL masks draws >= D (only the last step)
        auto step = [&](uint32_t i0, uint64_t z, auto tail_c) -> bool {
            constexpr bool TAIL = decltype(tail_c)::value;
            const uint32_t b0 = base + i0 + lane + 1;  // Lemire bound of slot 0
            uint32_t tv[R], mn = 0xffffffffu;
#pragma unroll
            for (int k = 0; k < R; ++k) {
                uint32_t slo;
                tv[k] = lemire32_slo(mix(z + (uint64_t)(32 * k) * kGamma), b0 + 32 * k, slo);
                const bool valid = !TAIL || i0 + 32 * k + lane < D;
                mn = valid ? min(mn, slo) : mn;
            }
            if (__any_sync(kFull, mn == 0u)) {  // rare: is a draw's pre-condition exact?
                bool fire_any = false;
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    bool fire;
                    (void)lemire32(mix(z + (uint64_t)(32 * k) * kGamma), b0 + 32 * k, fire);
                    fire_any |= fire && (!TAIL || i0 + 32 * k + lane < D);
                }
                if (__any_sync(kFull, fire_any)) return true;  // replay the vertex
            }
            uint32_t hk[R], old[R];
#pragma unroll
            for (int k = 0; k < R; ++k) {
                const uint32_t i = i0 + 32 * k + lane;
                hk[k] = (tv[k] * 0x9E3779B1u) >> shift;
                if (TAIL) st_sh_u16_if(HSa + 2 * i, hk[k], i < D);
                else st_sh_u16(HSa + 2 * i, hk[k]);
            }
#pragma unroll
            for (int k = 0; k < R; ++k) {  // all R atomics in flight before any result is used
                const uint32_t i = i0 + 32 * k + lane;
                const uint32_t addr = Fa + ((hk[k] >> 5) << 2), bit = 1u << (hk[k] & 31);
                old[k] = TAIL ? atom_or_sh_if(addr, bit, i < D) : atom_or_sh(addr, bit);
            }
#pragma unroll
            for (int k = 0; k < R; ++k) {
                const uint32_t i = i0 + 32 * k + lane;
                const bool sec = (old[k] >> (hk[k] & 31)) & 1u;  // a second comer (0 if masked)
                st_sh_u16_if(SLa + 2 * min(nsl, (uint32_t)kFwSLL - 1), hk[k], sec);
                nsl += sec ? 1u : 0u;
                const bool ch = (!TAIL || i < D) && tv[k] - base < i;  // t <= base + i always
                st_sh_u16_if(CLa + 2 * min(ncl, (uint32_t)kFwCLL - 1), i, ch);
                ncl += ch ? 1u : 0u;
            }
            return false;
        };
        if (!replay) {
            const uint32_t nfull = D / ITER;
            uint64_t z = key + (uint64_t)(lane + 1) * kGamma;
            for (uint32_t it = 0; it < nfull && !replay; ++it, z += (uint64_t)ITER * kGamma)
                replay = step(it * ITER, z, std::false_type{});
            if (!replay && nfull * ITER < D) replay = step(nfull * ITER, z, std::true_type{});
        }
        replay = replay || __any_sync(kFull, nsl > (uint32_t)kFwSLL || ncl > (uint32_t)kFwCLL);

        fw_resolve(a, fg, u, key, F, HS, SL, CLs, nsl, ncl, replay, ncol);
        for (int j = 0; j < kFwCLL; ++j) myCL[j] = 0;
        if (replay && lane == 0) {
            const unsigned long long s2 = atomicAdd(&a.counters[C_IRR_CURSOR], 1ull);
            FW_CHECK(s2 < a.row_end - a.row_begin, "replay list");
            irr_list[s2] = (uint32_t)u;  // capacity: one slot per row
        }
        __syncwarp();
    }
    ncol = warp_sum(ncol);
    if (lane == 0 && ncol) atomicAdd(&a.counters[C_COLLISIONS], ncol);
}
