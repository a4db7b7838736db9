// sngb_floyd_pipe.cuh -- k_floyd_pipe: k_floyd_lean's Floyd bookkeeping with the
// exact resolution done by the worker warps themselves, software-pipelined over
// the vertex loop (large n, 1024 < draws <= 4096: cfg4, cfg5).  Included by
// sngb_sampler.cu after sngb_floyd_bloom.cuh and sngb_floyd_lean.cuh.
//
// Why.  ncu on k_floyd_lean (cfg5, profiles/r02_ncu_floyd_lean_src_cfg5.md): a
// third of all warp samples sit at the top-of-vertex barrier waiting for the
// resolver warp, which is busy all the time -- one warp walks each vertex's
// ~240 group entries (6 % of the draws share a filter bit at B = 16) through a
// CAS hash at ~17 cycles per dependent instruction, 9 us per vertex.  The
// resolution is tiny but serial.  Here the 256 threads that found the entries
// resolve them, one or two entries per thread, and the three steps of a
// vertex's resolution ride on the barriers the next two vertices need anyway:
//
//   step s (vertex s of this block, parity s & 1), all 256 threads:
//     C  vertex s-2: empty the hash slots it used; thread 0 settles its chain
//        candidates (t_i in [base, base + i): graph.cpp:168 may meet an earlier
//        replacement j_k) against its collided bitmap, in index order
//     A  vertex s-1: insert my group entries (t, i) into its first-occurrence
//        hash (minimum index per value)
//     P1 vertex s: draws, filter bits, running tests        (k_floyd_lean)
//     -- barrier (with the OR of the threads' Lemire pre-condition) --
//     B  vertex s-1: look my entries up: an entry whose index is not the
//        minimum of its value collided (graph.cpp:168-170): its replacement j_i
//        becomes an extra, its bit goes to the collided bitmap
//     P2 vertex s: draws on a shared bit -> my warp's segment of the group
//        list, by ballot + popc (no atomics, no divergent push); chain
//        candidates -> the chain list
//     -- barrier --
//
// so a vertex costs two block barriers and no producer/consumer hand-off; the
// block is 8 worker warps (no resolver warp).  Lists, hashes and bitmaps are
// double-buffered by parity; two drain steps finish the last two vertices.
// List overflow and the Lemire reject pre-condition replay the vertex exactly
// (bloom_replay), as in k_floyd_lean.  Results equal k_floyd_bloom's bit for
// bit (tests/test_gpu_parity.py -k floyd_pipe).
#pragma once

constexpr int kPipeSeg = 64;          // group entries per warp and vertex
constexpr int kPipeHashLog2 = 9;
constexpr int kPipeSlots = 1 << kPipeHashLog2;
constexpr uint32_t kPipeMaxGroup = 384;  // entries per vertex the 512-slot hash takes
constexpr uint32_t kPipeNone = 0xffffffffu;

inline size_t pipe_smem_bytes(const BloomGeom& g) {
    return 4ull * g.words * 4                          // filter + shared-bit filter, x2 parity
           + 2ull * g.col_words * 4                    // collided bitmaps, x2 parity
           + 2ull * (kBloomThreads / 32) * kPipeSeg * 8  // group segments, x2 parity
           + 2ull * kChainCap * 4                      // chain lists, x2 parity
           + 2ull * kPipeSlots * 8;                    // first-occurrence hashes, x2 parity
}

// The vertices first, first + stride, ... (nv of them) of one block; `smem` is
// pipe_smem_bytes() of dynamic shared memory.  Called once per block by
// k_floyd_pipe and once per claimed chunk by k_duo (sngb_fused.cu).
template <int MAXR, bool SHT = false>
__device__ __forceinline__ void floyd_pipe_run(const SamplerArgs& a, unsigned char* smem,
                                               const uint64_t first, const uint64_t stride,
                                               const uint32_t nv) {
    constexpr int kT = kBloomThreads;
    constexpr int kW = kT / 32;
    // filter words (2^B / 32): bloom_geometry gives B = 15 up to 2048 draws (MAXR <= 8) and
    // B = 16 above, so the table size and the distance between a vertex's filter and
    // its shared-bit filter are compile-time constants (immediate offsets, no add)
    constexpr uint32_t WB = MAXR >= 9 ? 2048u : 1024u;
    constexpr uint32_t kShOff = 2 * WB * 4;  // bytes from filt[par] to shared_bits[par]
    const uint32_t W = a.col_words;
    uint32_t* filt = reinterpret_cast<uint32_t*>(smem);          // [2][WB]
    uint32_t* shared_bits = filt + 2 * WB;                         // [2][WB]
    uint32_t* colbits = shared_bits + 2 * WB;                      // [2][W]
    unsigned long long* glist =
        reinterpret_cast<unsigned long long*>(colbits + 2 * W);   // [2][kW][kPipeSeg]
    uint32_t* clist = reinterpret_cast<uint32_t*>(glist + 2 * kW * kPipeSeg);  // [2][kChainCap]
    unsigned long long* htab =
        reinterpret_cast<unsigned long long*>(clist + 2 * kChainCap);  // [2][kPipeSlots]
    __shared__ unsigned long long s_key[2];  // [parity] the vertex's stream key (thread 0 computes it)
    __shared__ uint32_t s_wc[2][kW];  // [parity][warp] group entries
    __shared__ uint32_t s_ng[2];      // [parity] group entries of the vertex
    __shared__ uint32_t s_cc[2];      // [parity] chain candidates
    __shared__ uint32_t s_ovf[2];     // [parity] a list overflowed

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const EdgeSink xs{a.extras, a.extras_capacity, &a.counters[C_EXTRA_CURSOR], 0};
    const uint32_t D = a.draws, base = a.base;
    unsigned long long ncol = 0, nrep = 0;
    auto emit = [&](uint64_t u, uint32_t e) {  // extra pair (u, partner of value e)
        const unsigned long long s2 = atomicAdd(xs.cursor, 1ull);
        if (s2 < xs.capacity)
            xs.keys[s2] = ((unsigned long long)u << 32) | (e + (e >= (uint32_t)u ? 1u : 0u));
    };

    for (uint32_t s = tid; s < 4 * WB + 2 * W; s += kT) filt[s] = 0;
    for (uint32_t s = tid; s < 2 * kPipeSlots; s += kT) htab[s] = ~0ull;
    if (tid < 2 * kW) (&s_wc[0][0])[tid] = 0;
    if (tid < 2) s_ng[tid] = s_cc[tid] = s_ovf[tid] = 0;
    if (tid == 0) s_key[0] = vertex_key(a.seed_mixed, first);  // vertex 0; vertex s + 1 in step s
    __syncthreads();

    const uint64_t dz = (uint64_t)kT * kGamma;  // counter step between a thread's draws
    // MAXR = ceil(D / kT): slots r < MAXR - 1 are full, the last one holds D - kT (MAXR - 1) draws
    const bool in_tail = (uint32_t)tid < D - kT * (MAXR - 1);
    constexpr uint32_t wmask = (WB - 1) << 2;      // byte offset of t's filter word
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
        uint32_t tr[MAXR];
        uint32_t tmax = 0;
        bool fired = false;
        uint32_t fa = 0;
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
            fa = smem_addr(filt + par * WB);
            if constexpr (SHT) {
                // shared draws: the head gather wrote t_i (and whether the stream met the
                // Lemire pre-condition or the test hook) for this row
                const uint32_t* tv = a.tbuf + (u - a.tbuf_row0) * D + tid;
#pragma unroll
                for (int r = 0; r < MAXR; ++r)
                    tr[r] = (r < MAXR - 1 || in_tail) ? __ldcs(tv + kT * r) : 0u;
                fired = tid == 0 && a.tflags[u - a.tbuf_row0] != 0;
#pragma unroll
                for (int r = 0; r < MAXR; ++r) {
                    const uint32_t t = tr[r];
                    if (r < MAXR - 1 || in_tail) {
                        tmax = max(tmax, t);
                        const uint32_t off = (t >> 3) & wmask, bit = 1u << (t & 31);
                        pipe_red_or_off<kShOff>(fa + off, atom_or_sh(fa + off, bit) & bit);
                    }
                }
            } else {
                const uint64_t key = s_key[par];  // vertex_key(a.seed_mixed, u)
                const uint64_t z0 = key + (uint64_t)(tid + 1) * kGamma;  // stream_at(key, i + 1)
                uint32_t smin = 0xffffffffu;
#pragma unroll
                for (int r = 0; r < MAXR; ++r) {
                    uint32_t slo;
                    const uint32_t t = lemire32_slo(mix(z0 + (uint64_t)r * dz), b0 + kT * r, slo);
                    tr[r] = t;
                    if (r < MAXR - 1 || in_tail) {
                        smin = min(smin, slo);
                        tmax = max(tmax, t);
                        const uint32_t off = (t >> 3) & wmask, bit = 1u << (t & 31);
                        pipe_red_or_off<kShOff>(fa + off, atom_or_sh(fa + off, bit) & bit);
                    }
                }
                fired = hook_thread && (u % a.force_mod) == 0;
                if (smin == 0u) {  // rare (2^-32 per draw): the exact pre-condition, lo < bound
#pragma unroll 1
                    for (int r = 0; r < MAXR; ++r) {
                        bool fi;
                        lemire32(mix(z0 + (uint64_t)r * dz), b0 + kT * r, fi);
                        fired |= fi && (r < MAXR - 1 || in_tail);
                    }
                }
            }
        }
        // (a shared flag + bar.sync instead of bar.red.or measured the same: 258.1 vs 257.3 ms)
        const bool any_fired = __syncthreads_or(fired);
        if (tid == 0 && s + 1 < nv) s_key[par ^ 1u] = vertex_key(a.seed_mixed, u + stride);

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
        auto replay = [&]() {
            __syncthreads();
            if (tid == 0) {
                ++nrep;
                ncol += bloom_replay(vertex_key(a.seed_mixed, u), u, a.n, base, filt, 4 * WB, xs);
                s_cc[par] = s_ovf[par] = 0;
            }
            if (tid < kW) s_wc[par][tid] = 0;
            __syncthreads();
            for (uint32_t x = tid; x < 4 * WB; x += kT) filt[x] = 0;
        };

        if (has_v) {
            if (any_fired) {
                replay();
            } else {
                // ---- P2: vertex s ----
                unsigned long long* wl = glist + (par * kW + warp) * kPipeSeg;
                uint32_t wpos = 0;
#pragma unroll
                for (int r = 0; r < MAXR; ++r) {
                    const uint32_t t = tr[r];
                    const uint32_t off = (t >> 3) & wmask, bit = 1u << (t & 31);
                    const bool hit =
                        (pipe_ld_off<kShOff>(fa + off) & bit) && (r < MAXR - 1 || in_tail);
                    const uint32_t m = __ballot_sync(kFull, hit);
                    const uint32_t pos = wpos + __popc(m & lt);
                    if (hit && pos < kPipeSeg)
                        wl[pos] = ((unsigned long long)t << 32) | ((uint32_t)tid + kT * r);
                    wpos += __popc(m);
                }
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
            }
        }
        __syncthreads();
        if (has_v && !any_fired && s_ovf[par]) {  // list overflow: exact replay
            replay();
            __syncthreads();
        }
    }
    ncol = warp_sum(ncol);
    nrep = warp_sum(nrep);
    if (lane == 0) {
        if (ncol) atomicAdd(&a.counters[C_COLLISIONS], ncol);
        if (nrep) atomicAdd(&a.counters[C_IRREGULAR], nrep);
    }
}

template <int MAXR, bool SHT>
__global__ void __launch_bounds__(kBloomThreads, 4) k_floyd_pipe(const SamplerArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint64_t first = a.row_begin + blockIdx.x;
    const uint32_t nv =
        first < a.row_end ? (uint32_t)((a.row_end - first + gridDim.x - 1) / gridDim.x) : 0u;
    floyd_pipe_run<MAXR, SHT>(a, smem, first, gridDim.x, nv);
}
