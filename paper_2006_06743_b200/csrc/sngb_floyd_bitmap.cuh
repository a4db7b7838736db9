// sngb_floyd_bitmap.cuh -- k_floyd_bitmap, Floyd bookkeeping for small n
// (the chosen-value set fits a per-warp bitmap of n-1 bits).  Included by
// sngb_sampler.cu.
//
// Small n means many collisions (cfg1: ~100 of 2000 draws per vertex collide,
// and ~200 draws can hit an earlier replacement), which overflows the
// dup/chain lists of k_floyd_fast.  Here one warp walks a vertex's draws in
// reference order, 32 at a time, with an exact membership bitmap:
//   in_prev : bit t set by an earlier chunk;
//   dup     : an earlier lane of this chunk drew the same t.  Every lane ORs
//             its own t first; a lane that did not see t before but gets its
//             bit back set shares t with another lane of the chunk, and only
//             then (a ballot, ~32^2/2n of the chunks) is the chunk resolved
//             exactly by match.any (0.5 lane-ops per SM-cycle: too slow to
//             run on every chunk);
//   chain   : t equals the replacement j_l of an earlier collided lane of
//             this chunk -- resolved by an in-order lane scan, only when the
//             (rare) precondition base + c0 <= t < j holds for some lane.
// Every chosen value (t, or j for a collided draw) is then set in the bitmap.
// A Lemire reject pre-condition replays the vertex exactly (lane 0).
#pragma once

constexpr int kBitmapStage = 128;

__global__ void __launch_bounds__(512) k_floyd_bitmap(const SamplerArgs a) {
    extern __shared__ __align__(16) uint32_t bsmem[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    const uint64_t gw = (uint64_t)blockIdx.x * wpb + wib;
    const uint64_t nw = (uint64_t)gridDim.x * wpb;
    const uint32_t words = a.col_words;  // bitmap words per warp (multiple of 4)
    uint32_t* bm = bsmem + (size_t)wib * words;
    unsigned long long* sbuf =
        reinterpret_cast<unsigned long long*>(bsmem + (size_t)wpb * words) + (size_t)wib * kBitmapStage;
    const EdgeSink xs{a.extras, a.extras_capacity, &a.counters[C_EXTRA_CURSOR], 0};
    WarpStage<kBitmapStage> stage{sbuf, 0};
    unsigned long long ncol = 0, nrep = 0;
    const uint32_t D = a.draws, base = a.base;

    auto clear = [&]() {
        uint4* b4 = reinterpret_cast<uint4*>(bm);
        for (uint32_t w = lane; w < words / 4; w += 32) b4[w] = make_uint4(0, 0, 0, 0);
        __syncwarp();
    };

    for (uint64_t u = a.row_begin + gw; u < a.row_end; u += nw) {
        clear();
        const uint64_t key = vertex_key(a.seed_mixed, u);
        bool replay = false;
        // draws of the next chunk are computed one chunk ahead (independent of
        // the bitmap operations, so the RNG overlaps their latency); the stream
        // counter is carried incrementally and the test hook resolved per vertex
        const uint32_t hook = (a.force_mod != 0 && (u % a.force_mod) == 0) ? D / 2 : 0xffffffffu;
        uint64_t z = key + (uint64_t)(lane + 1) * kGamma;  // stream_at(key, i + 1), i = lane
        bool fire_next;
        uint32_t t_next = lemire32(mix(z), base + lane + 1, fire_next);
        fire_next = (fire_next || (uint32_t)lane == hook) && (uint32_t)lane < D;
        for (uint32_t c0 = 0; c0 < D; c0 += 32) {
            const uint32_t i = c0 + lane;
            const bool valid = i < D;
            const bool fire = fire_next;
            const uint32_t t = valid ? t_next : 0u;
            z += 32ull * kGamma;
            if (c0 + 32 < D) {
                t_next = lemire32(mix(z), base + i + 33, fire_next);
                fire_next = (fire_next || i + 32 == hook) && i + 32 < D;
            }
            if (__ballot_sync(kFull, fire)) {
                replay = true;
                break;
            }
            const bool in_prev = valid && ((bm[t >> 5] >> (t & 31)) & 1u);
            // set t now: a collided draw's t is in the set anyway, so the final
            // bitmap is unchanged (the replacements j are added below)
            const uint32_t old = valid ? atomicOr(&bm[t >> 5], 1u << (t & 31)) : 0u;
            const bool clash = valid && !in_prev && ((old >> (t & 31)) & 1u);
            bool col = in_prev;
            if (__ballot_sync(kFull, clash)) {
                const unsigned mm = __match_any_sync(kFull, valid ? t : (0xffffffffu - lane));
                col = valid && (in_prev || (mm & lanemask_lt()) != 0);
            }
            const uint32_t j = base + i;  // Floyd's replacement value for draw i
            if (__ballot_sync(kFull, valid && !col && t >= base + c0 && t < j)) {
                for (int l = 0; l < 31; ++l) {
                    const bool cl = __shfl_sync(kFull, col, l);
                    if (cl && lane > l && valid && !col && t == base + c0 + l) col = true;
                }
            }
            if (valid && col) atomicOr(&bm[j >> 5], 1u << (j & 31));
            __syncwarp();
            const unsigned cm = __ballot_sync(kFull, col);
            if (lane == 0) ncol += __popc(cm);
            stage.push(col, ((unsigned long long)u << 32) | (j + (j >= (uint32_t)u ? 1u : 0u)), xs,
                       lane);
        }
        if (replay) {  // exact sequential replay of graph.cpp:163-174
            clear();
            if (lane == 0) {
                ++nrep;
                SeqStream st{key, 0};
                const uint64_t pool = a.n - 1;
                for (uint64_t jj = base; jj < pool; ++jj) {
                    const uint32_t t = (uint32_t)st.next_below(jj + 1);
                    uint32_t e = t;
                    if ((bm[t >> 5] >> (t & 31)) & 1u) e = (uint32_t)jj;
                    bm[e >> 5] |= 1u << (e & 31);
                    const unsigned long long s2 = atomicAdd(xs.cursor, 1ull);
                    if (s2 < xs.capacity)
                        xs.keys[s2] = ((unsigned long long)u << 32) | (e + (e >= (uint32_t)u ? 1u : 0u));
                }
            }
            __syncwarp();
        }
    }
    stage.flush(xs, lane);
    if (lane == 0) {
        if (ncol) atomicAdd(&a.counters[C_COLLISIONS], ncol);
        if (nrep) atomicAdd(&a.counters[C_IRREGULAR], nrep);
    }
}
