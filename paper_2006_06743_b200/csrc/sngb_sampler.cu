// sngb_sampler.cu -- Floyd bookkeeping of the sampled eps-graph (k_floyd).
//
// Reference: graph.cpp:161-174 (Floyd's algorithm over [0, n-2] with the
// rng.hpp:35-48 Lemire draw), run one vertex at a time with an
// std::unordered_set.  The draw values t_i need no state (counter i+1, SURVEY
// Appendix C); only the Floyd replacements need bookkeeping:
//
//     draw i collides  <=>  t_i in S_{i-1} = {t_0..t_{i-1}} U {j_k : k < i collided}
//     (j_k = base + k is draw k's replacement, base = n-1-draws)
//
// which splits into an ORDER-FREE part and a short ordered chain:
//
//   dupT_i  = t_i equals an earlier t_k          -> first occurrence via a
//             shared-memory hash of (t, min index), all draws in parallel;
//   chain_i = t_i = j_k for a collided k < i     -> only possible when
//             t_i >= base; k = t_i - base; resolved in index order.
//
// Three kernels, chosen by launch_sampler:
//   k_floyd_bitmap (sngb_floyd_bitmap.cuh)  n <= 32 k: exact per-warp bitmap,
//                                           draws in reference order;
//   k_floyd_bloom  (sngb_floyd_bloom.cuh)   draws <= 4096: conflict-free bit
//                                           filter + resolver warp (the
//                                           BASELINE configs 2-5);
//   k_floyd        (this file)              anything else: one block per
//                                           vertex, (t, min index) hash in
//                                           shared memory or L2 scratch.
// Every kernel emits the replacement partner j_i + (j_i >= u) of every
// collided draw as an "extra" pair for k_extras, and replays a vertex whose
// stream meets the Lemire reject pre-condition exactly and sequentially (all
// of its partners become extras).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <mutex>
#include <set>
#include <type_traits>
#include <utility>
#include <cstdlib>

#include "sngb_device.cuh"
#include "sngb_internal.cuh"
#include "sngb_rng.cuh"

namespace sngb {

namespace {

constexpr int kFloydThreads = 256;
constexpr int kFloydWarps = kFloydThreads / 32;
constexpr int kFloydStage = 64;
constexpr unsigned long long kEmpty64 = ~0ull;  // t < n-1 < 2^32-1, never a real key

__device__ __forceinline__ uint32_t hslot(uint32_t t, uint32_t shift) {
    return (t * 0x9E3779B1u) >> shift;
}

// The table is bucketized: 4 entries (t << 32 | first index) per 32-byte
// bucket, read with two 16-byte shared loads, linear probing over buckets.
// Load factor <= 0.5, so a probe almost always ends in the home bucket and
// the lanes of a warp stay converged (a slot-wise linear probe at 0.6 load
// left warps iterating at 2-4 active lanes).  Entries are filled in slot
// order and never emptied within a vertex, so the first slot holding t is
// unique and every draw of t meets it.
struct Bucket {
    unsigned long long e[4];
};

__device__ __forceinline__ Bucket load_bucket(const unsigned long long* tab, uint32_t b) {
    const unsigned long long* p = tab + 4 * (size_t)b;
    Bucket r;
    asm volatile("ld.volatile.v2.u64 {%0, %1}, [%2];" : "=l"(r.e[0]), "=l"(r.e[1]) : "l"(p));
    asm volatile("ld.volatile.v2.u64 {%0, %1}, [%2];" : "=l"(r.e[2]), "=l"(r.e[3]) : "l"(p + 2));
    return r;
}

// Insert (t, i); the entry of t keeps the minimum index (first occurrence).
__device__ __forceinline__ void insert_min(unsigned long long* tab, uint32_t t, uint32_t i,
                                           uint32_t mask, uint32_t shift) {
    const unsigned long long mine = ((unsigned long long)t << 32) | i;
    uint32_t b = hslot(t, shift);
    for (;;) {
        const Bucket bk = load_bucket(tab, b);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            unsigned long long cur = bk.e[k];
            if (cur == kEmpty64) {
                cur = atomicCAS(&tab[4 * (size_t)b + k], kEmpty64, mine);
                if (cur == kEmpty64) return;
            }
            if ((uint32_t)(cur >> 32) == t) {
                if ((uint32_t)cur > i) atomicMin(&tab[4 * (size_t)b + k], mine);
                return;
            }
        }
        b = (b + 1) & mask;
    }
}

__device__ __forceinline__ uint32_t first_index(const unsigned long long* tab, uint32_t t,
                                                uint32_t mask, uint32_t shift) {
    uint32_t b = hslot(t, shift);
    for (;;) {
        const Bucket bk = load_bucket(tab, b);
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if ((uint32_t)(bk.e[k] >> 32) == t) return (uint32_t)bk.e[k];
        b = (b + 1) & mask;
    }
}

// Single-thread insert-if-absent for the exact sequential replay.
__device__ bool insert_seq(unsigned long long* tab, uint32_t t, uint32_t mask, uint32_t shift) {
    uint32_t b = hslot(t, shift);
    for (;;) {
        for (int k = 0; k < 4; ++k) {
            unsigned long long& cur = tab[4 * (size_t)b + k];
            if (cur == kEmpty64) {
                cur = (unsigned long long)t << 32;
                return true;
            }
            if ((uint32_t)(cur >> 32) == t) return false;
        }
        b = (b + 1) & mask;
    }
}

__device__ __forceinline__ uint32_t draw_t(uint64_t key, uint32_t i, uint32_t base, bool& fire) {
    return lemire32(stream_at(key, (uint64_t)i + 1), base + i + 1, fire);
}

template <bool SHARED>
__global__ void __launch_bounds__(kFloydThreads) k_floyd(const SamplerArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t P = 4 * (a.hash_mask + 1);  // entries (4 per bucket)
    const uint32_t W = a.col_words;  // words of one D-bit bitmap (multiple of 4)
    unsigned long long* tab = SHARED ? reinterpret_cast<unsigned long long*>(smem)
                                     : a.scratch64 + (uint64_t)blockIdx.x * P;
    uint32_t* colbits = reinterpret_cast<uint32_t*>(smem + (SHARED ? (size_t)P * 8 : 0));
    uint32_t* cbits = colbits + W;
    unsigned long long* sbuf = reinterpret_cast<unsigned long long*>(cbits + W);
    const int tid = threadIdx.x, lane = tid & 31, wib = tid >> 5;
    WarpStage<kFloydStage> stage{sbuf + wib * kFloydStage, 0};
    const EdgeSink xs{a.extras, a.extras_capacity, &a.counters[C_EXTRA_CURSOR], 0};
    const uint32_t D = a.draws, base = a.base, mask = a.hash_mask, shift = a.hash_shift;
    unsigned long long ncol = 0, nirr = 0;

    for (uint64_t u = a.row_begin + blockIdx.x; u < a.row_end; u += gridDim.x) {
        // ---- clear (table + both bitmaps) ----
        {
            ulonglong2* t2 = reinterpret_cast<ulonglong2*>(tab);
            for (uint32_t s = tid; s < P / 2; s += kFloydThreads) t2[s] = make_ulonglong2(kEmpty64, kEmpty64);
            uint4* b4 = reinterpret_cast<uint4*>(colbits);
            for (uint32_t s = tid; s < (2 * W) / 4; s += kFloydThreads) b4[s] = make_uint4(0, 0, 0, 0);
        }
        __syncthreads();
        const uint64_t key = vertex_key(a.seed_mixed, u);

        // ---- phase 1: every draw inserts (t, i); slot keeps the first index ----
        bool fired = false;
        for (uint32_t i = tid; i < D; i += kFloydThreads) {
            bool f;
            const uint32_t t = draw_t(key, i, base, f);
            fired |= f || test_fire(a.force_mod, u, i, D);
            insert_min(tab, t, i, mask, shift);
        }
        if (__syncthreads_or(fired)) {
            // ---- irregular vertex: exact sequential replay (graph.cpp:163-174) ----
            for (uint32_t s = tid; s < P; s += kFloydThreads) tab[s] = kEmpty64;
            __syncthreads();
            if (tid == 0) {
                ++nirr;
                SeqStream st{key, 0};
                const uint64_t pool = a.n - 1;
                for (uint64_t jj = base; jj < pool; ++jj) {
                    const uint32_t t = (uint32_t)st.next_below(jj + 1);
                    uint32_t e = t;
                    if (!insert_seq(tab, t, mask, shift)) {
                        insert_seq(tab, (uint32_t)jj, mask, shift);
                        e = (uint32_t)jj;
                    }
                    const uint32_t pe = e + (e >= (uint32_t)u ? 1u : 0u);
                    const unsigned long long slot = atomicAdd(xs.cursor, 1ull);
                    if (slot < xs.capacity) xs.keys[slot] = ((unsigned long long)u << 32) | pe;
                }
            }
            __syncthreads();
            continue;
        }

        // ---- phase 2: classify: dupT -> collided; possible chain -> candidate ----
        bool anycand = false;
        for (uint32_t i = tid; i < D; i += kFloydThreads) {
            bool f;
            const uint32_t t = draw_t(key, i, base, f);
            if (first_index(tab, t, mask, shift) != i) {
                atomicOr(&colbits[i >> 5], 1u << (i & 31));
            } else if (t >= base && t - base < i) {
                atomicOr(&cbits[i >> 5], 1u << (i & 31));
                anycand = true;
            }
        }
        // ---- phase 3: chains t_i = j_k (k collided, k < i), in index order ----
        if (__syncthreads_or(anycand)) {
            if (tid == 0) {
                for (uint32_t w = 0; w < W; ++w) {
                    uint32_t bits = cbits[w];
                    while (bits) {
                        const uint32_t b = __ffs(bits) - 1;
                        bits &= bits - 1;
                        const uint32_t i = 32 * w + b;
                        bool f;
                        const uint32_t k = draw_t(key, i, base, f) - base;
                        if ((colbits[k >> 5] >> (k & 31)) & 1u) colbits[i >> 5] |= 1u << (i & 31);
                    }
                }
            }
            __syncthreads();
        }
        // ---- phase 4: emit Floyd replacements j_i of collided draws ----
        for (uint32_t i0 = 0; i0 < D; i0 += kFloydThreads) {
            const uint32_t i = i0 + tid;
            const bool col = i < D && ((colbits[i >> 5] >> (i & 31)) & 1u);
            const unsigned cm = __ballot_sync(kFull, col);
            if (lane == 0) ncol += __popc(cm);
            const uint32_t j = base + i;
            const uint32_t pj = j + (j >= (uint32_t)u ? 1u : 0u);
            stage.push(col, ((unsigned long long)u << 32) | pj, xs, lane);
        }
        __syncthreads();
    }
    stage.flush(xs, lane);
    if (lane == 0) {
        if (ncol) atomicAdd(&a.counters[C_COLLISIONS], ncol);
        if (nirr && wib == 0) atomicAdd(&a.counters[C_IRREGULAR], nirr);
    }
}

#ifndef SNGB_SHARE_DRAWS
#define SNGB_SHARE_DRAWS 0
#endif
#include "sngb_floyd_bitmap.cuh"
#include "sngb_floyd_bloom.cuh"
#include "sngb_floyd_warp.cuh"
#include "sngb_floyd_lean.cuh"
#include "sngb_floyd_pipe.cuh"
#ifndef SNGB_FW_R
#define SNGB_FW_R 8  // draw slots per lane per step of k_floyd_warp
#endif

}  // namespace

// Geometry of the per-vertex tables.
void floyd_geometry(uint32_t draws, uint32_t& slots, uint32_t& col_words) {
    uint32_t buckets = 16;
    while (20 * buckets < 8 * draws) buckets <<= 1;  // 4 * buckets >= 1.6 * draws: load <= 0.625
    slots = 4 * buckets;
    col_words = ((draws + 31) / 32 + 3) & ~3u;
}

size_t floyd_smem_bytes(uint32_t draws, bool shared_table) {
    uint32_t slots, cw;
    floyd_geometry(draws, slots, cw);
    return (shared_table ? (size_t)slots * 8 : 0) + (size_t)cw * 8 +
           (size_t)kFloydWarps * kFloydStage * 8;
}

bool floyd_shared(uint32_t draws) { return floyd_smem_bytes(draws, true) <= 200 * 1024; }

size_t floyd_scratch_bytes(uint32_t draws, int num_sms, uint64_t rows) {
    // k_floyd_warp's replay list (one u32 per row); k_floyd's L2 tables
    if (floyd_shared(draws)) return rows * 4;
    uint32_t slots, cw;
    floyd_geometry(draws, slots, cw);
    return std::max<size_t>((size_t)num_sms * 2 * slots * 8, rows * 4);
}

// A kernel's dynamic shared-memory limit is raised once per device to the
// opt-in maximum: concurrent callers (the batched API's host workers) with
// different sizes must never lower it under another's launch.
cudaError_t raise_smem_limit(const void* kernel) {
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    int dev = 0, mx = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    if (done.count({kernel, dev})) return cudaSuccess;
    cudaError_t e = cudaDeviceGetAttribute(&mx, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa{};
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, kernel);  // less its static shared memory
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 mx - (int)fa.sharedSizeBytes);
    if (e == cudaSuccess) done.insert({kernel, dev});
    return e;
}

// k_floyd_pipe pays where a vertex has many group entries for one resolver warp
// (about draws^2 / 2^B of them: cfg5 240, cfg4 93).  A sweep over the draw count on
// the final kernels (profiles/r02_pipe_threshold.jsonl, n = 4 M, 64 rows per block):
// k_floyd_lean is ahead up to 2600 draws at B = 16 (103 entries: 32.4 vs 32.8 ms; 2100:
// 25.4 vs 27.2; 1500 at B = 15: 20.6 vs 20.7), k_floyd_pipe at 2048 draws (B = 15, 128
// entries: 27.0 vs 30.6 ms), 3000 (137: 36.6 vs 38.9) and everywhere above (4096: 56.6
// vs 62.8), so it takes over from 120 entries.  SNGB_FLOYD_PIPE=0|1 forces the choice.
static bool pipe_wanted(uint32_t D) {
    if (D <= 1024 || D > 4096) return false;
    if (const char* penv = std::getenv("SNGB_FLOYD_PIPE")) return std::atoi(penv) != 0;
    const BloomGeom bg = bloom_geometry(D);
    return (uint64_t)D * D >= (120ull << bg.bits_log2);
}

bool sampler_uses_pipe(uint64_t n, uint32_t draws) {
    const uint64_t bm_words = (((n - 1) + 31) / 32 + 3) & ~3ull;
    if (bm_words * 4 <= 9216 && !std::getenv("SNGB_FLOYD_NO_BITMAP")) return false;
    const char* fwenv = std::getenv("SNGB_FLOYD_WARP");
    if (fwenv && std::atoi(fwenv) == 1 && !std::getenv("SNGB_FLOYD_BLOOM")) return false;
    return n - 2 < 0xffffffffull && pipe_wanted(draws);
}

// Shared draws (builds with -DSNGB_SHARE_DRAWS=1, then SNGB_SHARE_T=1): wherever
// launch_sampler would run the filter kernels on more than 1024 draws per vertex and
// the head gather runs, the gather writes its draws and k_floyd_pipe reads them
// (sngb_api.cu pipelines row chunks through a bounded buffer).  Bit-exact, and no
// faster (cfg5 613 vs 606 ms: the stores cost the L1TEX-bound gather what the loads
// save the sampler, profiles/r02_ab_share.jsonl), hence a build flag.
bool share_eligible(uint64_t n, uint32_t draws) {
#if !SNGB_SHARE_DRAWS
    (void)n;
    (void)draws;
    return false;
#endif
    const char* se = std::getenv("SNGB_SHARE_T");
    if (!se || std::atoi(se) == 0) return false;
    // an explicit choice of Floyd kernel (A/B runs, the parity tests) keeps its own draws
    if (std::getenv("SNGB_FLOYD_PIPE") || std::getenv("SNGB_FLOYD_LEAN")) return false;
    if (draws <= 1024 || draws > 4096 || n - 2 >= 0xffffffffull) return false;
    const uint64_t bm_words = (((n - 1) + 31) / 32 + 3) & ~3ull;
    if (bm_words * 4 <= 9216 && !std::getenv("SNGB_FLOYD_NO_BITMAP")) return false;
    const char* fwenv = std::getenv("SNGB_FLOYD_WARP");
    return !(fwenv && std::atoi(fwenv) == 1 && !std::getenv("SNGB_FLOYD_BLOOM"));
}

cudaError_t launch_sampler(const SamplerArgs& in, cudaStream_t s, int num_sms) {
    const uint64_t rows = in.row_end - in.row_begin;
    if (rows == 0 || in.draws == 0) return cudaSuccess;
    SamplerArgs a = in;
    const uint32_t D = a.draws;
    // small n: exact per-warp bitmap of the chosen values, draws in reference order
    // (up to 9 KB per warp: n <= 73 k, 2 blocks of 8 warps per SM)
    const uint64_t bm_words = (((a.n - 1) + 31) / 32 + 3) & ~3ull;
    if (bm_words * 4 <= 9216 && !std::getenv("SNGB_FLOYD_NO_BITMAP")) {
        a.col_words = (uint32_t)bm_words;
        // warps per block: the most resident warps per SM for this bitmap size
        // (shared memory bound for large bitmaps: 8-warp blocks fit 2 per SM at
        // n = 70 k, i.e. 16 warps; 11-warp blocks fit 22), SNGB_BITMAP_WPB overrides
        const size_t per_warp = bm_words * 4 + kBitmapStage * 8;
        const cudaError_t attr_rc = raise_smem_limit(reinterpret_cast<const void*>(k_floyd_bitmap));
        if (attr_rc != cudaSuccess) return attr_rc;
        int wpb = 8, best = 0;
        static thread_local uint64_t memo_words = 0;  // the search costs ~13 occupancy queries
        static thread_local int memo_wpb = 8;
        if (const char* ev = std::getenv("SNGB_BITMAP_WPB")) wpb = std::max(1, std::min(16, std::atoi(ev)));
        else if (memo_words == bm_words) wpb = memo_wpb;
        else
            for (int w = 4; w <= 16; ++w) {
                int pb = 0;
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pb, k_floyd_bitmap, w * 32, w * per_warp);
                if (pb * w > best) best = pb * w, wpb = w, memo_wpb = w, memo_words = bm_words;
            }
        const size_t smem = (size_t)wpb * per_warp;
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_floyd_bitmap, wpb * 32, smem);
        if (per_sm < 1) per_sm = 1;
        const uint64_t want = (rows + wpb - 1) / wpb, cap = (uint64_t)num_sms * per_sm;
        k_floyd_bitmap<<<(unsigned)(want < cap ? want : cap), wpb * 32, smem, s>>>(a);
        note_launch(1);
        return cudaGetLastError();
    }
    // large n, draws <= 1024: a warp per vertex (k_floyd_warp; its shared memory is
    // small enough for ~30 warps per SM: cfg3 3.9 vs 5.2 ms for k_floyd_bloom); larger
    // draws keep k_floyd_bloom (cfg4 52 vs 51 ms, cfg5 335 vs 322 ms:
    // profiles/r02_floyd_warp_r_sweep.jsonl).  SNGB_FLOYD_WARP=0 never, 1 always.
    const char* fwenv = std::getenv("SNGB_FLOYD_WARP");
    const int fwmode = fwenv ? std::atoi(fwenv) : 2;
    if (D <= 4096 && a.n - 2 < 0xffffffffull && a.scratch64 && !std::getenv("SNGB_FLOYD_BLOOM") &&
        (fwmode == 1 || (fwmode == 2 && D <= 1024))) {
        const FwGeom fg = fw_geometry(D);
        const size_t smem = fg.warp_bytes();
        auto k = D <= 1024 ? k_floyd_warp<4> : k_floyd_warp<SNGB_FW_R>;
        cudaError_t e = raise_smem_limit(reinterpret_cast<const void*>(k));
        if (e != cudaSuccess) return e;
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 32, smem);
        if (per_sm < 1) per_sm = 1;
        if (const char* ev = std::getenv("SNGB_SAMPLER_BPSM"))
            if (std::atoi(ev) > 0 && std::atoi(ev) < per_sm) per_sm = std::atoi(ev);
        const uint64_t cap = (uint64_t)num_sms * per_sm;
        const unsigned grid = a.rows_per_block
                                  ? (unsigned)((rows + a.rows_per_block - 1) / a.rows_per_block)
                                  : (unsigned)(rows < cap ? rows : cap);
        k<<<grid, 32, smem, s>>>(a, fg);
        note_launch(1);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        uint32_t cap_slots = 1;
        while (cap_slots < 2 * D + 2) cap_slots <<= 1;
        e = raise_smem_limit(reinterpret_cast<const void*>(k_replay_list));
        if (e != cudaSuccess) return e;
        k_replay_list<<<num_sms * 8, 32, (size_t)cap_slots * 4, s>>>(
            a, reinterpret_cast<const uint32_t*>(a.scratch64), cap_slots);
        note_launch(1);
        return cudaGetLastError();
    }
    // large n, draws <= 4096: filter + exact resolution of the few shared bits
    if (D <= 4096 && a.n - 2 < 0xffffffffull) {
        const BloomGeom bg = bloom_geometry(D);
        a.hash_mask = bg.words;
        a.key_bits = bg.bits_log2;
        a.col_words = bg.col_words;
        const size_t smem = bloom_smem_bytes(bg);
        // draws per worker thread = ceil(D / 256), every slot computed.  Above
        // 1024 draws k_floyd_lean (same tables and resolver, ~half the worker
        // instructions); SNGB_FLOYD_LEAN=0 keeps k_floyd_bloom for A/B runs.
        const char* lenv = std::getenv("SNGB_FLOYD_LEAN");
        const bool lean = D > 1024 && !(lenv && std::atoi(lenv) == 0);
        using KFn = void (*)(const SamplerArgs);
        static constexpr KFn kLean[12] = {k_floyd_lean<5>,  k_floyd_lean<6>,  k_floyd_lean<7>,
                                          k_floyd_lean<8>,  k_floyd_lean<9>,  k_floyd_lean<10>,
                                          k_floyd_lean<11>, k_floyd_lean<12>, k_floyd_lean<13>,
                                          k_floyd_lean<14>, k_floyd_lean<15>, k_floyd_lean<16>};
        // k_floyd_pipe: k_floyd_lean's workers resolve their own group entries,
        // pipelined over the vertex loop (no resolver warp); SNGB_FLOYD_PIPE=0|1
        const bool pipe = pipe_wanted(D) || a.tbuf;  // shared draws: k_floyd_pipe reads them
        if (pipe) {
            static constexpr KFn kPipe[12] = {
                k_floyd_pipe<5, false>,  k_floyd_pipe<6, false>,  k_floyd_pipe<7, false>,
                k_floyd_pipe<8, false>,  k_floyd_pipe<9, false>,  k_floyd_pipe<10, false>,
                k_floyd_pipe<11, false>, k_floyd_pipe<12, false>, k_floyd_pipe<13, false>,
                k_floyd_pipe<14, false>, k_floyd_pipe<15, false>, k_floyd_pipe<16, false>};
#if SNGB_SHARE_DRAWS
            static constexpr KFn kPipeT[12] = {
                k_floyd_pipe<5, true>,  k_floyd_pipe<6, true>,  k_floyd_pipe<7, true>,
                k_floyd_pipe<8, true>,  k_floyd_pipe<9, true>,  k_floyd_pipe<10, true>,
                k_floyd_pipe<11, true>, k_floyd_pipe<12, true>, k_floyd_pipe<13, true>,
                k_floyd_pipe<14, true>, k_floyd_pipe<15, true>, k_floyd_pipe<16, true>};
            KFn kp = (a.tbuf ? kPipeT : kPipe)[(D + kBloomThreads - 1) / kBloomThreads - 5];
#else
            if (a.tbuf) return cudaErrorInvalidValue;  // built without the shared-draws kernels
            KFn kp = kPipe[(D + kBloomThreads - 1) / kBloomThreads - 5];
#endif
            const size_t psmem = pipe_smem_bytes(bg);
            cudaError_t e = raise_smem_limit(reinterpret_cast<const void*>(kp));
            if (e != cudaSuccess) return e;
            int per_sm = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kp, kBloomThreads, psmem);
            if (per_sm < 1) per_sm = 1;
            if (const char* ev = std::getenv("SNGB_SAMPLER_BPSM"))
                if (std::atoi(ev) > 0 && std::atoi(ev) < per_sm) per_sm = std::atoi(ev);
            const uint64_t cap = (uint64_t)num_sms * per_sm;
            const unsigned grid = a.rows_per_block
                                      ? (unsigned)((rows + a.rows_per_block - 1) / a.rows_per_block)
                                      : (unsigned)(rows < cap ? rows : cap);
            kp<<<grid, kBloomThreads, psmem, s>>>(a);
            note_launch(1);
            return cudaGetLastError();
        }
        KFn k = lean ? kLean[(D + kBloomThreads - 1) / kBloomThreads - 5]
                : D <= 768    ? k_floyd_bloom<3>
                : D <= 1024   ? k_floyd_bloom<4>
                : D <= 2048   ? k_floyd_bloom<8>
                : D <= 2560   ? k_floyd_bloom<10>
                : D <= 3072   ? k_floyd_bloom<12>
                              : k_floyd_bloom<16>;
        cudaError_t e = raise_smem_limit(reinterpret_cast<const void*>(k));
        if (e != cudaSuccess) return e;
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kBloomBlock, smem);
        if (per_sm < 1) per_sm = 1;
        // SNGB_SAMPLER_BPSM: cap the persistent grid (co-residency with the gather)
        if (const char* e = std::getenv("SNGB_SAMPLER_BPSM"))
            if (std::atoi(e) > 0 && std::atoi(e) < per_sm) per_sm = std::atoi(e);
        const uint64_t cap = (uint64_t)num_sms * per_sm;
        const unsigned grid = a.rows_per_block
                                  ? (unsigned)((rows + a.rows_per_block - 1) / a.rows_per_block)
                                  : (unsigned)(rows < cap ? rows : cap);
        k<<<grid, kBloomBlock, smem, s>>>(a);
        note_launch(1);
        return cudaGetLastError();
    }
    // generic path: 64-bit (t, first index) entries, any draws
    uint32_t slots, cw64;
    floyd_geometry(D, slots, cw64);
    a.hash_mask = slots / 4 - 1;
    a.hash_shift = 32 - __builtin_ctz(slots / 4);
    a.col_words = cw64;
    const bool sh = floyd_shared(D);
    const size_t smem = floyd_smem_bytes(D, sh);
    auto k = sh ? k_floyd<true> : k_floyd<false>;
    cudaError_t e = raise_smem_limit(reinterpret_cast<const void*>(k));
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kFloydThreads, smem);
    if (per_sm < 1) per_sm = 1;
    if (!sh) per_sm = 2;  // scratch holds num_sms * 2 tables
    const uint64_t cap = (uint64_t)num_sms * per_sm;
    k<<<(unsigned)(rows < cap ? rows : cap), kFloydThreads, smem, s>>>(a);
    note_launch(1);
    return cudaGetLastError();
}

}  // namespace sngb
