// sngb_fused.cu -- k_sample_head: the Floyd bookkeeping (graph.cpp:161-174) and
// the head-filter gather (sngb_head.cu) of large narrow-row problems in one
// kernel, one warp per vertex, each draw generated once (cfg3, cfg4, cfg5).
//
// Why.  As two kernels (k_floyd_bloom + k_gather_head) each draw
//   t_i = Lemire(mix(key + (i+1) gamma), base + i + 1)   (rng.hpp:26,35-48)
// is generated twice and costs ~100 SASS instructions in each (ncu:
// profiles/r02_ncu_floyd_cfg5.md, r01_ncu_head_cfg5.md).  Earlier fusions:
// v3 block per vertex (barriers: 831 ms on cfg5), v4 one pass with the draws
// in global scratch (318 GB of write-back: 978 ms), v6 two regenerating passes
// (5.2 warp-instructions per draw: 750 ms), against 654 ms for the two kernels.
// Here a warp owns a vertex and keeps only each draw's 16-bit filter hash in
// shared memory (D x 2 bytes), so the one pass over the draws does everything:
//
//   P1  draw i (lane i mod 32, R slots per step): t_i; a running test of the
//       Lemire reject pre-condition (rng.hpp:43, ~1e-12 per draw) that cuts
//       the vertex at its first fired draw; the partner's head load (exact
//       reject, sngb_head.cu) and survivors' fp32 test (sngb_epstest.cuh);
//       h_i = hash(t_i) -> HS[i]; OR bit h_i into a warp-private 2^B-bit filter
//       F -- a draw finding its bit already set records h_i in its lane's
//       second-comer list SL; t_i in [base, base + i) -> the lane's chain list.
//   P2  F := the bits in SL (exactly the bits hit by >= 2 draws); scan HS: the
//       draws on such a bit -> the lane's group list GL (indices, SL's slots).
//   R   GL's values (regenerated: ~6 % of the draws) in a small hash (F's
//       memory) keyed by t with the minimum index: a draw whose value has a
//       smaller index collides (graph.cpp:168-169: its replacement
//       j_i = base + i is inserted instead); then the chain candidates in index
//       order against the collided set.  Every collided draw's replacement is
//       emitted as an extra pair (tested by k_extras).
// A fired draw or a list overflow sends the vertex to the exact sequential
// replay (k_replay_list: true Stream semantics, every partner an extra); its
// gather stops at the first fired draw, as k_gather_head's does.  Results are
// the two-kernel path's bit for bit (tests/test_gpu_parity.py -k "fused or head").
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "sngb_device.cuh"
#include "sngb_epstest.cuh"
#include "sngb_head.cuh"
#include "sngb_gather_head.cuh"
#include "sngb_internal.cuh"
#include "sngb_rng.cuh"

#ifndef SNGB_FUSED_MINB
#define SNGB_FUSED_MINB 8
#endif
#ifndef SNGB_FUSED_R
#define SNGB_FUSED_R 8
#endif

namespace sngb {

namespace {

#include "sngb_floyd_bloom.cuh"
#include "sngb_floyd_warp.cuh"
#include "sngb_floyd_lean.cuh"
#include "sngb_floyd_head.cuh"
#include "sngb_floyd_pipe.cuh"
#include "sngb_floyd_headpipe.cuh"

constexpr int kFStage = 64;  // edge staging per warp (accepts are rare here)

__host__ __device__ inline uint32_t fused_q_cap(int R, int step) { return ((32 * R + step) + 3) & ~3u; }
__host__ __device__ inline uint32_t fused_warp_bytes(const FwGeom& fg, int R, int step) {
    return fg.warp_bytes() + fused_q_cap(R, step) * 4 + kFStage * 8;
}

template <int KIND, int G, int V, int R>
__global__ void __launch_bounds__(32, 8)
    k_sample_head(const SamplerArgs a, const GatherArgs g, const HeadArgs h, const FwGeom fg) {
    constexpr int NG = 32 / G;
    constexpr int UF = 2;            // fp32 rows per group per step
    constexpr int STEP = NG * UF;    // survivors per fp32 step
    constexpr uint32_t ITER = 32 * R;
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t lane = threadIdx.x & 31;
    const int q = lane % G, grp = lane / G;
    const bool leader = (q == 0);
    const uint32_t D = a.draws, base = a.base;
    const uint32_t shift = 32 - fg.B, FW = fg.FW;

    // the warp's shared memory (one warp per block): k_floyd_warp's layout + queue + stage
    uint32_t* F = reinterpret_cast<uint32_t*>(smem);
    uint16_t* HS = reinterpret_cast<uint16_t*>(F + FW);
    uint16_t* SL = HS + 2 * fg.hs_words;  // [32][kFwSLL]
    uint16_t* CLs = SL + 32 * kFwSLL;     // [32][kFwCLL]
    uint32_t* Q = reinterpret_cast<uint32_t*>(CLs + 32 * kFwCLL);
    unsigned long long* stg = reinterpret_cast<unsigned long long*>(Q + fused_q_cap(R, STEP));
    const uint32_t Fa = smem_addr(F), HSa = smem_addr(HS), Qa = smem_addr(Q);
    const uint32_t SLa = smem_addr(SL + lane * kFwSLL), CLa = smem_addr(CLs + lane * kFwCLL);
    uint16_t* myCL = CLs + lane * kFwCLL;
    uint32_t* irr_list = reinterpret_cast<uint32_t*>(a.scratch64);  // the replay list

    const float4* __restrict__ P = reinterpret_cast<const float4*>(g.tp.pts);
    const void* __restrict__ H = h.head;
    const uint32_t W = g.tp.stride / 4;
    const float reject = h.reject;
    const uint64_t pol = evict_first_policy();  // survivor rows must not evict the heads

    WarpStage<kFStage> stage{stg, 0};
    TestStats st;
    unsigned long long gpairs = 0, tails = 0, ncol = 0;
    for (int j = 0; j < kFwCLL; ++j) myCL[j] = 0;  // chain lists start empty (0 = no entry)

    uint64_t u = 0, chunk_end = 0;
    auto grab = [&]() {
        unsigned long long b0 = 0;
        if (lane == 0) b0 = atomicAdd(g.work, (unsigned long long)g.grab);
        b0 = __shfl_sync(kFull, b0, 0);
        u = a.row_begin + b0;
        chunk_end = u + g.grab < a.row_end ? u + g.grab : a.row_end;
    };
    grab();
    for (; u < chunk_end; (u + 1 >= chunk_end) ? grab() : (void)(++u)) {
        F4x2 qv[V];
#pragma unroll
        for (int vv = 0; vv < V; ++vv) {
            const uint32_t c = q + G * vv;
            qv[vv] = to_x2(ldg_row(P + u * W + (c < W ? c : W - 1)));
        }
        const uint32_t hq = head_load<KIND>(H, (uint32_t)u);
        const uint64_t key = vertex_key(a.seed_mixed, u);
        for (uint32_t w = lane; w < FW / 4; w += 32) st_sh_zero16(Fa + 16 * w);
        __syncwarp();

        // fp32 test of queue entries [e0, e0 + STEP) of which those < qend are real
        auto fp32_step = [&](uint32_t e0, uint32_t qend) {
            F4x2 rows[UF][V];
            uint32_t pe[UF];
            bool oke[UF];
#pragma unroll
            for (int uu = 0; uu < UF; ++uu) {
                const uint32_t e = e0 + grp + NG * uu;
                oke[uu] = e < qend;
                pe[uu] = ld_sh(Qa + 4 * (oke[uu] ? e : e0));
#pragma unroll
                for (int vv = 0; vv < V; ++vv) {
                    const uint32_t c = q + G * vv;
                    const uint64_t row = (oke[uu] && c < W) ? pe[uu] : u;
                    rows[uu][vv] = ldg_row2_ef(P + row * W + (c < W ? c : W - 1), pol);
                }
            }
            __syncwarp();
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
        };

        // ---- P1: every draw once (test hook: a hooked vertex fires at draw D/2) ----
        uint32_t limit = (a.force_mod != 0 && (u % a.force_mod) == 0) ? D / 2 : D;
        bool replay = limit < D;
        uint32_t qn = 0, nsl = 0, ncl = 0;
        // one step of R slots; TAIL masks the draws >= limit.  Returns true when a
        // draw of this step fired (limit cut): the step is then redone as a tail.
        auto step = [&](uint32_t i0, uint64_t z, auto tail_c) -> bool {
            constexpr bool TAIL = decltype(tail_c)::value;
            const uint32_t b0 = base + i0 + lane + 1;  // Lemire bound of slot 0
            uint32_t tv[R], mn = 0xffffffffu;
#pragma unroll
            for (int k = 0; k < R; ++k) {
                uint32_t slo;
                tv[k] = lemire32_slo(mix(z + (uint64_t)(32 * k) * kGamma), b0 + 32 * k, slo);
                const bool valid = !TAIL || i0 + 32 * k + lane < limit;
                mn = valid ? min(mn, slo) : mn;
            }
            if (__any_sync(kFull, mn == 0u)) {  // rare: the exact pre-condition, first fired draw
                uint32_t f = limit;
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    bool fire;
                    (void)lemire32(mix(z + (uint64_t)(32 * k) * kGamma), b0 + 32 * k, fire);
                    const uint32_t i = i0 + 32 * k + lane;
                    if (fire && i < f) f = i;
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) f = min(f, __shfl_xor_sync(kFull, f, o));
                if (f < limit) {
                    limit = f;
                    replay = true;
                    if (!TAIL) return true;  // redo this step as a tail
                }
            }
            uint32_t pv[R];
#pragma unroll
            for (int k = 0; k < R; ++k) {
                const uint32_t i = i0 + 32 * k + lane;
                const uint32_t p = tv[k] + (tv[k] >= (uint32_t)u ? 1u : 0u);
                pv[k] = (!TAIL || i < limit) ? p : (uint32_t)u;
            }
            uint32_t hb[R];
#pragma unroll
            for (int k = 0; k < R; ++k) hb[k] = head_load<KIND>(H, pv[k]);  // in flight from here
            if (!replay) {  // the Floyd bookkeeping (skipped once the vertex will be replayed)
                uint32_t hk[R], old[R];
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    const uint32_t i = i0 + 32 * k + lane;
                    hk[k] = (tv[k] * 0x9E3779B1u) >> shift;
                    if (TAIL) st_sh_u16_if(HSa + 2 * i, hk[k], i < limit);
                    else st_sh_u16(HSa + 2 * i, hk[k]);
                }
#pragma unroll
                for (int k = 0; k < R; ++k) {  // all R atomics in flight before any result is used
                    const uint32_t i = i0 + 32 * k + lane;
                    const uint32_t addr = Fa + ((hk[k] >> 5) << 2), bit = 1u << (hk[k] & 31);
                    old[k] = TAIL ? atom_or_sh_if(addr, bit, i < limit) : atom_or_sh(addr, bit);
                }
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    const uint32_t i = i0 + 32 * k + lane;
                    const bool sec = (old[k] >> (hk[k] & 31)) & 1u;  // a second comer (0 if masked)
                    st_sh_u16_if(SLa + 2 * min(nsl, (uint32_t)kFwSLL - 1), hk[k], sec);
                    nsl += sec ? 1u : 0u;
                    const bool ch = (!TAIL || i < limit) && tv[k] - base < i;  // t <= base + i
                    st_sh_u16_if(CLa + 2 * min(ncl, (uint32_t)kFwCLL - 1), i, ch);
                    ncl += ch ? 1u : 0u;
                }
            }
#pragma unroll
            for (int k = 0; k < R; ++k) {
                const uint32_t i = i0 + 32 * k + lane;
                const bool keep = (!TAIL || i < limit) && !(head_q<KIND>(hq, hb[k]) > reject);
                const unsigned km = __ballot_sync(kFull, keep);
                if (keep) st_sh(Qa + 4 * (qn + __popc(km & lanemask_lt())), pv[k]);
                qn += __popc(km);
            }
            __syncwarp();
            if (qn >= (uint32_t)STEP) {
                uint32_t e0 = 0;
#pragma unroll 1
                for (; e0 + STEP <= qn; e0 += STEP) fp32_step(e0, qn);
                const uint32_t rem = qn - e0;  // < STEP: move them to the front
                const uint32_t mp = lane < rem ? ld_sh(Qa + 4 * (e0 + lane)) : 0u;
                __syncwarp();
                if (lane < rem) st_sh(Qa + 4 * lane, mp);
                qn = rem;
                __syncwarp();
            }
            return false;
        };
        {
            uint64_t z = key + (uint64_t)(lane + 1) * kGamma;
            uint32_t i0 = 0;
            for (; i0 + ITER <= limit; i0 += ITER, z += (uint64_t)ITER * kGamma)
                if (step(i0, z, std::false_type{})) break;  // fired: redo as the tail below
            if (i0 < limit) step(i0, z, std::true_type{});
        }
        if (qn) fp32_step(0, qn);
        if (lane == 0) gpairs += limit;

        // ---- P2 + R: the collided draws (k_floyd_warp's resolution) ----
        replay = replay || __any_sync(kFull, nsl > (uint32_t)kFwSLL || ncl > (uint32_t)kFwCLL);
        __syncwarp();
        fw_resolve(a, fg, u, key, F, HS, SL, CLs, nsl, ncl, replay, ncol);
        for (int j = 0; j < kFwCLL; ++j) myCL[j] = 0;
        if (replay && lane == 0) {
            const unsigned long long s2 = atomicAdd(&a.counters[C_IRR_CURSOR], 1ull);
            irr_list[s2] = (uint32_t)u;  // capacity: one slot per row
        }
        __syncwarp();
    }
    stage.flush(g.sink, lane);
    st.pairs = gpairs;
    flush_stats(st, gpairs, g.counters, lane);
    const unsigned long long tw = warp_sum(tails);
    if (lane == 0 && tw) atomicAdd(&g.counters[C_TAIL_PAIRS], tw);
    ncol = warp_sum(ncol);
    if (lane == 0 && ncol) atomicAdd(&a.counters[C_COLLISIONS], ncol);
}

template <int KIND, int G, int V>
cudaError_t fused_one(SamplerArgs a, GatherArgs ga, const HeadArgs& h, cudaStream_t s,
                      int num_sms) {
    constexpr int R = SNGB_FUSED_R;
    constexpr int STEP = (32 / G) * 2;
    auto k = k_sample_head<KIND, G, V, R>;
    const FwGeom fg = fw_geometry(a.draws);
    const size_t smem = fused_warp_bytes(fg, R, STEP);  // one warp per block
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 32, smem);
    if (per_sm < 1) per_sm = 1;
    const uint64_t rows = a.row_end - a.row_begin;
    const uint64_t cap = (uint64_t)num_sms * per_sm;
    const unsigned grid = (unsigned)(rows < cap ? rows : cap);
    ga.grab = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(32, rows / ((uint64_t)grid * 16)));
    k<<<grid, 32, smem, s>>>(a, ga, h, fg);
    note_launch(1);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    // the listed vertices' exact replays (usually none: one small launch)
    uint32_t cap_slots = 1;
    while (cap_slots < 2 * a.draws + 2) cap_slots <<= 1;
    const size_t rsmem = (size_t)cap_slots * 4;
    e = cudaFuncSetAttribute(k_replay_list, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsmem);
    if (e != cudaSuccess) return e;
    k_replay_list<<<num_sms * 8, 32, rsmem, s>>>(a, reinterpret_cast<const uint32_t*>(a.scratch64),
                                                 cap_slots);
    note_launch(1);
    return cudaGetLastError();
}

template <int KIND>
cudaError_t fused_kind(const SamplerArgs& sa, const GatherArgs& ga, const HeadArgs& h,
                       cudaStream_t s, int num_sms) {
    const uint32_t W = ga.tp.stride / 4;
    if (W <= 2) return fused_one<KIND, 2, 1>(sa, ga, h, s, num_sms);
    if (W <= 4) return fused_one<KIND, 4, 1>(sa, ga, h, s, num_sms);
    if (W <= 8) return fused_one<KIND, 8, 1>(sa, ga, h, s, num_sms);
    if (W <= 16) return fused_one<KIND, 16, 1>(sa, ga, h, s, num_sms);
    if (W <= 32) return fused_one<KIND, 32, 1>(sa, ga, h, s, num_sms);
    return cudaErrorInvalidValue;
}

// k_floyd_head (sngb_floyd_head.cuh): block per vertex, draws 1024 < D <= 4096
template <int KIND, int G, int V>
cudaError_t fh_one(SamplerArgs a, const GatherArgs& ga, const HeadArgs& h, cudaStream_t s,
                   int num_sms) {
    const BloomGeom bg = bloom_geometry(a.draws);
    a.hash_mask = bg.words;
    a.key_bits = bg.bits_log2;
    a.col_words = bg.col_words;
    const uint32_t scap = (a.draws + 3) & ~3u;  // every draw may survive the head
    const size_t smem = fh_smem_bytes(bg, scap);
    auto k = k_floyd_head<KIND, G, V>;
    // the opt-in maximum, never lowered under a concurrent caller's launch
    int dev = 0, mx = 0;
    cudaGetDevice(&dev);
    cudaError_t e = cudaDeviceGetAttribute(&mx, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa{};
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, k);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, mx - (int)fa.sharedSizeBytes);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kFhBlock, smem);
    if (per_sm < 1) per_sm = 1;
    const uint64_t rows = a.row_end - a.row_begin;
    const uint64_t cap = (uint64_t)num_sms * per_sm;
    k<<<(unsigned)(rows < cap ? rows : cap), kFhBlock, smem, s>>>(a, ga, h, scap);
    note_launch(1);
    return cudaGetLastError();
}

template <int KIND>
cudaError_t fh_kind(const SamplerArgs& sa, const GatherArgs& ga, const HeadArgs& h,
                    cudaStream_t s, int num_sms) {
    // the testers' row shape: one or two lanes per survivor row, so a warp has
    // 32-256 rows in flight and reduces with at most one shuffle
    const uint32_t W = ga.tp.stride / 4;
    if (W <= 1) return fh_one<KIND, 1, 1>(sa, ga, h, s, num_sms);
    if (W <= 2) return fh_one<KIND, 1, 2>(sa, ga, h, s, num_sms);
    if (W <= 4) return fh_one<KIND, 1, 4>(sa, ga, h, s, num_sms);
    return fh_one<KIND, 2, 4>(sa, ga, h, s, num_sms);
}

// ---- k_duo: the Floyd bookkeeping (floyd_pipe_run) and the head gather
// (gather_head_body) as two roles of ONE launch, so both are resident on every
// SM for the whole step.  As two launches the gather's persistent blocks fill
// the register file and the sampler only runs in its drain; yet the two bodies
// lean on different units -- the gather on the L1TEX tag stage (one random head
// per SM-cycle, issue 63 %), the Floyd workers on the issue slots and the
// shared-memory data stage -- so side by side they overlap.  Blocks start in
// the role their index picks (half and half per SM under breadth-first block
// placement), claim work dynamically (gather: ga.work rows; Floyd: fwork chunks
// of fgrab consecutive vertices) and switch role when their queue is empty.
// Every draw is still generated twice; the results are those of the two kernels.
template <int KIND, int G, int V, int R, int MAXR>
__global__ void __launch_bounds__(kBloomThreads, 4)
    k_duo(const SamplerArgs sa, const GatherArgs ga, const HeadArgs h, unsigned long long* fwork,
          uint32_t fgrab, uint32_t split) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ unsigned long long s_c0;
    const bool floyd_first = split ? ((blockIdx.x / split) & 1u) != 0 : (blockIdx.x & 1u) != 0;
    const uint64_t rows = sa.row_end - sa.row_begin;
    for (int pass = 0; pass < 2; ++pass) {
        if ((pass == 0) == floyd_first) {
            for (;;) {
                if (threadIdx.x == 0) s_c0 = atomicAdd(fwork, (unsigned long long)fgrab);
                __syncthreads();
                const unsigned long long c0 = s_c0;
                __syncthreads();
                if (c0 >= rows) break;
                const uint32_t nv = (uint32_t)(rows - c0 < fgrab ? rows - c0 : fgrab);
                floyd_pipe_run<MAXR>(sa, smem, sa.row_begin + c0, 1, nv);
            }
        } else {
            unsigned long long* stage_mem = reinterpret_cast<unsigned long long*>(smem);
            uint32_t* queue_mem =
                reinterpret_cast<uint32_t*>(smem + (size_t)kWarpsPerBlock * kStage * 8);
            gather_head_body<KIND, G, V, R>(ga, h, stage_mem, queue_mem);
        }
        __syncthreads();
    }
}

template <int KIND, int G, int MAXR>
cudaError_t duo_one(SamplerArgs a, GatherArgs ga, const HeadArgs& h, cudaStream_t s, int num_sms) {
    constexpr int R = SNGB_HEAD_R;
    const BloomGeom bg = bloom_geometry(a.draws);
    a.hash_mask = bg.words;
    a.key_bits = bg.bits_log2;
    a.col_words = bg.col_words;
    const size_t gsmem = (size_t)kWarpsPerBlock * (kStage * 8 + gather_head_qcap<G, R>() * 4);
    const size_t smem = std::max(pipe_smem_bytes(bg), gsmem);
    auto k = k_duo<KIND, G, 1, R, MAXR>;
    int dev = 0, mx = 0;
    cudaGetDevice(&dev);
    cudaError_t e = cudaDeviceGetAttribute(&mx, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa{};
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, k);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, mx - (int)fa.sharedSizeBytes);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kBloomThreads, smem);
    if (per_sm < 1) per_sm = 1;
    const uint64_t rows = a.row_end - a.row_begin;
    // gather: ~16 claims per resident warp, at most 32 rows per claim (as launch_gather_head's caller)
    const uint64_t warps = (uint64_t)num_sms * 64;
    ga.grab = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(32, rows / (warps * 16)));
    const char* ge = std::getenv("SNGB_DUO_GRAB");
    const uint32_t fgrab = ge && std::atoi(ge) > 0 ? (uint32_t)std::atoi(ge) : 64u;
    const char* se = std::getenv("SNGB_DUO_SPLIT");  // 0: roles alternate by block index
    const uint32_t split = se ? (uint32_t)std::atoi(se) : (uint32_t)num_sms;
    k<<<(unsigned)(num_sms * per_sm), kBloomThreads, smem, s>>>(a, ga, h, ga.work + 1, fgrab, split);
    note_launch(1);
    return cudaGetLastError();
}

// the shapes instantiated: cfg4's (16-byte rows, 2500 draws) and cfg5's (128-byte
// rows, 4000 draws); others keep the two kernels
bool duo_shape(uint32_t draws, uint32_t stride) {
    const uint32_t W = stride / 4, maxr = (draws + kBloomThreads - 1) / kBloomThreads;
    return (W <= 2 && maxr == 10) || (W > 4 && W <= 8 && maxr == 16);
}

template <int KIND>
cudaError_t duo_kind(const SamplerArgs& sa, const GatherArgs& ga, const HeadArgs& h,
                     cudaStream_t s, int num_sms) {
    if (ga.tp.stride / 4 <= 2) return duo_one<KIND, 2, 10>(sa, ga, h, s, num_sms);
    return duo_one<KIND, 8, 16>(sa, ga, h, s, num_sms);
}

// k_floyd_headpipe (sngb_floyd_headpipe.cuh): the workers of k_floyd_pipe also take
// the head test and the survivors' fp32 test; one RNG pass
template <int KIND, int G, int MAXR>
cudaError_t fhp_one(SamplerArgs a, const GatherArgs& ga, const HeadArgs& h, cudaStream_t s,
                    int num_sms) {
    const BloomGeom bg = bloom_geometry(a.draws);
    a.hash_mask = bg.words;
    a.key_bits = bg.bits_log2;
    a.col_words = bg.col_words;
    const size_t smem = fhp_smem_bytes(bg);
    auto k = k_floyd_headpipe<KIND, G, MAXR>;
    int dev = 0, mx = 0;
    cudaGetDevice(&dev);
    cudaError_t e = cudaDeviceGetAttribute(&mx, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa{};
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, k);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, mx - (int)fa.sharedSizeBytes);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kBloomThreads, smem);
    if (per_sm < 1) per_sm = 1;
    const char* ge = std::getenv("SNGB_FHP_GRAB");
    const uint32_t grab = ge && std::atoi(ge) > 0 ? (uint32_t)std::atoi(ge) : 64u;
    const uint64_t rows = a.row_end - a.row_begin;
    const uint64_t want = (rows + grab - 1) / grab, cap = (uint64_t)num_sms * per_sm;
    k<<<(unsigned)(want < cap ? want : cap), kBloomThreads, smem, s>>>(a, ga, h, grab);
    note_launch(1);
    return cudaGetLastError();
}

template <int KIND>
cudaError_t fhp_kind(const SamplerArgs& sa, const GatherArgs& ga, const HeadArgs& h,
                     cudaStream_t s, int num_sms) {
    if (ga.tp.stride / 4 <= 2) return fhp_one<KIND, 2, 10>(sa, ga, h, s, num_sms);
    return fhp_one<KIND, 8, 16>(sa, ga, h, s, num_sms);
}

bool fh_eligible(uint32_t draws, uint32_t stride) {
    const char* e = std::getenv("SNGB_FH");
    return draws > 1024 && draws <= 4096 && stride / 4 <= 8 && !(e && std::atoi(e) == 0);
}

}  // namespace

#ifndef SNGB_FUSED_DEFAULT
#define SNGB_FUSED_DEFAULT 0
#endif
constexpr int kFusedDefault = SNGB_FUSED_DEFAULT;

bool fused_eligible(uint64_t n, uint32_t draws, uint32_t stride) {
    // SNGB_FUSED=0 keeps the two kernels, 1 fuses every eligible shape, 2 (auto)
    // also needs few chain candidates per vertex (about draws^2 / 2n <= 4: they
    // are resolved sequentially by one lane).  Eligible wherever launch_sampler
    // would pick k_floyd_bloom (n beyond the per-warp bitmap kernel's 73 k, or
    // SNGB_FLOYD_NO_BITMAP; draws <= 4096) for rows of <= 32 float4.
    const char* e = std::getenv("SNGB_FUSED");
    const int mode = e ? std::atoi(e) : kFusedDefault;
    if (mode == 0 || draws < 1 || draws > 4096 || n - 2 >= 0xffffffffull || stride / 4 > 32)
        return false;
    if (mode == 2 && (uint64_t)draws * draws > 8 * n) return false;
    if ((mode == 3 || mode == 4) && !duo_shape(draws, stride))
        return false;  // k_duo / k_floyd_headpipe: two shapes instantiated
    const uint64_t bm_words = (((n - 1) + 31) / 32 + 3) & ~3ull;
    return bm_words * 4 > 9216 || std::getenv("SNGB_FLOYD_NO_BITMAP") != nullptr;
}

size_t fused_scratch_bytes(uint32_t draws, uint64_t rows, int num_sms) {
    (void)draws;
    (void)num_sms;
    return rows * 4;  // the replay list: at most one entry per row
}

cudaError_t launch_floyd_head(const SamplerArgs& in, const GatherArgs& ga, const HeadArgs& h,
                              cudaStream_t s, int num_sms) {
    const uint64_t rows = in.row_end - in.row_begin;
    if (rows == 0 || in.draws == 0) return cudaSuccess;
    {
        const char* fe = std::getenv("SNGB_FUSED");
        if ((fe ? std::atoi(fe) : kFusedDefault) == 4) {  // one RNG pass, the workers do it all
            if (!ga.work || !duo_shape(in.draws, ga.tp.stride)) return cudaErrorInvalidValue;
            switch (h.kind) {
                case kHeadU16x2: return fhp_kind<kHeadU16x2>(in, ga, h, s, num_sms);
                case kHeadU8x4: return fhp_kind<kHeadU8x4>(in, ga, h, s, num_sms);
                default: return fhp_kind<kHeadU8x2>(in, ga, h, s, num_sms);
            }
        }
        if ((fe ? std::atoi(fe) : kFusedDefault) == 3) {  // the two kernels as roles of one launch
            if (!ga.work || !duo_shape(in.draws, ga.tp.stride)) return cudaErrorInvalidValue;
            switch (h.kind) {
                case kHeadU16x2: return duo_kind<kHeadU16x2>(in, ga, h, s, num_sms);
                case kHeadU8x4: return duo_kind<kHeadU8x4>(in, ga, h, s, num_sms);
                default: return duo_kind<kHeadU8x2>(in, ga, h, s, num_sms);
            }
        }
    }
    if (fh_eligible(in.draws, ga.tp.stride)) {  // block per vertex, survivors off the workers' path
        switch (h.kind) {
            case kHeadU16x2: return fh_kind<kHeadU16x2>(in, ga, h, s, num_sms);
            case kHeadU8x4: return fh_kind<kHeadU8x4>(in, ga, h, s, num_sms);
            default: return fh_kind<kHeadU8x2>(in, ga, h, s, num_sms);
        }
    }
    if (!ga.work || !in.scratch64) return cudaErrorInvalidValue;  // zeroed counter, scratch
    switch (h.kind) {
        case kHeadU16x2: return fused_kind<kHeadU16x2>(in, ga, h, s, num_sms);
        case kHeadU8x4: return fused_kind<kHeadU8x4>(in, ga, h, s, num_sms);
        default: return fused_kind<kHeadU8x2>(in, ga, h, s, num_sms);
    }
}

}  // namespace sngb
