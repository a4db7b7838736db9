// sngb_head.cu -- the head filter for narrow rows that do not stay in L2: an
// exact early reject on a compact, L2-resident copy of each row's first two
// coordinates, so most sampled pairs never touch the fp32 table in HBM.
//
// Why.  A random row from HBM costs one DRAM access whether it is 16, 32, 64
// or 128 bytes wide (measured on B200, tools/gather_ceiling.cu: 6.3e10, 4.9e10,
// 4.2e10 and 4.2e10 random rows/s), so on a table like cfg5's (20 M x 128 B =
// 2.56 GB) fewer bytes per row buy nothing -- only a table that fits the 126 MB
// L2 does.  Two 16-bit coordinates per row is 4 bytes (cfg5: 80 MB).
//
// Quantisation (host plan, head_plan).  s is a power of two >= (max - min)/65534
// over all values and lo' = floor(min/s)*s, so q = rint((a - lo')/s) fits 16 bits
// and |a - (lo' + s q)| <= s/2 (1 + 2^-30) (the fp64 evaluation, as in
// sngb_quant.cu).  For a pair and s' = s(1 + 2^-30), per coordinate
// |(a_j - b_j) - s(qa_j - qb_j)| <= s', hence over the two head coordinates
// (triangle inequality)  |a_h - b_h| >= s*sqrt(Q) - s'*sqrt(2),  Q = sum_h dq^2,
// and the full squared distance S >= |a_h - b_h|^2.  So
//     Q > B = ((sqrt(eps2 (1 + 2^-40)) + s' sqrt(2)) / s)^2   =>   S > eps2 (1 + 2^-40)
// and the reference's fp64 sum (within (d+1) 2^-53 S of S, distance.hpp:75-83)
// exceeds eps2: it rejects.  The kernel evaluates Q in fp32 (dq exact, two
// roundings), so it compares against B (1 + 2^-20) rounded up.  Pairs the head
// does not reject take the unchanged fp32 test (guard band, exact fp64 recheck in
// the band: sngb_epstest.cuh) on their fp32 rows.  Decisions are the reference's
// whatever the data; only the speed depends on how many pairs the head rejects
// (cfg5: ~95 %, the pairs from different clusters).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "sngb_device.cuh"
#include "sngb_epstest.cuh"
#include "sngb_internal.cuh"
#include "sngb_rng.cuh"

namespace sngb {

bool head_plan(double lo, double hi, uint32_t d, double eps2, HeadPlan& p) {
    if (d < 2) return false;
    const double need = (hi - lo) / 65534.0 * (1.0 + 1e-12);
    if (!(need > 0.0) || !std::isfinite(need)) return false;
    int e = 0;
    std::frexp(need, &e);  // need = m * 2^e, m in [0.5, 1)
    const double s = std::ldexp(1.0, e);
    p.s = s;
    p.lo = std::floor(lo / s) * s;
    const double sp = s * (1.0 + std::ldexp(1.0, -30));
    const double e_hi = eps2 * (1.0 + std::ldexp(1.0, -40));
    const double tb = (std::sqrt(e_hi) + sp * std::sqrt(2.0)) / s;
    const double b = tb * tb * (1.0 + std::ldexp(1.0, -20));
    p.args.reject = std::nextafter((float)b, INFINITY);
    // useless if the rejection radius covers the data's whole range
    return std::sqrt(b) * s < 0.5 * (hi - lo) * std::sqrt(2.0);
}

namespace {

// thread per row: the first two values of the padded fp32 row -> two u16
__global__ void k_head_quantize(const float* __restrict__ pts, uint32_t stride, uint64_t n,
                                double lo, double inv_s, uint32_t* __restrict__ out) {
    for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
         r += (uint64_t)gridDim.x * blockDim.x) {
        const float2 v = __ldg(reinterpret_cast<const float2*>(pts + r * stride));
        const double x0 = rint(((double)v.x - lo) * inv_s), x1 = rint(((double)v.y - lo) * inv_s);
        const uint32_t q0 = x0 <= 0.0 ? 0u : (x0 >= 65535.0 ? 65535u : (uint32_t)x0);
        const uint32_t q1 = x1 <= 0.0 ? 0u : (x1 >= 65535.0 ? 65535u : (uint32_t)x1);
        out[r] = q0 | (q1 << 16);
    }
}

__device__ __forceinline__ float head_q(uint32_t a, uint32_t b) {
    const float dx = (float)((int)(a & 0xffffu) - (int)(b & 0xffffu));
    const float dy = (float)((int)(a >> 16) - (int)(b >> 16));
    return __fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy));
}

// k_gather_head: one warp per query row (dynamic row claiming, as k_gather).
// Each lane owns one draw per 32-draw chunk (R chunks per step): regenerate t_i
// (counter i+1), read the partner's 4-byte head (L2), reject exactly on the
// head; survivors are queued per warp and, UF per G-lane group at a time, take
// the fp32 test on their full rows (G lanes x V float4 per row, as the narrow
// k_gather path: masked pairs and columns past the row end read the query row).
template <int G, int V, int R>
__global__ void __launch_bounds__(256, V >= 4 ? 2 : 4) k_gather_head(const GatherArgs a, const HeadArgs h) {
    constexpr int NG = 32 / G;
    constexpr int UF = 2;               // fp32 rows per group per step
    constexpr int STEP = NG * UF;       // survivors per fp32 step
    constexpr int QCAP = 32 * R + STEP;  // queue: < STEP left over + one chunk's worth
    __shared__ unsigned long long s_stage[kWarpsPerBlock][kStage];
    __shared__ uint32_t s_queue[kWarpsPerBlock][QCAP];

    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int q = lane % G, g = lane / G;
    const bool leader = (q == 0);
    const uint64_t gw = (uint64_t)blockIdx.x * kWarpsPerBlock + wib;
    const uint64_t nw = (uint64_t)gridDim.x * kWarpsPerBlock;
    const float4* __restrict__ P = reinterpret_cast<const float4*>(a.tp.pts);
    const uint32_t* __restrict__ H = h.head;
    const uint32_t W = a.tp.stride / 4;
    const uint32_t plo = a.part_lo, phi = a.part_hi;
    const float reject = h.reject;
    uint32_t* queue = s_queue[wib];

    WarpStage<kStage> stage{s_stage[wib], 0};
    TestStats st;
    unsigned long long gpairs = 0, tails = 0;

    uint64_t u = a.row_begin + gw, chunk_end = a.row_end;
    auto grab = [&]() {
        unsigned long long b0 = 0;
        if (lane == 0) b0 = atomicAdd(a.work, (unsigned long long)a.grab);
        b0 = __shfl_sync(kFull, b0, 0);
        u = a.row_begin + b0;
        chunk_end = u + a.grab < a.row_end ? u + a.grab : a.row_end;
    };
    if (a.work) grab();
    for (; u < chunk_end; (a.work && u + 1 >= chunk_end) ? grab() : (void)(u += a.work ? 1 : nw)) {
        F4x2 qv[V];
#pragma unroll
        for (int vv = 0; vv < V; ++vv) {
            const uint32_t c = q + G * vv;
            qv[vv] = to_x2(ldg_row(P + u * W + (c < W ? c : W - 1)));
        }
        const uint32_t hq = __ldg(H + u);
        uint32_t qn = 0;  // queued survivors (warp-uniform)

        // fp32 test of queue entries [e0, e0 + STEP) of which those < qend are real
        auto fp32_step = [&](uint32_t e0, uint32_t qend) {
            F4x2 rows[UF][V];
            uint32_t pe[UF];
            bool oke[UF];
#pragma unroll
            for (int uu = 0; uu < UF; ++uu) {
                const uint32_t e = e0 + g + NG * uu;
                oke[uu] = e < qend;
                pe[uu] = queue[oke[uu] ? e : e0];
#pragma unroll
                for (int vv = 0; vv < V; ++vv) {
                    const uint32_t c = q + G * vv;
                    const uint64_t row = (oke[uu] && c < W) ? pe[uu] : u;
                    rows[uu][vv] = ldg_row2(P + row * W + (c < W ? c : W - 1));
                }
            }
            __syncwarp();  // scheduling fence: all UF*V loads in flight together
#pragma unroll
            for (int uu = 0; uu < UF; ++uu) {
                Acc2 acc;
#pragma unroll
                for (int vv = 0; vv < V; ++vv) diff2x2(qv[vv], rows[uu][vv], acc);
                float s = acc2_sum(acc);
#pragma unroll
                for (int o = G / 2; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
                const bool accd = decide(s, oke[uu], leader, g * G, a.tp, u, pe[uu], st);
                tails += (oke[uu] && leader) ? 1u : 0u;
                stage.push(leader && accd, edge_key(u, pe[uu], a.sink.nb), a.sink, lane);
            }
        };

        uint32_t limit = a.draws;
        uint64_t z = vertex_key(a.seed_mixed, u) + (uint64_t)(lane + 1) * kGamma;
        for (uint32_t i0 = 0; i0 < limit; i0 += 32 * R, z += (uint64_t)(32 * R) * kGamma) {
            uint32_t pv[R];
            uint32_t first_fire = 0xffffffffu;
#pragma unroll
            for (int k = 0; k < R; ++k) {
                const uint32_t i = i0 + 32 * k + lane;
                const bool valid = i < limit;
                bool fire = false;
                uint32_t t = 0;
                if (valid) {
                    t = lemire32(mix(z + (uint64_t)(32 * k) * kGamma), a.base + i + 1, fire);
                    fire |= test_fire(a.force_mod, u, i, a.draws);
                }
                pv[k] = t + (t >= (uint32_t)u ? 1u : 0u);
                const unsigned fm = __ballot_sync(kFull, valid && fire);
                if (fm && first_fire == 0xffffffffu) first_fire = i0 + 32 * k + __ffs(fm) - 1;
            }
            if (first_fire != 0xffffffffu) limit = first_fire;  // irregular: cut here
            uint32_t hb[R];
#pragma unroll
            for (int k = 0; k < R; ++k) hb[k] = __ldg(H + pv[k]);  // pv < n always
#pragma unroll
            for (int k = 0; k < R; ++k) {
                const uint32_t i = i0 + 32 * k + lane;
                const bool live = i < limit && pv[k] >= plo && pv[k] < phi;
                gpairs += live ? 1u : 0u;
                const bool keep = live && !(head_q(hq, hb[k]) > reject);
                const unsigned km = __ballot_sync(kFull, keep);
                if (keep) queue[qn + __popc(km & lanemask_lt())] = pv[k];
                qn += __popc(km);
            }
            __syncwarp();
            if (qn >= (uint32_t)STEP) {
                uint32_t e0 = 0;
#pragma unroll 1
                for (; e0 + STEP <= qn; e0 += STEP) fp32_step(e0, qn);
                const uint32_t rem = qn - e0;  // < STEP: move them to the front
                const uint32_t mp = (uint32_t)lane < rem ? queue[e0 + lane] : 0u;
                __syncwarp();
                if ((uint32_t)lane < rem) queue[lane] = mp;
                qn = rem;
                __syncwarp();
            }
        }
        if (qn) fp32_step(0, qn);
        __syncwarp();
    }
    stage.flush(a.sink, lane);
    st.pairs = gpairs;
    flush_stats(st, gpairs, a.counters, lane);
    const unsigned long long tw = warp_sum(tails);
    if (lane == 0 && tw) atomicAdd(&a.counters[C_TAIL_PAIRS], tw);
}

template <int G, int V, int R>
cudaError_t head_one(const GatherArgs& a, const HeadArgs& h, cudaStream_t s, int num_sms) {
    auto k = k_gather_head<G, V, R>;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 256, 0);
    if (per_sm < 1) per_sm = 1;
    const uint64_t rows = a.row_end - a.row_begin;
    const uint64_t want = (rows + kWarpsPerBlock - 1) / kWarpsPerBlock;
    const uint64_t cap = (uint64_t)num_sms * per_sm;
    k<<<(unsigned)(want < cap ? want : cap), 256, 0, s>>>(a, h);
    note_launch(1);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_head_quantize(const float* pts, uint32_t stride, uint64_t n, const HeadPlan& p,
                                 uint32_t* out, cudaStream_t s, int num_sms) {
    uint64_t blocks = (n + 255) / 256;
    if (blocks > (uint64_t)num_sms * 16) blocks = (uint64_t)num_sms * 16;
    k_head_quantize<<<(unsigned)(blocks ? blocks : 1), 256, 0, s>>>(pts, stride, n, p.lo,
                                                                     1.0 / p.s, out);
    note_launch(1);
    return cudaGetLastError();
}

cudaError_t launch_gather_head(const GatherArgs& a, const HeadArgs& h, cudaStream_t s, int num_sms) {
    if (a.row_end <= a.row_begin) return cudaSuccess;
    const uint32_t W = a.tp.stride / 4;  // stride is a multiple of 4 for d >= 3
    if (W <= 2) return head_one<2, 1, 4>(a, h, s, num_sms);
    if (W <= 4) return head_one<4, 1, 4>(a, h, s, num_sms);
    if (W <= 8) return head_one<8, 1, 4>(a, h, s, num_sms);
    if (W <= 16) return head_one<16, 1, 4>(a, h, s, num_sms);
    if (W <= 32) return head_one<32, 1, 4>(a, h, s, num_sms);
    if (W <= 64) return head_one<32, 2, 4>(a, h, s, num_sms);
    if (W <= 128) return head_one<32, 4, 2>(a, h, s, num_sms);
    if (W <= 256) return head_one<32, 8, 2>(a, h, s, num_sms);
    return cudaErrorInvalidValue;
}

}  // namespace sngb
