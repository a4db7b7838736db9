// sngb_quant.cu -- the 8-bit filter for wide rows: the gather reads an 8-bit
// copy of the points (4x fewer bytes than fp32) and still decides every pair
// exactly as the reference does.
//
// Quantisation.  s is a power of two >= (max - min)/254 and lo' = floor(min/s)*s,
// so q = rint((a - lo')/s) in [0, 255] is computed exactly in fp64 (up to a
// relative 2^-45 in a - lo' for tiny |a|) and a = lo' + s*q + e with
// |e| <= s/2 * (1 + 2^-30).  Each row stores one chunk with its norms (the head
// norm, over the first kHeadVals values, and N = sum q^2), then its bytes, zero
// padded to 16-byte chunks.
//
// Filter.  For a pair, Q2 = sum (qa - qb)^2 = Na + Nb - 2 sum qa*qb is an exact
// integer (DP4A).  With Dk = s*dqk, |Ek| <= s' = s(1 + 2^-30), Q1 = sum |dqk| <=
// sqrt(d Q2) (Cauchy-Schwarz), the true squared distance S satisfies
//   S <= sum (s|dqk| + s')^2          <= (s*sqrt(Q2) + s'*sqrt(d))^2
//   S >= sum (dk^2 - 2|dk|s')         >= s^2 Q2 - 2 s s' sqrt(d Q2)
// and the reference's fp64 sum is within (d+1) 2^-53 S of S.  Hence
//   Q2 <= A  = ((sqrt(eps2 (1 - 2^-40)) - s' sqrt(d)) / s)^2      => accept
//   Q2 >  B  = ((s' sqrt(d) + sqrt(s'^2 d + eps2 (1 + 2^-40))) / s)^2 => reject
// (A rounded down, B up, with a relative 2^-30 margin for the fp64 evaluation),
// and a pair with A < Q2 <= B is re-evaluated with the reference's exact fp64
// operation order on the fp32 rows -- the same recheck the fp32 filter uses.
// The host enables the path only when that band is narrow relative to eps
// (a data set with a huge value range relative to eps keeps the fp32 filter).
//
// Early rejection (k_gather_q8s, rows of >= kSplitMinRW chunks).  The partial
// sum over the row's head, Q2h = Nha + Nhb - 2 sum_head qa*qb, satisfies
// Q2h <= Q2, so Q2h > B rejects exactly; only the survivors read their tail.
// A sampled pair is far more often a non-neighbour than a neighbour (eps is
// small against the typical distance), so most pairs cost the head's bytes.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "sngb_device.cuh"
#include "sngb_epstest.cuh"
#include "sngb_internal.cuh"
#include "sngb_rng.cuh"

namespace sngb {

bool q8_split(uint32_t nd) {
    const char* e = std::getenv("SNGB_Q8_SPLIT");  // 0 off, 1 on (default: by width)
    const int mode = e ? std::atoi(e) : -1;
    return mode == 0 ? false : (mode == 1 ? nd + 1 >= kHead + 1 : nd + 1 >= kSplitMinRW);
}

bool q8_plan(double lo, double hi, uint32_t d, double eps2, Q8Plan& p) {
    const double need = (hi - lo) / 254.0 * (1.0 + 1e-12);
    if (!(need > 0.0) || !std::isfinite(need)) return false;
    int e = 0;
    std::frexp(need, &e);  // need = m * 2^e, m in [0.5, 1)
    const double s = std::ldexp(1.0, e);
    p.s = s;
    p.lo = std::floor(lo / s) * s;
    const double sp = s * (1.0 + std::ldexp(1.0, -30));
    const double sd = std::sqrt((double)d);
    const double e_lo = eps2 * (1.0 - std::ldexp(1.0, -40));
    const double e_hi = eps2 * (1.0 + std::ldexp(1.0, -40));
    const double qmax = (double)d * 255.0 * 255.0;  // largest possible Q2
    const double ta = (std::sqrt(e_lo) - sp * sd) / s;
    const double a = ta > 0.0 ? std::floor(ta * ta * (1.0 - std::ldexp(1.0, -30))) : -1.0;
    const double tb = (sp * sd + std::sqrt(sp * sp * d + e_hi)) / s;
    const double b = std::ceil(tb * tb * (1.0 + std::ldexp(1.0, -30)));
    p.args.accept_max = (int32_t)std::min(a, qmax + 1.0);
    p.args.reject_min = (int32_t)std::min(b, qmax + 1.0);
    // worthwhile if the band is narrow in distance units (<= 25 % of eps wide)
    const double band = (std::sqrt(std::max(b, 0.0)) - std::sqrt(std::max(a, 0.0))) * s;
    return a >= 0.0 && band <= 0.25 * std::sqrt(eps2);
}

namespace {

// warp per row: the norm chunk (N over the head's values, N over the row), then
// bytes q of the row's d values, zero padded
// perm (optional): stored value k is column perm[k] -- the columns in order of
// decreasing variance, so the head holds the most discriminative ones (a
// distance is invariant under a common permutation of the coordinates).
__global__ void k_quantize(const float* __restrict__ pts, uint32_t stride, uint64_t n, uint32_t d,
                           double lo, double inv_s, uint32_t nd, uint4* __restrict__ out,
                           const double* __restrict__ pts64, const uint32_t* __restrict__ perm) {
    const int lane = threadIdx.x & 31;
    const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t r = gw; r < n; r += nw) {
        const float* row = pts + r * stride;
        uint4* orow = out + r * (nd + 1);
        uint32_t norm = 0, norm_head = 0;
        for (uint32_t c = lane; c < nd; c += 32) {
            uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
            for (int j4 = 0; j4 < 4; ++j4) {
                const uint32_t k0 = 16 * c + 4 * j4;
                if (k0 >= d) break;  // rows are 16-byte aligned with a stride of ceil4(d)
                double vs[4];
                if (perm) {  // permuted columns: scalar loads from the (L1-resident) row
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint32_t col = k0 + j < d ? __ldg(perm + k0 + j) : 0u;
                        vs[j] = k0 + j >= d ? 0.0 : (pts64 ? pts64[r * d + col] : (double)__ldg(row + col));
                    }
                } else if (pts64) {  // fp64 input: quantise the caller's values themselves
#pragma unroll
                    for (int j = 0; j < 4; ++j) vs[j] = k0 + j < d ? pts64[r * d + k0 + j] : 0.0;
                } else {
                    const float4 v = __ldg(reinterpret_cast<const float4*>(row + k0));
                    vs[0] = v.x, vs[1] = v.y, vs[2] = v.z, vs[3] = v.w;
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const double x = rint((vs[j] - lo) * inv_s);
                    const uint32_t q = k0 + j >= d ? 0u  // padding past d quantises to 0
                                       : x <= 0.0 ? 0u : (x >= 255.0 ? 255u : (uint32_t)x);
                    w[j4] |= q << (8 * j);
                    norm += q * q;
                    norm_head += c < kHead - 1 ? q * q : 0u;
                }
            }
            orow[1 + c] = make_uint4(w[0], w[1], w[2], w[3]);
        }
        norm = __reduce_add_sync(kFull, norm);
        norm_head = __reduce_add_sync(kFull, norm_head);
        if (lane == 0) orow[0] = make_uint4(norm_head, norm, 0, 0);
    }
}

// Permuted columns from fp32 rows: each warp stages its row in shared memory
// with 16-byte loads, then gathers the stored order from there (a scalar load
// per value from global memory measured 2.5x slower than the unpermuted pass).
__global__ void __launch_bounds__(128) k_quantize_perm(const float* __restrict__ pts, uint32_t stride,
                                                       uint64_t n, uint32_t d, double lo, double inv_s,
                                                       uint32_t nd, uint4* __restrict__ out,
                                                       const uint32_t* __restrict__ perm) {
    __shared__ __align__(16) float s_row[4][kQ8MaxD];
    __shared__ uint16_t s_perm[kQ8MaxD];
    for (uint32_t k = threadIdx.x; k < d; k += blockDim.x) s_perm[k] = (uint16_t)__ldg(perm + k);
    __syncthreads();
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    float* srow = s_row[wib];
    for (uint64_t r = gw; r < n; r += nw) {
        const float4* row4 = reinterpret_cast<const float4*>(pts + r * stride);
        for (uint32_t k4 = lane; k4 < stride / 4; k4 += 32)
            reinterpret_cast<float4*>(srow)[k4] = __ldg(row4 + k4);
        __syncwarp();
        uint4* orow = out + r * (nd + 1);
        uint32_t norm = 0, norm_head = 0;
        for (uint32_t c = lane; c < nd; c += 32) {
            uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const uint32_t k = 16 * c + j;
                uint32_t q = 0;  // padding past d quantises to 0
                if (k < d) {
                    const double x = rint(((double)srow[s_perm[k]] - lo) * inv_s);
                    q = x <= 0.0 ? 0u : (x >= 255.0 ? 255u : (uint32_t)x);
                }
                w[j >> 2] |= q << (8 * (j & 3));
                norm += q * q;
                norm_head += c < kHead - 1 ? q * q : 0u;
            }
            orow[1 + c] = make_uint4(w[0], w[1], w[2], w[3]);
        }
        norm = __reduce_add_sync(kFull, norm);
        norm_head = __reduce_add_sync(kFull, norm_head);
        if (lane == 0) orow[0] = make_uint4(norm_head, norm, 0, 0);
        __syncwarp();
    }
}

__device__ __forceinline__ uint32_t dot16(uint4 a, uint4 b, uint32_t acc) {
    acc = __dp4a(a.x, b.x, acc);
    acc = __dp4a(a.y, b.y, acc);
    acc = __dp4a(a.z, b.z, acc);
    return __dp4a(a.w, b.w, acc);
}

// Wide-row gather over the 8-bit rows: the k_gather G = 32 structure (dynamic
// row claiming, draws regenerated from their counters, live pairs compacted
// per 32-draw chunk, U rows per step behind a warp-sync fence, transposed
// reduce-scatter leaving pair k's sum in lane 32k/U) with integer arithmetic.
template <int V8, int U>
__global__ void __launch_bounds__(256, 2) k_gather_q8(const GatherArgs a, const Q8Args q8) {
    __shared__ unsigned long long s_stage[kWarpsPerBlock][kStage];
    __shared__ uint32_t s_list[kWarpsPerBlock][32];
    constexpr int SPAN = 32 / U;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint64_t gw = (uint64_t)blockIdx.x * kWarpsPerBlock + wib;
    const uint64_t nw = (uint64_t)gridDim.x * kWarpsPerBlock;
    const uint4* __restrict__ Q = q8.rows;
    const uint32_t RW = q8.nd + 1;
    const uint32_t plo = a.part_lo, phi = a.part_hi;
    uint32_t* list = s_list[wib];
    WarpStage<kStage> stage{s_stage[wib], 0};
    TestStats st;
    unsigned long long gpairs = 0;

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
        uint4 qq[V8];
        uint32_t nu = 0;
#pragma unroll
        for (int vv = 0; vv < V8; ++vv) {
            const uint32_t c = lane + 32 * vv;
            qq[vv] = c < RW ? __ldg(Q + u * RW + c) : make_uint4(0, 0, 0, 0);
            if (c == 0) {
                nu = qq[vv].y;
                qq[vv] = make_uint4(0, 0, 0, 0);
            }
        }
        nu = __reduce_add_sync(kFull, nu);  // one lane holds the query's norm
        uint32_t limit = a.draws;
        uint64_t z = vertex_key(a.seed_mixed, u) + (uint64_t)(lane + 1) * kGamma;
        for (uint32_t i0 = 0; i0 < limit; i0 += 32, z += 32ull * kGamma) {
            const uint32_t i = i0 + lane;
            const bool valid = i < limit;
            bool fire = false;
            uint32_t t = 0;
            if (valid) {
                t = lemire32(mix(z), a.base + i + 1, fire);
                fire |= test_fire(a.force_mod, u, i, a.draws);
            }
            const uint32_t p = t + (t >= (uint32_t)u ? 1u : 0u);
            const unsigned fm = __ballot_sync(kFull, valid && fire);
            if (fm) limit = i0 + __ffs(fm) - 1;  // irregular vertex: cut here
            const bool live = i < limit && p >= plo && p < phi;
            const unsigned m = __ballot_sync(kFull, live);
            if (live) list[__popc(m & lanemask_lt())] = p;
            const uint32_t nlive = __popc(m);
            __syncwarp();
#pragma unroll 1
            for (uint32_t j0 = 0; j0 < nlive; j0 += U) {
                uint4 rows[U][V8];
#pragma unroll
                for (int uu = 0; uu < U; ++uu) {
                    const uint32_t j = j0 + uu;
                    const uint32_t pv = list[j < nlive ? j : j0];
#pragma unroll
                    for (int vv = 0; vv < V8; ++vv) {
                        const uint32_t c = lane + 32 * vv;
                        rows[uu][vv] = c < RW ? __ldg(Q + (uint64_t)pv * RW + c)
                                              : make_uint4(0, 0, 0, 0);
                    }
                }
                __syncwarp();  // scheduling fence: all U*V8 loads in flight together
                int ps[U];
#pragma unroll
                for (int uu = 0; uu < U; ++uu) {
                    uint32_t dot = 0, nv = 0;
#pragma unroll
                    for (int vv = 0; vv < V8; ++vv) {
                        const uint32_t c = lane + 32 * vv;
                        dot = dot16(qq[vv], rows[uu][vv], dot);  // query norm chunk is zeroed
                        if (c == 0) nv = rows[uu][vv].y;
                    }
                    ps[uu] = (int)nv - 2 * (int)dot;  // partial of Nb - 2 sum qa qb
                }
#pragma unroll
                for (int o = 16, mm = U; mm > 1; o >>= 1, mm >>= 1) {
                    const bool hi = (lane & o) != 0;
#pragma unroll
                    for (int k = 0; k < mm / 2; ++k) {
                        const int mine = hi ? ps[k + mm / 2] : ps[k];
                        const int other = hi ? ps[k] : ps[k + mm / 2];
                        ps[k] = mine + __shfl_xor_sync(kFull, other, o);
                    }
                }
#pragma unroll
                for (int o = SPAN / 2; o > 0; o >>= 1) ps[0] += __shfl_xor_sync(kFull, ps[0], o);
                const uint32_t pj = j0 + lane / SPAN;
                const bool okm = (lane % SPAN) == 0 && pj < nlive;
                const uint32_t pm = list[okm ? pj : j0];
                const int q2 = (int)nu + ps[0];
                const bool acc = okm && q2 <= q8.accept_max;
                if (okm && q2 > q8.accept_max && q2 <= q8.reject_min) {  // band: k_band decides
                    band_push(a.tp, u, pm, __int_as_float(0x7fc00000));
                    st.band++;
                }
                gpairs += okm ? 1u : 0u;
                stage.push(acc, edge_key(u, pm, a.sink.nb), a.sink, lane);
            }
            __syncwarp();
        }
    }
    stage.flush(a.sink, lane);
    st.pairs = gpairs;
    flush_stats(st, gpairs, a.counters, lane);
}

// Early-reject gather for wide rows.  Phase A: a quarter warp per pair reads the
// pair's head (kHead chunks, the norm chunk first; two chunks per lane), 32 pairs
// per warp step;
// pairs whose head sum already exceeds reject_min are rejected, the others are
// queued with Q2h + Nta.  Phase B: the full warp finishes UB queued pairs per
// step over the tail chunks plus the norm chunk (for Ntb = N - Nhead).  Both
// lists hold one query row's pairs and run in whole steps as they fill (live
// partners accumulate across 32-draw chunks: a launch restricted to a partner
// slice finds few per chunk), the remainders at the end of the row.
template <int VT, int UA, int UB>
__global__ void __launch_bounds__(256, 2) k_gather_q8s(const GatherArgs a, const Q8Args q8) {
    __shared__ unsigned long long s_stage[kWarpsPerBlock][kStage];
    __shared__ uint32_t s_list[kWarpsPerBlock][64];
    __shared__ uint32_t s_qp[kWarpsPerBlock][64];
    __shared__ int s_qh[kWarpsPerBlock][64];
    static_assert(UA == 16, "phase A leaves one pair per lane");
    constexpr int SPANB = 32 / UB;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    // phase A: a quarter warp per pair, lane q of it holding head chunks q and q + 8
    const int hc = lane & 7;
    const uint64_t gw = (uint64_t)blockIdx.x * kWarpsPerBlock + wib;
    const uint64_t nw = (uint64_t)gridDim.x * kWarpsPerBlock;
    const uint4* __restrict__ Q = q8.rows;
    const uint32_t RW = q8.nd + 1, T = RW - kHead;  // tail chunks; slot T = norm chunk
    const uint32_t plo = a.part_lo, phi = a.part_hi;
    uint32_t* list = s_list[wib];
    uint32_t* qp = s_qp[wib];
    int* qh2 = s_qh[wib];
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
        uint4 qh = __ldg(Q + u * RW + hc);
        const uint4 qh8 = __ldg(Q + u * RW + hc + 8);
        const uint32_t nha = __shfl_sync(kFull, qh.x, 0), nfa = __shfl_sync(kFull, qh.y, 0);
        if (hc == 0) qh = make_uint4(0, 0, 0, 0);
        uint4 qt[VT];
#pragma unroll
        for (int v = 0; v < VT; ++v) {
            const uint32_t sl = lane + 32 * v;
            qt[v] = sl < T ? __ldg(Q + u * RW + kHead + sl) : make_uint4(0, 0, 0, 0);
        }
        const int nta = (int)(nfa - nha);
        uint32_t qn = 0;  // queued survivors (warp-uniform)

        // phase B over queue entries [e0, e0 + UB) of which those < qend are real
        auto tail_step = [&](uint32_t e0, uint32_t qend) {
            uint4 rows[UB][VT];
#pragma unroll
            for (int uu = 0; uu < UB; ++uu) {
                const uint32_t e = e0 + uu;
                const uint32_t pv = qp[e < qend ? e : e0];
#pragma unroll
                for (int v = 0; v < VT; ++v) {
                    const uint32_t sl = lane + 32 * v;
                    // slots past T re-read the norm chunk: the query is zero there
                    rows[uu][v] = __ldg(Q + (uint64_t)pv * RW + (sl < T ? kHead + sl : 0));
                }
            }
            __syncwarp();  // scheduling fence: all UB*VT loads in flight together
            int ps[UB];
#pragma unroll
            for (int uu = 0; uu < UB; ++uu) {
                uint32_t dot = 0;
                int nt = 0;
#pragma unroll
                for (int v = 0; v < VT; ++v) {
                    dot = dot16(qt[v], rows[uu][v], dot);  // the query's slot T is zero
                    if (lane + 32 * v == T) nt = (int)(rows[uu][v].y - rows[uu][v].x);
                }
                ps[uu] = nt - 2 * (int)dot;
            }
#pragma unroll
            for (int o = 16, mm = UB; mm > 1; o >>= 1, mm >>= 1) {
                const bool hi = (lane & o) != 0;
#pragma unroll
                for (int k = 0; k < mm / 2; ++k) {
                    const int mine = hi ? ps[k + mm / 2] : ps[k];
                    const int other = hi ? ps[k] : ps[k + mm / 2];
                    ps[k] = mine + __shfl_xor_sync(kFull, other, o);
                }
            }
#pragma unroll
            for (int o = SPANB / 2; o > 0; o >>= 1) ps[0] += __shfl_xor_sync(kFull, ps[0], o);
            const uint32_t e = e0 + lane / SPANB;
            const bool okm = (lane % SPANB) == 0 && e < qend;
            const uint32_t pm = qp[okm ? e : e0];
            const int q2 = qh2[okm ? e : e0] + ps[0];
            const bool acc = okm && q2 <= q8.accept_max;
            if (okm && q2 > q8.accept_max && q2 <= q8.reject_min) {  // band: k_band decides
                band_push(a.tp, u, pm, __int_as_float(0x7fc00000));
                st.band++;
            }
            tails += okm ? 1u : 0u;
            stage.push(acc, edge_key(u, pm, a.sink.nb), a.sink, lane);
        };

        // phase A over list[0, nA), nA <= 2*UA: heads, survivors appended to the queue
        auto head_step = [&](uint32_t nA) {
            // 8 pairs per quarter warp: two 16-byte chunks per lane per pair (one
            // row address for both), a 3-level transposed reduce-scatter over the
            // quarter warp -- half the address and shuffle work of a half warp
            // per pair with one chunk per lane
            constexpr int UQ = 8;
            uint4 r0[UQ], r1[UQ];
#pragma unroll
            for (int k = 0; k < UQ; ++k) {  // pairs past nA re-read pair 0's head (masked below)
                const uint32_t j = (lane >> 3) * UQ + k;
                const uint4* rp = Q + (size_t)list[j < nA ? j : 0] * RW + hc;
                r0[k] = __ldg(rp);
                r1[k] = __ldg(rp + 8);
            }
            __syncwarp();
            int ps[UQ];
#pragma unroll
            for (int k = 0; k < UQ; ++k)
                ps[k] = (hc == 0 ? (int)r0[k].x : 0) -
                        2 * (int)dot16(qh8, r1[k], dot16(qh, r0[k], 0u));
#pragma unroll
            for (int o = 4, mm = UQ; mm > 1; o >>= 1, mm >>= 1) {
                const bool hi = (lane & o) != 0;
#pragma unroll
                for (int k = 0; k < mm / 2; ++k) {
                    const int mine = hi ? ps[k + mm / 2] : ps[k];
                    const int other = hi ? ps[k] : ps[k + mm / 2];
                    ps[k] = mine + __shfl_xor_sync(kFull, other, o);
                }
            }
            const uint32_t pj = lane;  // pair of this lane
            const bool okm = pj < nA;
            const int q2h = (int)nha + ps[0];
            const bool keep = okm && q2h <= q8.reject_min;  // else Q2 >= Q2h > B: reject
            gpairs += okm ? 1u : 0u;
            const unsigned km = __ballot_sync(kFull, keep);
            if (keep) {
                const uint32_t slot = qn + __popc(km & lanemask_lt());
                qp[slot] = list[pj];
                qh2[slot] = q2h + nta;
            }
            qn += __popc(km);
            __syncwarp();
        };
        // phase B in whole steps; the remainder (< UB) moves to the front
        auto drain = [&]() {
            if (qn < (uint32_t)UB) return;
            uint32_t e0 = 0;
#pragma unroll 1
            for (; e0 + UB <= qn; e0 += UB) tail_step(e0, qn);
            const uint32_t rem = qn - e0;
            uint32_t mp = 0;
            int mh = 0;
            if ((uint32_t)lane < rem) mp = qp[e0 + lane], mh = qh2[e0 + lane];
            __syncwarp();
            if ((uint32_t)lane < rem) qp[lane] = mp, qh2[lane] = mh;
            qn = rem;
            __syncwarp();
        };

        uint32_t nl = 0;  // live partners waiting for phase A (warp-uniform)
        uint32_t limit = a.draws;
        uint64_t z = vertex_key(a.seed_mixed, u) + (uint64_t)(lane + 1) * kGamma;
        const uint32_t* pre = nullptr;  // bucketed partner list of this launch's slices
        if (a.partners) {
            const uint64_t r = u - a.partners_row0;
            const uint32_t* o = a.poff + r * (a.nbuckets + 1);
            const uint32_t lo = __ldg(o + a.blo);
            pre = a.partners + r * a.draws + lo;
            limit = __ldg(o + a.bhi) - lo;
        }
        for (uint32_t i0 = 0; i0 < limit; i0 += 32, z += 32ull * kGamma) {
            const uint32_t i = i0 + lane;
            uint32_t p;
            if (pre) {
                p = i < limit ? __ldg(pre + i) : 0u;
            } else {
                const bool valid = i < limit;
                bool fire = false;
                uint32_t t = 0;
                if (valid) {
                    t = lemire32(mix(z), a.base + i + 1, fire);
                    fire |= test_fire(a.force_mod, u, i, a.draws);
                }
                p = t + (t >= (uint32_t)u ? 1u : 0u);
                const unsigned fm = __ballot_sync(kFull, valid && fire);
                if (fm) limit = i0 + __ffs(fm) - 1;  // irregular vertex: cut here
            }
            const bool live = i < limit && p >= plo && p < phi;
            const unsigned m = __ballot_sync(kFull, live);
            if (live) list[nl + __popc(m & lanemask_lt())] = p;
            nl += __popc(m);
            __syncwarp();
            if (nl >= 2 * UA) {
                head_step(2 * UA);
                const uint32_t rem = nl - 2 * UA;  // < 32: move them to the front
                const uint32_t mp = (uint32_t)lane < rem ? list[2 * UA + lane] : 0u;
                __syncwarp();
                if ((uint32_t)lane < rem) list[lane] = mp;
                nl = rem;
                __syncwarp();
            }
            drain();
        }
        if (nl) head_step(nl);
        drain();
        if (qn) tail_step(0, qn);
        __syncwarp();
    }
    stage.flush(a.sink, lane);
    st.pairs = gpairs;
    flush_stats(st, gpairs, a.counters, lane);
    const unsigned long long tw = warp_sum(tails);
    if (lane == 0 && tw) atomicAdd(&a.counters[C_TAIL_PAIRS], tw);
}

// Floyd replacement pairs through the 8-bit filter: one pair per warp step
template <int V8>
__global__ void __launch_bounds__(256) k_extras_q8(const ExtrasArgs a, const Q8Args q8) {
    __shared__ unsigned long long s_stage[kWarpsPerBlock][kStage];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint64_t gw = (uint64_t)blockIdx.x * kWarpsPerBlock + wib;
    const uint64_t nw = (uint64_t)gridDim.x * kWarpsPerBlock;
    const uint4* __restrict__ Q = q8.rows;
    const uint32_t RW = q8.nd + 1;
    WarpStage<kStage> stage{s_stage[wib], 0};
    TestStats st;
    uint64_t count = *a.count_ptr;
    if (count > a.capacity) count = a.capacity;
    for (uint64_t p = gw; p < count; p += nw) {
        const unsigned long long rec = a.extras[p];
        const uint64_t u = rec >> 32, v = rec & 0xffffffffull;
        int part = 0;
        uint32_t dot = 0;
#pragma unroll
        for (int vv = 0; vv < V8; ++vv) {
            const uint32_t c = lane + 32 * vv;
            if (c == 0) {
                part = (int)(__ldg(Q + u * RW).y + __ldg(Q + v * RW).y);
            } else if (c < RW) {
                dot = dot16(__ldg(Q + u * RW + c), __ldg(Q + v * RW + c), dot);
            }
        }
        part -= 2 * (int)dot;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(kFull, part, o);
        const bool acc = part <= q8.accept_max;
        if (lane == 0 && !acc && part <= q8.reject_min) {  // band: k_band decides
            band_push(a.tp, u, v, __int_as_float(0x7fc00000));
            st.band++;
        }
        if (lane == 0) st.pairs++;
        stage.push(lane == 0 && acc, edge_key(u, v, a.sink.nb), a.sink, lane);
    }
    stage.flush(a.sink, lane);
    flush_stats(st, 0, a.counters, lane);
}

// Floyd replacement pairs through the head/tail filter (rows that take
// k_gather_q8s): half a warp per pair reads both heads (one chunk per lane,
// the norm chunk first); only pairs the heads do not reject read their tails
// (VT chunks per lane).  Nothing is shared between pairs, so every row is read
// in full per pair: the early reject saves ~2/3 of the bytes.
template <int VT>
__global__ void __launch_bounds__(256) k_extras_q8s(const ExtrasArgs a, const Q8Args q8) {
    __shared__ unsigned long long s_stage[kWarpsPerBlock][kStage];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int half = lane >> 4, hc = lane & 15;
    const uint64_t gw = (uint64_t)blockIdx.x * kWarpsPerBlock + wib;
    const uint64_t nw = (uint64_t)gridDim.x * kWarpsPerBlock;
    const uint4* __restrict__ Q = q8.rows;
    const uint32_t RW = q8.nd + 1, T = RW - kHead;
    WarpStage<kStage> stage{s_stage[wib], 0};
    TestStats st;
    uint64_t count = *a.count_ptr;
    if (count > a.capacity) count = a.capacity;
    for (uint64_t p0 = gw * 2; p0 < count; p0 += nw * 2) {
        const uint64_t p = p0 + half;
        const bool ok = p < count;
        const unsigned long long rec = a.extras[ok ? p : p0];
        const uint64_t u = rec >> 32, v = rec & 0xffffffffull;
        const uint4 x = __ldg(Q + u * RW + hc), y = __ldg(Q + v * RW + hc);
        int part = hc == 0 ? (int)(x.x + y.x) : -2 * (int)dot16(x, y, 0u);
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) part += __shfl_xor_sync(kFull, part, o);
        const bool need_tail = ok && part <= q8.reject_min;  // else Q2 >= Q2h > B: reject
        int q2 = part;
        if (__any_sync(kFull, need_tail)) {
            int t = hc == 0 ? (int)((x.y - x.x) + (y.y - y.x)) : 0;  // tail norms
            uint32_t dot = 0;
#pragma unroll
            for (int k = 0; k < VT; ++k) {
                const uint32_t sl = hc + 16 * k;
                if (sl < T)
                    dot = dot16(__ldg(Q + u * RW + kHead + sl), __ldg(Q + v * RW + kHead + sl), dot);
            }
            t -= 2 * (int)dot;
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) t += __shfl_xor_sync(kFull, t, o);
            q2 += t;
        }
        const bool leader = hc == 0 && ok;
        const bool acc = leader && need_tail && q2 <= q8.accept_max;
        if (leader && need_tail && q2 > q8.accept_max && q2 <= q8.reject_min) {  // k_band decides
            band_push(a.tp, u, v, __int_as_float(0x7fc00000));
            st.band++;
        }
        if (leader) st.pairs++;
        stage.push(acc, edge_key(u, v, a.sink.nb), a.sink, lane);
    }
    stage.flush(a.sink, lane);
    flush_stats(st, 0, a.counters, lane);
}

template <int V8>
cudaError_t extras_q8_one(const ExtrasArgs& a, const Q8Args& q, cudaStream_t s, int num_sms) {
    auto k = k_extras_q8<V8>;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 256, 0);
    if (per_sm < 1) per_sm = 1;
    const uint64_t want = (a.capacity + kWarpsPerBlock - 1) / kWarpsPerBlock;
    const uint64_t cap = (uint64_t)num_sms * per_sm;
    const uint64_t g = want < cap ? want : cap;
    k<<<(unsigned)(g ? g : 1), 256, 0, s>>>(a, q);
    note_launch(1);
    return cudaGetLastError();
}

template <typename K>
cudaError_t q8_launch(K k, const GatherArgs& a, const Q8Args& q, cudaStream_t s, int num_sms) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 256, 0);
    if (per_sm < 1) per_sm = 1;
    const uint64_t rows = a.row_end - a.row_begin;
    const uint64_t want = (rows + kWarpsPerBlock - 1) / kWarpsPerBlock;
    const uint64_t cap = (uint64_t)num_sms * per_sm;
    k<<<(unsigned)(want < cap ? want : cap), 256, 0, s>>>(a, q);
    note_launch(1);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_quantize(const float* pts, uint32_t stride, uint64_t n, uint32_t d,
                            const Q8Plan& p, uint4* out, cudaStream_t s, int num_sms,
                            const double* pts64) {
    const uint32_t nd = (d + 15) / 16;
    uint64_t blocks = (n + 7) / 8;
    if (blocks > (uint64_t)num_sms * 16) blocks = (uint64_t)num_sms * 16;
    if (p.perm && !pts64) {
        uint64_t b4 = (n + 3) / 4;
        if (b4 > (uint64_t)num_sms * 32) b4 = (uint64_t)num_sms * 32;
        k_quantize_perm<<<(unsigned)(b4 ? b4 : 1), 128, 0, s>>>(pts, stride, n, d, p.lo, 1.0 / p.s,
                                                                 nd, out, p.perm);
    } else {
        k_quantize<<<(unsigned)(blocks ? blocks : 1), 256, 0, s>>>(pts, stride, n, d, p.lo,
                                                                    1.0 / p.s, nd, out, pts64, p.perm);
    }
    note_launch(1);
    return cudaGetLastError();
}

namespace {
// per-column sum and sum of squares of rows [0, n), shifted by the column's
// value in row 0 (ranking only needs the order of the variances; the shift
// keeps fp32 partial sums meaningful under a large common offset): thread per
// column of a 32-column strip, rows strided over gridDim.y, 8 rows in flight
__global__ void k_colstats(const float* __restrict__ pts, uint32_t stride, uint64_t n, uint32_t d,
                           const double* __restrict__ pts64, double* __restrict__ stats) {
    const uint32_t col = blockIdx.x * 32 + (threadIdx.x & 31);
    const uint64_t ry = blockIdx.y * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const uint64_t rs = (uint64_t)gridDim.y * (blockDim.x >> 5);
    if (col >= d) return;
    auto val = [&](uint64_t r) -> float {
        return pts64 ? (float)pts64[r * d + col] : __ldg(pts + r * stride + col);
    };
    const float x0 = val(0);
    float s1 = 0.f, s2 = 0.f;
    uint64_t r = ry;
    for (; r + 7 * rs < n; r += 8 * rs) {
        float x[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = val(r + k * rs) - x0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            s1 += x[k];
            s2 += x[k] * x[k];
        }
    }
    for (; r < n; r += rs) {
        const float x = val(r) - x0;
        s1 += x;
        s2 += x * x;
    }
    atomicAdd(&stats[col], (double)s1);
    atomicAdd(&stats[d + col], (double)s2);
}
}  // namespace

cudaError_t launch_colstats(const float* pts, uint32_t stride, uint64_t n, uint32_t d,
                            const double* pts64, double* stats, cudaStream_t s, int num_sms) {
    cudaError_t e = cudaMemsetAsync(stats, 0, 2 * (size_t)d * sizeof(double), s);
    if (e != cudaSuccess) return e;
    const uint32_t gx = (d + 31) / 32;
    uint32_t gy = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)num_sms * 8 / gx, (n + 63) / 64));
    k_colstats<<<dim3(gx, gy), 256, 0, s>>>(pts, stride, n, d, pts64, stats);
    note_launch(1);
    return cudaGetLastError();
}

template <int VT>
cudaError_t extras_q8s_one(const ExtrasArgs& a, const Q8Args& q, cudaStream_t s, int num_sms) {
    auto k = k_extras_q8s<VT>;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 256, 0);
    if (per_sm < 1) per_sm = 1;
    const uint64_t want = (a.capacity + 2 * kWarpsPerBlock - 1) / (2 * kWarpsPerBlock);
    const uint64_t cap = (uint64_t)num_sms * per_sm;
    const uint64_t g = want < cap ? want : cap;
    k<<<(unsigned)(g ? g : 1), 256, 0, s>>>(a, q);
    note_launch(1);
    return cudaGetLastError();
}

cudaError_t launch_extras_q8(const ExtrasArgs& a, const Q8Args& q, cudaStream_t s, int num_sms) {
    if (a.capacity == 0) return cudaSuccess;
    if (q8_split(q.nd)) {
        switch ((q.nd + 1 - kHead + 15) / 16) {  // tail chunks per lane of a half warp
            case 1: return extras_q8s_one<1>(a, q, s, num_sms);
            case 2: return extras_q8s_one<2>(a, q, s, num_sms);
            case 3: return extras_q8s_one<3>(a, q, s, num_sms);
            case 4: return extras_q8s_one<4>(a, q, s, num_sms);
            case 5: return extras_q8s_one<5>(a, q, s, num_sms);
            case 6: return extras_q8s_one<6>(a, q, s, num_sms);
            default: break;  // wider rows: one pair per warp below
        }
    }
    switch ((q.nd + 1 + 31) / 32) {
        case 1: return extras_q8_one<1>(a, q, s, num_sms);
        case 2: return extras_q8_one<2>(a, q, s, num_sms);
        case 3: return extras_q8_one<3>(a, q, s, num_sms);
        default: return cudaErrorInvalidValue;
    }
}

namespace {
// Bucketed partner lists, warp per row: every draw of k_gather (counter i+1,
// Lemire, p = t + (t >= u)) held in registers (D <= 32 * MAXC), cut at an
// irregular vertex's first fired draw, counted per partner slice, prefix-summed
// and scattered slice by slice (ballot ranks keep draw order within a slice).
template <int MAXC>
__global__ void __launch_bounds__(256) k_partners(const GatherArgs a, uint32_t* __restrict__ lists,
                                                  uint32_t* __restrict__ offsets) {
    const int lane = threadIdx.x & 31;
    const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint32_t D = a.draws, B = a.nbuckets;
    const uint64_t n = a.n;
    auto bound = [&](uint32_t b) { return (uint32_t)(n * b / B); };
    for (uint64_t u = a.row_begin + gw; u < a.row_end; u += nw) {
        uint32_t pv[MAXC];
        uint32_t limit = D;
        uint64_t z = vertex_key(a.seed_mixed, u) + (uint64_t)(lane + 1) * kGamma;
#pragma unroll
        for (int c = 0; c < MAXC; ++c, z += 32ull * kGamma) {
            const uint32_t i = 32 * c + lane;
            bool fire = false;
            const uint32_t t = lemire32(mix(z), a.base + i + 1, fire);
            fire = i < D && (fire || test_fire(a.force_mod, u, i, D));
            const unsigned fm = __ballot_sync(kFull, fire);
            if (fm && limit == D) limit = 32 * c + __ffs(fm) - 1;
            pv[c] = t + (t >= (uint32_t)u ? 1u : 0u);
        }
        uint32_t bk[MAXC];  // slice of each draw, B = not live
#pragma unroll
        for (int c = 0; c < MAXC; ++c) {
            const uint32_t i = 32 * c + lane;
            uint32_t b = (uint32_t)((uint64_t)pv[c] * B / n);
            if (b + 1 < B && bound(b + 1) <= pv[c]) ++b;
            if (b > 0 && bound(b) > pv[c]) --b;
            bk[c] = i < limit ? b : B;
        }
        uint32_t* off = offsets + (u - a.row_begin) * (B + 1);
        uint32_t* out = lists + (u - a.row_begin) * D;
        uint32_t pos = 0;  // running offset of slice b
        for (uint32_t b = 0; b < B; ++b) {
            if (lane == 0) off[b] = pos;
#pragma unroll
            for (int c = 0; c < MAXC; ++c) {
                const unsigned m = __ballot_sync(kFull, bk[c] == b);
                if (bk[c] == b) out[pos + __popc(m & lanemask_lt())] = pv[c];
                pos += __popc(m);
            }
        }
        if (lane == 0) off[B] = pos;
    }
}
}  // namespace

cudaError_t launch_partners(const GatherArgs& a, uint32_t* lists, uint32_t* offsets, cudaStream_t s,
                            int num_sms) {
    if (a.row_end <= a.row_begin || a.draws == 0) return cudaSuccess;
    uint64_t blocks = (a.row_end - a.row_begin + 7) / 8;
    if (blocks > (uint64_t)num_sms * 8) blocks = (uint64_t)num_sms * 8;
    const unsigned g = (unsigned)blocks;
    if (a.draws <= 256) k_partners<8><<<g, 256, 0, s>>>(a, lists, offsets);
    else if (a.draws <= 512) k_partners<16><<<g, 256, 0, s>>>(a, lists, offsets);
    else if (a.draws <= 1024) k_partners<32><<<g, 256, 0, s>>>(a, lists, offsets);
    else return cudaErrorInvalidValue;
    note_launch(1);
    return cudaGetLastError();
}

cudaError_t launch_gather_q8(const GatherArgs& a, const Q8Args& q, cudaStream_t s, int num_sms) {
    if (a.row_end <= a.row_begin) return cudaSuccess;
    const uint32_t rw = q.nd + 1;
    if (q8_split(q.nd)) {
        switch ((rw - kHead + 1 + 31) / 32) {  // tail chunks + the norm chunk
            // UA 16, UB 8 (measured on cfg2: gather 1.21 ms; UA 8 1.40, UA 4 1.73, UB 4
            // 1.32; 3 blocks/SM 1.31-1.76); UB 4 where 8 would spill
            case 1: return q8_launch(k_gather_q8s<1, 16, 8>, a, q, s, num_sms);
            case 2: return q8_launch(k_gather_q8s<2, 16, 8>, a, q, s, num_sms);
            case 3: return q8_launch(k_gather_q8s<3, 16, 4>, a, q, s, num_sms);
            default: return cudaErrorInvalidValue;
        }
    }
    // 8 rows per step (measured: U = 2 3.48 ms, 4 2.77 ms, 8 2.62 ms on cfg2)
    switch ((rw + 31) / 32) {
        case 1: return q8_launch(k_gather_q8<1, 8>, a, q, s, num_sms);
        case 2: return q8_launch(k_gather_q8<2, 8>, a, q, s, num_sms);
        case 3: return q8_launch(k_gather_q8<3, 8>, a, q, s, num_sms);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace sngb
