// sngb_head.cu -- the head filter for narrow rows: an exact early reject on a
// compact, L2-resident copy of a few coordinates of each row, so most sampled
// pairs never read their fp32 row.
//
// Why.  A random row from HBM costs one DRAM access whether it is 16, 32, 64
// or 128 bytes wide (measured on B200, tools/gather_ceiling.cu: 6.3e10, 4.9e10,
// 4.2e10 and 4.2e10 random rows/s), so on a table like cfg5's (20 M x 128 B =
// 2.56 GB) fewer bytes per row buy nothing -- only a table that stays in L2
// does.  L2 keeps a line near the SMs that read it on both dies, so a table
// read uniformly by all SMs stays resident only up to about half the 126 MB
// (an 80 MB head table measured a 43 % hit rate).  Three head formats, picked
// by the host so the table fits: four 8-bit coordinates (4 B), two 16-bit
// coordinates (4 B), two 8-bit coordinates (2 B; cfg5: 40 MB).  On L2-resident
// tables the head also saves instructions: one 2-4 byte load and a few integer
// ops instead of a G-lane row gather and reduction per pair.
//
// Quantisation (host plan, head_plan).  s is a power of two >= (max - min)/(2^b - 2)
// over all values and lo' = floor(min/s)*s, so q = rint((a - lo')/s) fits b bits
// and |a - (lo' + s q)| <= s/2 (1 + 2^-30) (the fp64 evaluation, as in
// sngb_quant.cu).  For a pair and s' = s(1 + 2^-30), per coordinate
// |(a_j - b_j) - s(qa_j - qb_j)| <= s', hence over the k head coordinates
// (triangle inequality)  |a_h - b_h| >= s*sqrt(Q) - s'*sqrt(k),  Q = sum_h dq^2,
// and the full squared distance S >= |a_h - b_h|^2.  So
//     Q > B = ((sqrt(eps2 (1 + 2^-40)) + s' sqrt(k)) / s)^2   =>   S > eps2 (1 + 2^-40)
// and the reference's fp64 sum (within (d+1) 2^-53 S of S, distance.hpp:75-83)
// exceeds eps2: it rejects.  Q is exact for 8-bit heads (DP4A of |dq|) and fp32
// with two roundings for 16-bit ones (dq exact), so the kernel compares against
// B (1 + 2^-20) rounded up.  Pairs the head does not reject take the unchanged
// fp32 test (guard band, exact fp64 recheck in the band: sngb_epstest.cuh) on
// their fp32 rows.  Decisions are the reference's whatever the data; only the
// speed depends on how many pairs the head rejects (cfg5: ~95 %, the pairs from
// different clusters).
#include <cuda_runtime.h>

#include <cmath>
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "sngb_device.cuh"
#include "sngb_epstest.cuh"
#include "sngb_head.cuh"
#include "sngb_gather_head.cuh"
#include "sngb_internal.cuh"
#include "sngb_rng.cuh"


namespace sngb {

bool head_plan(double lo, double hi, uint32_t d, double eps2, int kind, HeadPlan& p) {
    const int bits = kind == kHeadU16x2 ? 16 : 8;
    const uint32_t k = std::min<uint32_t>(d, kind == kHeadU8x4 ? 4u : 2u);
    if (k < 2) return false;
    const double need = (hi - lo) / (std::ldexp(1.0, bits) - 2.0) * (1.0 + 1e-12);
    if (!(need > 0.0) || !std::isfinite(need)) return false;
    int e = 0;
    std::frexp(need, &e);  // need = m * 2^e, m in [0.5, 1)
    const double s = std::ldexp(1.0, e);
    p.s = s;
    p.lo = std::floor(lo / s) * s;
    p.args.kind = kind;
    p.args.coords = k;
    const double sp = s * (1.0 + std::ldexp(1.0, -30));
    const double e_hi = eps2 * (1.0 + std::ldexp(1.0, -40));
    const double tb = (std::sqrt(e_hi) + sp * std::sqrt((double)k)) / s;
    const double b = tb * tb * (1.0 + std::ldexp(1.0, -20));
    p.args.reject = std::nextafter((float)b, INFINITY);
    // useless if the rejection radius covers the data's whole range
    return std::sqrt(b) * s < 0.5 * (hi - lo) * std::sqrt((double)k);
}

namespace {

// thread per row: the first k values of the padded fp32 row -> the head word
template <int KIND>
__global__ void k_head_quantize(const float* __restrict__ pts, uint32_t stride, uint64_t n,
                                uint32_t k, double lo, double inv_s, void* __restrict__ out) {
    constexpr double qmax = KIND == kHeadU16x2 ? 65535.0 : 255.0;
    for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
         r += (uint64_t)gridDim.x * blockDim.x) {
        // stride >= 4 (d >= 3): the first 16 bytes of the row are in the table
        const float4 v = __ldg(reinterpret_cast<const float4*>(pts + r * stride));
        const float vs[4] = {v.x, v.y, v.z, v.w};
        uint32_t w = 0;
#pragma unroll
        for (int j = 0; j < (KIND == kHeadU8x4 ? 4 : 2); ++j) {
            const double x = rint(((double)vs[j] - lo) * inv_s);
            const uint32_t q = (uint32_t)j >= k ? 0u : (x <= 0.0 ? 0u : (x >= qmax ? (uint32_t)qmax : (uint32_t)x));
            w |= q << (j * (KIND == kHeadU16x2 ? 16 : 8));
        }
        if (KIND == kHeadU8x2) static_cast<uint16_t*>(out)[r] = (uint16_t)w;
        else static_cast<uint32_t*>(out)[r] = w;
    }
}

// k_gather_head: the body lives in sngb_gather_head.cuh (shared with k_duo).
template <int KIND, int G, int V, int R>
__global__ void __launch_bounds__(256, V >= 4 ? 2 : 4) k_gather_head(const GatherArgs a, const HeadArgs h) {
    __shared__ unsigned long long s_stage[kWarpsPerBlock][kStage];
    __shared__ uint32_t s_queue[kWarpsPerBlock][gather_head_qcap<G, R>()];
    gather_head_body<KIND, G, V, R>(a, h, &s_stage[0][0], &s_queue[0][0]);
}

template <int KIND, int G, int V, int R>
cudaError_t head_one(const GatherArgs& a, const HeadArgs& h, cudaStream_t s, int num_sms) {
    auto k = k_gather_head<KIND, G, V, R>;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 256, 0);
    if (per_sm < 1) per_sm = 1;
    // SNGB_GATHER_BPSM: cap the persistent grid (co-residency with the sampler)
    if (const char* e = std::getenv("SNGB_GATHER_BPSM"))
        if (std::atoi(e) > 0 && std::atoi(e) < per_sm) per_sm = std::atoi(e);
    const uint64_t rows = a.row_end - a.row_begin;
    const uint64_t want = (rows + kWarpsPerBlock - 1) / kWarpsPerBlock;
    const uint64_t cap = (uint64_t)num_sms * per_sm;
    k<<<(unsigned)(want < cap ? want : cap), 256, 0, s>>>(a, h);
    note_launch(1);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_head_quantize(const float* pts, uint32_t stride, uint64_t n, const HeadPlan& p,
                                 void* out, cudaStream_t s, int num_sms) {
    uint64_t blocks = (n + 255) / 256;
    if (blocks > (uint64_t)num_sms * 16) blocks = (uint64_t)num_sms * 16;
    const unsigned g = (unsigned)(blocks ? blocks : 1);
    const uint32_t k = p.args.coords;
    switch (p.args.kind) {
        case kHeadU16x2: k_head_quantize<kHeadU16x2><<<g, 256, 0, s>>>(pts, stride, n, k, p.lo, 1.0 / p.s, out); break;
        case kHeadU8x4: k_head_quantize<kHeadU8x4><<<g, 256, 0, s>>>(pts, stride, n, k, p.lo, 1.0 / p.s, out); break;
        default: k_head_quantize<kHeadU8x2><<<g, 256, 0, s>>>(pts, stride, n, k, p.lo, 1.0 / p.s, out); break;
    }
    note_launch(1);
    return cudaGetLastError();
}

namespace {
template <int KIND>
cudaError_t head_dispatch(const GatherArgs& a, const HeadArgs& h, cudaStream_t s, int num_sms) {
    const uint32_t W = a.tp.stride / 4;  // stride is a multiple of 4 for d >= 3
    constexpr int R = SNGB_HEAD_R;  // 32-draw chunks per step
    if (W <= 2) return head_one<KIND, 2, 1, R>(a, h, s, num_sms);
    if (W <= 4) return head_one<KIND, 4, 1, R>(a, h, s, num_sms);
    if (W <= 8) return head_one<KIND, 8, 1, R>(a, h, s, num_sms);
    if (W <= 16) return head_one<KIND, 16, 1, R>(a, h, s, num_sms);
    if (W <= 32) return head_one<KIND, 32, 1, R>(a, h, s, num_sms);
    if (W <= 64) return head_one<KIND, 32, 2, R>(a, h, s, num_sms);
    if (W <= 128) return head_one<KIND, 32, 4, 2>(a, h, s, num_sms);
    if (W <= 256) return head_one<KIND, 32, 8, 2>(a, h, s, num_sms);
    return cudaErrorInvalidValue;
}
}  // namespace

cudaError_t launch_gather_head(const GatherArgs& a, const HeadArgs& h, cudaStream_t s, int num_sms) {
    if (a.row_end <= a.row_begin) return cudaSuccess;
    switch (h.kind) {
        case kHeadU16x2: return head_dispatch<kHeadU16x2>(a, h, s, num_sms);
        case kHeadU8x4: return head_dispatch<kHeadU8x4>(a, h, s, num_sms);
        default: return head_dispatch<kHeadU8x2>(a, h, s, num_sms);
    }
}

}  // namespace sngb
