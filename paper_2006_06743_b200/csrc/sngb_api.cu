// sngb_api.cu -- the C ABI (include/sngb.h): validation, device pools,
// stage orchestration on one CUDA stream.
//
// Orchestration of sng::sng_dbscan (clusterer.cpp:54-65):
//   validate (clusterer.hpp:19-23, graph.cpp:17-21, dataset.hpp:21-27)
//   -> prepare points (padded fp32 layout, non-finite check)        [sync #1]
//   -> k_sampler (Floyd collisions)  -> k_gather (hot) -> k_extras
//   -> read cursors, retry with larger pools on overflow            [sync #2]
//   -> sort + unique (graph.cpp:34-40) -> cluster (clusterer.cpp:7-52)
//   -> read counters                                                [sync #3]
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <thread>
#include <atomic>
#include <string>
#include <vector>

#include "sngb.h"
#include "sngb_host.cuh"
#include "sngb_internal.cuh"
#include "sngb_rng.cuh"

using namespace sngb;

static thread_local uint64_t sngb_t_launch_hand = 0, sngb_t_launch_lib = 0;

void sngb::note_launch(int hand_written, int library) {
    sngb_t_launch_hand += hand_written;
    sngb_t_launch_lib += library;
}

namespace sngb {
namespace host {

thread_local std::string g_detail;
std::string& detail() { return g_detail; }
void reset_launches() {
    sngb_t_launch_hand = 0;
    sngb_t_launch_lib = 0;
}
uint64_t hand_launches() { return sngb_t_launch_hand; }
uint64_t lib_launches() { return sngb_t_launch_lib; }




std::mutex g_ctx_mu;
std::vector<std::unique_ptr<DevCtx>> g_ctx;


int device_count() {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

DevCtx& get_ctx(int dev, int slot) {
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    const size_t idx = (size_t)dev * kMaxSlots + (size_t)slot;
    if (g_ctx.size() <= idx) g_ctx.resize(idx + 1);
    if (!g_ctx[idx]) {
        auto c = std::make_unique<DevCtx>();
        c->dev = dev;
        CK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, dev));
        int l2 = 0;
        CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
        c->l2_bytes = (uint64_t)l2;
        CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        int prio_lo = 0, prio_hi = 0;
        CK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
        CK(cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, prio_lo));
        CK(cudaStreamCreateWithPriority(&c->hi, cudaStreamNonBlocking, prio_hi));
        CK(cudaEventCreateWithFlags(&c->hi_fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->hi_join, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->join, cudaEventDisableTiming));
        CK(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&c->qev, cudaEventDisableTiming));
        for (auto& e : c->sh_g) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        for (auto& e : c->sh_f) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->pev, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->up_start, cudaEventDisableTiming));
        for (auto& e : c->up_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CK(cudaMallocHost(&c->h_counters, C_COUNT * sizeof(unsigned long long)));
        CK(cudaMallocHost(&c->h_colstats, 2 * kQ8MaxD * sizeof(double)));
        CK(cudaMallocHost(&c->h_perm, kQ8MaxD * sizeof(uint32_t)));
        for (auto& e : c->ev) CK(cudaEventCreate(&e));
        g_ctx[idx] = std::move(c);
    }
    return *g_ctx[idx];
}

int resolve_device(const sngb_opts* o) {
    if (o && o->device >= 0) return o->device;
    int d = 0;
    cudaGetDevice(&d);
    return d;
}

// Test hook (see test_fire() in sngb_internal.cuh): forces the exact sequential
// replay on every m-th vertex so the parity tests reach it.  Compiled only into
// the test build lib/libsngb_testhooks.so (-DSNGB_TEST_HOOKS, build.py); the
// product library always returns 0 and never reads the variable.
uint32_t test_force_mod() {
#ifdef SNGB_TEST_HOOKS
    const char* v = std::getenv("SNGB_TEST_FORCE_IRREGULAR");
    return v ? (uint32_t)std::strtoul(v, nullptr, 10) : 0u;
#else
    return 0u;
#endif
}

uint64_t env_u64(const char* name, uint64_t dflt) {
    const char* v = std::getenv(name);
    return v ? (uint64_t)std::strtoull(v, nullptr, 10) : dflt;
}

uint32_t bits_for(uint64_t x) {  // bits needed to represent x (>= 1)
    uint32_t b = 1;
    while (b < 64 && (x >> b) != 0) ++b;
    return b;
}

// graph.cpp:139-140, same double expression.
uint64_t draws_for(uint64_t n, double rate) {
    const uint64_t c = static_cast<uint64_t>(std::ceil(rate * static_cast<double>(n)));
    return std::min<uint64_t>(c, n - 1);
}

float f32_down(double x) {
    float f = (float)x;
    if ((double)f > x) f = nextafterf(f, -INFINITY);
    return f;
}
float f32_up(double x) {
    float f = (float)x;
    if ((double)f < x) f = nextafterf(f, INFINITY);
    return f;
}

// Guard band for the fp32 eps test.  With u = 2^-24, every pair's fp32 sum
// s32 (diff rounding + at most d+5 rounded accumulations, fused or not)
// satisfies |s32 - S| <= ((1+u)^(2d+12) - 1) S + (2d+16) 2^-149 for the exact
// S; the reference's fp64 sum is within (d+1) 2^-53 S of S.  rel below
// over-covers both, so s32 < lo => ref accepts, s32 > hi => ref rejects.
// fp64 input (round_dist > 0): the fp32 rows are the caller's values rounded to
// nearest, |x32 - x| <= 2^-24 |x| + 2^-150, so the Euclidean distance of the
// rounded rows is within round_dist = sqrt(d) (2^-23 max|x| + 2^-149) of the
// true one; the accept / reject thresholds move by that much in distance.
TestParams make_test(const float* pts, uint32_t stride, uint32_t d, double eps,
                     double round_dist = 0.0, int32_t metric = kMetricEuclid,
                     double round_max = 0.0) {
    TestParams tp{};
    tp.pts = pts;
    tp.stride = stride;
    tp.d = d;
    tp.eps2 = eps * eps;
    tp.eps = eps;
    tp.metric = metric;
    const double u = std::ldexp(1.0, -24);
    if (metric == kMetricManhattan) {
        // |s32 - S| <= ((1+u)^(d+2) - 1) S + (d+2) 2^-149 for S = sum |a - b|, any
        // order; fp64 input moves each |a_k - b_k| by <= 2 (2^-24 max|x| + 2^-150)
        const double rel = 1.25 * (d + 2.0) * u + 1e-12;
        const double abs_ = (d + 2.0) * std::ldexp(1.0, -148);
        const double rl1 = round_max > 0.0
                               ? d * 2.0 * (std::ldexp(round_max, -24) + std::ldexp(1.0, -150)) *
                                     (1.0 + 1e-9)
                               : 0.0;
        const double ea = eps * (1.0 - 1e-12) - rl1, eb = eps * (1.0 + 1e-12) + rl1;
        tp.lo_thr = ea > 0.0 ? f32_down(ea * (1.0 - rel) - abs_) : -1.0f;
        tp.hi_thr = f32_up(eb * (1.0 + rel) + abs_);
        tp.eps2f = (float)eps;
        return tp;
    }
    if (metric == kMetricCosine) {
        // the filter value is x = -c32, c32 = dot32 / (|a|32 |b|32): |c32 - C| <=
        // 2 gamma_d + 6u (Cauchy-Schwarz bounds the dot's error by gamma_d |a||b|);
        // fp64 input: rounding each row moves C by <= 4u more (+ margin)
        const double gd = d * u / (1.0 - d * u);
        const double dc = 1.25 * (2.0 * gd + 6.0 * u) + (round_max > 0.0 ? 1.25 * 8.0 * u : 0.0);
        const double edge = eps - 1.0;  // x <= eps - 1  <=>  1 - c <= eps
        tp.lo_thr = f32_down(edge - 1e-12 - dc);
        tp.hi_thr = f32_up(edge + 1e-12 + dc);
        tp.eps2f = (float)edge;
        return tp;
    }
    const double rel = (2.0 * d + 16.0) * std::ldexp(1.0, -24) * 1.25 + 1e-12;
    const double abs_ = (2.0 * d + 16.0) * std::ldexp(1.0, -148);
    const double ea = std::sqrt(tp.eps2) * (1.0 - 1e-12) - round_dist;  // accept below (distance)
    const double eb = std::sqrt(tp.eps2) * (1.0 + 1e-12) + round_dist;  // reject above
    const double lo = round_dist > 0.0 ? (ea > 0.0 ? ea * ea * (1.0 - rel) - abs_ : -1.0)
                                       : tp.eps2 * (1.0 - rel) - abs_;
    const double hi = round_dist > 0.0 ? eb * eb * (1.0 + rel) + abs_ : tp.eps2 * (1.0 + rel) + abs_;
    tp.lo_thr = lo > 0 ? f32_down(lo) : 0.0f;
    tp.hi_thr = hi < (double)FLT_MAX / 4 ? f32_up(hi) : INFINITY;
    tp.eps2f = (float)tp.eps2;
    return tp;
}

// Distance::within metric from opts->flags (SNGB_FLAG_MANHATTAN / _COSINE)
int32_t metric_of(const sngb_opts* o) {
    const uint32_t f = o ? o->flags : 0u;
    if (f & SNGB_FLAG_MANHATTAN) return kMetricManhattan;
    if (f & SNGB_FLAG_COSINE) return kMetricCosine;
    return kMetricEuclid;
}
bool metric_flags_ok(const sngb_opts* o) {
    const uint32_t f = o ? o->flags : 0u;
    return !((f & SNGB_FLAG_MANHATTAN) && (f & SNGB_FLAG_COSINE));
}

int validate(uint64_t n, uint32_t d, double eps, int32_t min_pts, double rate, bool need_minpts) {
    if (need_minpts) {
        // sng_dbscan: SngParams::validate first (clusterer.hpp:19-23: eps, min_pts,
        // rate), then build_sampled_graph's checks (graph.cpp:17-21: empty, dim)
        if (!(eps > 0.0)) return SNGB_ERR_EPS;
        if (min_pts < 1) return SNGB_ERR_MINPTS;
        if (!(rate > 0.0) || rate > 1.0) return SNGB_ERR_RATE;
        if (n == 0) return SNGB_ERR_EMPTY;
        if (d == 0) return SNGB_ERR_DIM;
    } else {
        // build_sampled_graph alone: validate_graph_params (graph.cpp:17-21: empty,
        // eps, dim), then the rate (graph.cpp:136)
        if (n == 0) return SNGB_ERR_EMPTY;
        if (!(eps > 0.0)) return SNGB_ERR_EPS;
        if (d == 0) return SNGB_ERR_DIM;
        if (!(rate > 0.0) || rate > 1.0) return SNGB_ERR_RATE;
    }
    if (n >= 0xffffff00ull) return SNGB_ERR_TOO_LARGE;
    return SNGB_OK;
}



// Number of L2-blocked gather phases.  A phase re-generates every draw
// (~0.35 SM-cycles each) and re-streams the query rows, and in exchange turns
// the partner gather into L2 hits; it pays while the row table is a small
// multiple of L2 and the rows are wide (cfg2: 219.5 MB of 3136-byte rows).
// Env SNGB_GATHER_PHASES forces a count; SNGB_L2_PHASE_BYTES sets the slice.
uint32_t gather_phases(const DevCtx& c, uint64_t n, uint32_t stride, uint64_t draws) {
    const uint64_t forced = env_u64("SNGB_GATHER_PHASES", 0);
    if (forced) return (uint32_t)std::min<uint64_t>(forced, std::max<uint64_t>(n, 1));
    const uint64_t table = n * stride * 4ull;
    const uint64_t slice = env_u64("SNGB_L2_PHASE_BYTES", (uint64_t)(0.5 * c.l2_bytes));
    if (slice == 0 || table <= slice || stride < 64 || draws == 0) return 1;
    // a phase re-generates every draw: ~1.2e-12 s per pair against ~2.3e-13*d s
    // of gather, so wider rows afford more phases (d = 1000: 0.5 % each)
    const uint64_t p = (table + slice - 1) / slice;
    const uint64_t cap = std::min<uint64_t>(16, std::max<uint64_t>(2, stride / 32));
    return p <= cap ? (uint32_t)p : 1u;
}


// Prepare points and run the graph build for rows [rb, re).  Leaves sorted
// unique compact keys in c.keys/keys_alt and their count in
// counters[C_UNIQUE] (device); one host sync (edge/extras counts, non-finite
// check).  With h_src, d_pts is an uninitialised device buffer of n x d floats
// that this call fills from the host in row chunks on c.copy, overlapped with
// the sampler and (L2-blocked case) with the gather of the chunks already in.
int build_graph(DevCtx& c, cudaStream_t s, Timer& tm, const float* d_pts, uint64_t n, uint32_t d,
                double eps, double rate, uint64_t seed, uint64_t rb, uint64_t re,
                GraphResult& gr, const float* h_src, const double* d_pts64, int32_t metric,
                bool upper_only) {
    unsigned long long* dc = nullptr;
    c.counters.ensure(C_COUNT * sizeof(unsigned long long));
    dc = c.counters.as<unsigned long long>();
    CK(cudaMemsetAsync(dc, 0, C_COUNT * sizeof(unsigned long long), s));

    // ---- points: padded device layout + finiteness (dataset.hpp:24-26) ----
    // The non-finite count is checked at the one host sync below (a rejected
    // dataset costs a wasted graph build, never a wrong answer: NaN rows fail
    // every eps-test).
    const uint32_t stride = d <= 2 ? 2u : ((d + 3u) & ~3u);
    const size_t align = stride == 2 ? 8 : 16;
    const bool f64 = d_pts64 != nullptr;  // fp64 input: rounded into the padded fp32 table
    const bool pad = f64 || stride != d || (reinterpret_cast<uintptr_t>(d_pts) % align) != 0;
    if (pad) c.pts.ensure(n * stride * sizeof(float));
    const float* pts = pad ? c.pts.as<float>() : d_pts;
    cudaStream_t gs = s;  // the gather's stream (c.hi under SNGB_PRIO)
    bool q8_try = false;  // wide rows: min/max for the 8-bit filter (sngb_quant.cu)
    bool head_try = false;  // narrow rows beyond L2: the head filter (sngb_head.cu)
    auto prepare_rows = [&](uint64_t lo, uint64_t hi) {
        if (hi <= lo) return;
        if (f64)
            CK(launch_prepare_points_f64(d_pts64 + lo * d, c.pts.as<float>() + lo * stride,
                                         hi - lo, d, stride, dc, gs));
        else
            CK(launch_prepare_points(d_pts + lo * d, pad ? c.pts.as<float>() + lo * stride : nullptr,
                                     hi - lo, d, stride, dc, q8_try || head_try, gs));
    };
    // after the last prepare: the min/max to the host, waited for only when the
    // 8-bit plan is made (the sampler is already running by then)
    // With the 8-bit filter also the per-column statistics of the rows prepared so
    // far (rows_ready): the head then holds the columns of largest variance.
    bool perm_try = false;
    uint64_t stats_rows = 0;
    auto minmax_to_host = [&](uint64_t rows_ready) {
        if (perm_try) {
            // the order of the column variances from a sample of the rows (the
            // first 8192: a full pass measured 60-110 us on cfg2's critical path)
            rows_ready = std::min<uint64_t>(rows_ready, 8192);
            CK(launch_colstats(pts, stride, rows_ready, d, d_pts64, c.colstats.as<double>(), gs,
                               c.num_sms));
            CK(cudaMemcpyAsync(c.h_colstats, c.colstats.p, 2ull * d * sizeof(double),
                               cudaMemcpyDeviceToHost, gs));
            stats_rows = rows_ready;
        }
        CK(cudaMemcpyAsync(&c.h_counters[C_QMIN], &dc[C_QMIN], 2 * sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, gs));
        // this call's non-finite count too (the filter plans read it; a stale value
        // from an earlier failed call must not switch the filters off)
        CK(cudaMemcpyAsync(&c.h_counters[C_NONFINITE], &dc[C_NONFINITE],
                           sizeof(unsigned long long), cudaMemcpyDeviceToHost, gs));
        CK(cudaEventRecord(c.qev, gs));
    };

    // ---- sampling geometry (graph.cpp:138-140) ----
    const uint64_t draws = draws_for(n, rate);
    const bool exhaustive = draws >= n - 1;
    // SNGB_Q8: 0 off, 1 auto (use when the band is narrow), 2 force (tests)
    const uint64_t q8_mode = env_u64("SNGB_Q8", 1);
    // the 8-bit gathers hold a row in <= 3 chunks per lane: d <= 16 * (3 * 32 - 1)
    q8_try = metric == kMetricEuclid && !exhaustive && d >= 128 && d <= kQ8MaxD && q8_mode != 0;
    perm_try = q8_try && env_u64("SNGB_Q8_PERM", 1) != 0;  // variance-ordered columns
    if (perm_try) c.colstats.ensure(2ull * d * sizeof(double));
    // SNGB_HEAD: 0 off, 1 auto, 2 force (tests); SNGB_HEAD_KIND picks the format.
    // Auto for large problems whose head table stays L2-resident (a table read
    // by every SM keeps about half the L2): 4-byte heads up to 0.4 L2, 2-byte
    // heads (cfg5) up to twice that many rows.  fp32 input only (fp64 rows would
    // need their rounding bound in the head too).
    const uint64_t head_mode = env_u64("SNGB_HEAD", 1);
    int head_kind = -1;
    {
        const uint64_t budget = c.l2_bytes * 2 / 5;
        head_kind = n * 4ull <= budget ? kHeadDefault4 : (n * 2ull <= budget ? kHeadU8x2 : -1);
        const uint64_t forced = env_u64("SNGB_HEAD_KIND", 99);
        if (forced <= 2) head_kind = (int)forced;
        if (head_mode == 2 && head_kind < 0) head_kind = kHeadU8x2;
        head_try = metric == kMetricEuclid && !exhaustive && !q8_try && d_pts64 == nullptr &&
                   d >= 3 && d <= 1024 && n >= 2 && head_kind >= 0 &&
                   (head_mode == 2 || (head_mode == 1 && n >= 65536));
    }
    const uint64_t rows = re - rb;
    const uint32_t nb = bits_for(n - 1);
    const uint64_t base = (n - 1) - draws;
    gr.draws = draws;
    gr.exhaustive = exhaustive;
    gr.nb = nb;

    // ---- capacities ----
    uint64_t pairs;
    if (exhaustive) {
        // rows [rb, re) pair with all v > u, and (a partial range) with all v < rb
        const double sum = (double)rows * (double)(n - 1) - ((double)re * (re - 1) - (double)rb * (rb - 1)) / 2.0;
        pairs = (uint64_t)std::max(0.0, sum) + (upper_only ? 0 : rows * rb);
    } else {
        pairs = rows * draws;
    }
    // expected Floyd collisions per vertex, sum_i i / (base + i + 1), bounded above
    // in closed form by D(D-1) / 2(base + 1) (a per-call loop over the draws
    // cost ~15 us of host time on cfg2, 80 us on cfg5)
    const double exp_col =
        exhaustive ? 0.0
                   : std::min((double)draws,
                              (double)draws * ((double)draws - 1.0) / (2.0 * ((double)base + 1.0)));
    uint64_t extras_cap =
        exhaustive ? 0 : (uint64_t)(1.5 * exp_col * (double)rows) + 4096 + 4 * draws;
    uint64_t edge_cap = std::min<uint64_t>(pairs + extras_cap + 1, std::max<uint64_t>(1ull << 24, pairs / 8));
    edge_cap = std::min<uint64_t>(edge_cap, 1ull << 28);
    edge_cap = std::max<uint64_t>(edge_cap, std::min<uint64_t>(c.edge_hint, pairs + extras_cap + 1));

    // Floyd tables (k_floyd, one block per vertex)
    uint32_t slots = 64, col_words = 4;
    if (!exhaustive) floyd_geometry((uint32_t)draws, slots, col_words);

    // fp64 input: the fp32 thresholds need max|x| before any test runs
    double round_dist = 0.0, max_abs = 0.0;
    if (f64) {
        prepare_rows(0, n);
        minmax_to_host(n);
        CK(cudaEventSynchronize(c.qev));
        const double lo = ordered_value64(~c.h_counters[C_QMIN]);
        const double hi = ordered_value64(c.h_counters[C_QMAX]);
        const double m = std::max(std::fabs(lo), std::fabs(hi));
        max_abs = m;
        round_dist = std::sqrt((double)d) * (std::ldexp(m, -23) + std::ldexp(1.0, -149)) *
                     (1.0 + 1e-9);
    }
    TestParams tp = make_test(pts, stride, d, eps, round_dist, metric, max_abs);
    tp.pts64 = d_pts64;
    if (metric == kMetricCosine) {
        c.rnorm.ensure(n * sizeof(float));
        tp.rnorm = c.rnorm.as<float>();
    }
    bool norms_done = metric != kMetricCosine;
    auto ensure_norms = [&]() {  // after the last prepare, before any cosine test
        if (norms_done) return;
        CK(launch_row_norms(tp, n, c.rnorm.as<float>(), dc, gs, c.num_sms));
        norms_done = true;
    };
    const uint64_t seed_mixed = seed_part(seed);
    const uint32_t phases = gather_phases(c, n, stride, draws);

    // ---- host upload in row chunks (chunk k = L2 phase k when phased) ----
    // (other metrics: one chunk -- the cosine row norms need every row first)
    // With the 8-bit filter (its table is L2-resident whole) the chunk count only
    // sets the triangle's granularity: finer chunks start the gather sooner and
    // leave less of it behind the last chunk (SNGB_Q8_CHUNKS, default 8).
    uint32_t chunks =
        h_src && metric == kMetricEuclid ? std::min<uint32_t>(phases, DevCtx::kMaxChunks) : 1;
    if (h_src && q8_try && n * d * 4ull >= (8ull << 20))
        chunks = (uint32_t)std::min<uint64_t>(
            std::max<uint64_t>(env_u64("SNGB_Q8_CHUNKS", 8), 1), DevCtx::kMaxChunks);
    auto chunk_lo = [&](uint32_t k) { return n * k / chunks; };
    // Host-upload 8-bit schedule: each landed slice k is tested against every
    // earlier row, which regenerated all of their draws per launch; instead the
    // draws' partners are bucketed by slice once, on the side stream while the
    // first chunk uploads (no point data needed), and each launch reads only
    // its slices' lists (SNGB_PARTNERS=0: regenerate)
    const bool pre_partners = h_src && q8_try && chunks > 1 && !exhaustive &&
                              q8_split((d + 15) / 16) && draws <= 1024 &&
                              (re - rb) * draws * 4ull <= (2ull << 30) &&
                              env_u64("SNGB_PARTNERS", 1) != 0;
    // issued after the sampler launch: a pageable source blocks the host while
    // it is staged, and the sampler should already be running by then
    auto start_upload = [&]() {
        CK(cudaEventRecord(c.up_start, s));  // after the caller's prior work on s
        CK(cudaStreamWaitEvent(c.copy, c.up_start, 0));
        for (uint32_t k = 0; k < chunks; ++k) {
            const uint64_t lo = chunk_lo(k), hi = chunk_lo(k + 1);
            CK(cudaMemcpyAsync(const_cast<float*>(d_pts) + lo * d, h_src + lo * d,
                               (hi - lo) * d * sizeof(float), cudaMemcpyHostToDevice, c.copy));
            CK(cudaEventRecord(c.up_ev[k], c.copy));
        }
        tm.mark_on(E_UPLOADED, c.copy);
    };
    // side_pre: the sampler on the side stream while this stream prepares the
    // points, waits for the filter plan and quantises; the gather then waits for
    // the sampler (run together they slow the gather more than they gain).  The
    // fork is recorded here, before the prepare pass.
    // Floyd bookkeeping fused into the head gather (sngb_fused.cu: every draw
    // generated once) when the head filter runs; the head plan decides, so the
    // sampler launch is held back until then
    const bool fuse_try = head_try && !exhaustive && fused_eligible(n, draws, stride);
    // shared draws: the head gather writes its draws, k_floyd_pipe reads them (the
    // sampler launch is held back until the head plan is known, as for fuse_try)
    const bool share_try =
        head_try && !exhaustive && !fuse_try && share_eligible(n, (uint32_t)draws);
    const bool side_pre = !exhaustive && !fuse_try && !share_try && !h_src && (q8_try || head_try) &&
                          !(stride <= 64 && (re - rb) >= 10000 && draws <= 1024) &&  // not overlap
                          env_u64("SNGB_OVERLAP", 2) != 1 && env_u64("SNGB_SIDE_PRE", 1) != 0;
    if (side_pre) CK(cudaEventRecord(c.fork, s));
    if (!h_src && !f64) {
        prepare_rows(0, n);
        if (q8_try || head_try) minmax_to_host(n);
    }
    tm.mark(E_PREPARED);
    bool q8_on = false, head_on = false;
    Q8Plan q8p{};
    HeadPlan hp{};
    uint32_t gphases = phases;  // partner slices of the gather (8-bit rows: their own count)
    // host upload state: leading chunks prepared / quantised on gs.  With the
    // 8-bit filter the plan is made from chunk 0 (q8_pipe) so the gather can
    // start while the rest uploads; the final sync checks that every value
    // fits the plan's range, else the build is redone with a global plan.
    uint32_t prepared = h_src ? 0 : chunks, quantized = 0;
    bool q8_pipe = false, q8_replan = false;

    // band list (pairs the filter cannot decide, resolved exactly by k_band)
    uint64_t band_cap = std::max<uint64_t>(1ull << 16, std::min<uint64_t>(pairs / 4096, 1ull << 24));
    band_cap = std::max<uint64_t>(band_cap, c.band_hint);
    for (int attempt = 0; attempt < 4; ++attempt) {
        c.keys.ensure(edge_cap * 8);
        c.band.ensure(band_cap * 16);
        tp.band = c.band.as<uint4>();
        tp.band_cursor = &dc[C_BAND_CURSOR];
        tp.band_cap = band_cap;
        c.extras.ensure(std::max<uint64_t>(extras_cap, 1) * 8);
        if (attempt > 0)
        {
            CK(cudaMemsetAsync(dc, 0, C_UNIQUE * sizeof(unsigned long long), s));
            CK(cudaMemsetAsync(&dc[C_BAND_CURSOR], 0, sizeof(unsigned long long), s));
            CK(cudaMemsetAsync(&dc[C_IRR_CURSOR], 0, sizeof(unsigned long long), s));
        }
        tm.mark(E_PREPARED);
        // Overlap: the sampler on the side stream concurrently with the
        // persistent, dynamically claimed gather (SNGB_OVERLAP 0 off, 1 on, 2
        // auto).  Auto for narrow-row problems of >= 10 k rows: cfg1 0.82 ->
        // 0.79 ms, cfg3-5 within 1 % of sequential (cfg5 668 vs 686 ms with
        // dynamic claiming, which a non-persistent gather grid lost); wide-row
        // problems run the sampler beside prepare/plan/quantise instead.
        const uint64_t ov = env_u64("SNGB_OVERLAP", 2);
        // (with the 4-block Floyd filter kernel and 32 rows per sampler block, draws >
        // 1024 lost: its blocks then crowd the gather's -- cfg5 876 vs 646 ms, cfg4 130
        // vs 96 ms; 8 rows per block win: cfg5 636 vs 656 ms, cfg4 92.5 vs 95.9 ms,
        // profiles/r02_overlap_rpb_cfg*.jsonl)
        const bool overlap =
            !exhaustive && (ov == 1 || (ov == 2 && stride <= 64 && (re - rb) >= 10000));
        // host upload: the sampler reads no points, so it also runs while they arrive
        const bool side = !exhaustive && !fuse_try && !share_try &&
                          (overlap || side_pre || (h_src && attempt == 0));
        if (pre_partners && attempt == 0) {  // before the sampler on the side stream
            c.partners.ensure((re - rb) * draws * 4ull);
            c.poff.ensure((re - rb) * (chunks + 1) * 4ull);
            GatherArgs pa{};
            pa.n = n;
            pa.row_begin = rb;
            pa.row_end = re;
            pa.draws = (uint32_t)draws;
            pa.base = (uint32_t)base;
            pa.seed_mixed = seed_mixed;
            pa.force_mod = test_force_mod();
            pa.nbuckets = chunks;
            CK(launch_partners(pa, c.partners.as<uint32_t>(), c.poff.as<uint32_t>(), c.side,
                               c.num_sms));
            CK(cudaEventRecord(c.pev, c.side));
        }
        auto make_sa = [&]() {
            SamplerArgs sa{};
            sa.n = n;
            sa.row_begin = rb;
            sa.row_end = re;
            sa.draws = (uint32_t)draws;
            sa.base = (uint32_t)base;
            sa.seed_mixed = seed_mixed;
            sa.force_mod = test_force_mod();
            const size_t scratch = fuse_try ? fused_scratch_bytes((uint32_t)draws, re - rb, c.num_sms)
                                            : floyd_scratch_bytes((uint32_t)draws, c.num_sms, re - rb);
            if (scratch) c.scratch.ensure(scratch);
            sa.scratch64 = scratch ? c.scratch.as<unsigned long long>() : nullptr;
            sa.extras = c.extras.as<unsigned long long>();
            sa.extras_capacity = extras_cap;
            sa.counters = dc;
            return sa;
        };
        if (!exhaustive && !fuse_try && !share_try) {
            SamplerArgs sa = make_sa();
            if (side) {
                // the Floyd bookkeeping needs no point data: run it on the side
                // stream while the gather runs here; non-persistent grids let the
                // block scheduler interleave the two kernels on every SM
                // non-persistent beside the gather (and during a host upload, where the
                // gather starts while it runs: cfg5 e2e 614 vs 943 ms persistent; 32
                // rows per block there, 625 vs 639 ms with 8)
                // (k_floyd_pipe: 64 rows per block, two drain steps each; cfg5 602 vs
                // 609 ms with 8, 630 ms persistent.  k_floyd_lean likes them too now that
                // it gains nothing beside the gather: cfg4 82.8 vs 84.7 ms with 8,
                // profiles/r02_lean_rpb_cfg4.jsonl)
                sa.rows_per_block = (uint32_t)env_u64(
                    "SNGB_SAMPLER_RPB",
                    draws > 1024 && draws <= 4096 ? 64 : (h_src ? 32 : (overlap ? 32 : 0)));
                if (!(side_pre && attempt == 0)) CK(cudaEventRecord(c.fork, s));
                CK(cudaStreamWaitEvent(c.side, c.fork, 0));
                tm.mark_on(E_SIDE0, c.side);
                CK(launch_sampler(sa, c.side, c.num_sms));
                tm.mark_on(E_SIDE1, c.side);
                tm.side = true;
                CK(cudaEventRecord(c.join, c.side));
            } else {
                if (sampler_uses_pipe(n, (uint32_t)draws) || (draws > 1024 && draws <= 4096))
                    sa.rows_per_block = (uint32_t)env_u64("SNGB_SAMPLER_RPB", 64);
                CK(launch_sampler(sa, s, c.num_sms));
            }
        }
        if (h_src && attempt == 0) start_upload();
        auto quantize_rows = [&](uint64_t r0, uint64_t r1) {
            if (r1 > r0)
                CK(launch_quantize(pts + r0 * stride, stride, r1 - r0, d, q8p,
                                   c.q8.as<uint4>() + r0 * (q8p.args.nd + 1), gs, c.num_sms,
                                   f64 ? d_pts64 + r0 * d : nullptr));
        };
        if ((q8_try || head_try) && (attempt == 0 || q8_replan)) {
            const bool pipe = q8_try && h_src && attempt == 0 && chunks > 1;
            if (h_src && attempt == 0) {
                const uint32_t upto = pipe ? 1 : chunks;
                for (uint32_t k = prepared; k < upto; ++k) {
                    CK(cudaStreamWaitEvent(gs, c.up_ev[k], 0));
                    prepare_rows(chunk_lo(k), chunk_lo(k + 1));
                }
                prepared = upto;
                minmax_to_host(chunk_lo(upto));
            }
            // a re-plan reads the global min/max kept in h_counters by the last sync
            if (!q8_replan) CK(cudaEventSynchronize(c.qev));
            const double lo = f64 ? ordered_value64(~c.h_counters[C_QMIN])
                                  : (double)ordered_value(~(uint32_t)c.h_counters[C_QMIN]);
            const double hi = f64 ? ordered_value64(c.h_counters[C_QMAX])
                                  : (double)ordered_value((uint32_t)c.h_counters[C_QMAX]);
            if (head_try) {
                const bool useful = head_plan(lo, hi, d, tp.eps2, head_kind, hp);
                head_on = !c.h_counters[C_NONFINITE] && (useful || (head_mode == 2 && hp.s > 0));
                gr.head = head_on ? (head_kind == kHeadU8x2 ? 2u : 4u) : 0u;
                if (head_on) {
                    // the head table (exclusive with the 8-bit rows)
                    // (+16: the fused kernel copies 2-byte heads as aligned 4-byte words)
                    c.q8.ensure(n * (head_kind == kHeadU8x2 ? 2ull : 4ull) + 16);
                    hp.args.head = c.q8.p;
                    CK(launch_head_quantize(pts, stride, n, hp, c.q8.p, gs, c.num_sms));
                    gphases = 1;  // the fp32 rows are read by survivors only
                }
            }
            const bool useful = q8_try && q8_plan(lo, hi, d, tp.eps2, q8p);
            q8_on = q8_try && !c.h_counters[C_NONFINITE] && (useful || (q8_mode == 2 && q8p.s > 0));
            gr.q8 = q8_on;
            q8_pipe = q8_on && pipe;
            q8_replan = false;
            if (!head_on) gphases = phases;
            if (q8_on && perm_try && stats_rows > 0 && !q8_replan) {
                // column order by decreasing variance (stable): the head's 240 values
                // are the most spread-out coordinates (a real image's constant
                // borders go last); any order is exact
                const double m = (double)stats_rows;
                std::vector<double> var(d);
                for (uint32_t k = 0; k < d; ++k) {
                    const double mu = c.h_colstats[k] / m;
                    var[k] = c.h_colstats[d + k] / m - mu * mu;
                }
                std::vector<uint32_t> order(d);
                for (uint32_t k = 0; k < d; ++k) order[k] = k;
                std::stable_sort(order.begin(), order.end(),
                                 [&](uint32_t x, uint32_t y) { return var[x] > var[y]; });
                bool identity = true;
                for (uint32_t k = 0; k < d; ++k) {
                    c.h_perm[k] = order[k];
                    identity = identity && order[k] == k;
                }
                // worth a permuted quantisation only if the natural head holds
                // much less variance than the best one (an image's blank border;
                // cfg2's iid columns: no -- there it costs the step 0.1 ms)
                double nat = 0.0, best = 0.0;
                for (uint32_t k = 0; k < std::min<uint32_t>(d, kHeadVals); ++k) {
                    nat += std::max(0.0, var[k]);
                    best += std::max(0.0, var[order[k]]);
                }
                if (nat >= 0.5 * best) identity = true;
                q8p.perm = nullptr;
                if (!identity) {
                    c.perm.ensure(d * sizeof(uint32_t));
                    CK(cudaMemcpyAsync(c.perm.p, c.h_perm, d * sizeof(uint32_t),
                                       cudaMemcpyHostToDevice, gs));
                    q8p.perm = c.perm.as<uint32_t>();
                }
            }
            if (q8_on) {
                const uint32_t nd = (d + 15) / 16;
                c.q8.ensure(n * (nd + 1) * 16ull);
                q8p.args.rows = c.q8.as<uint4>();
                q8p.args.nd = nd;
                if (q8_pipe) {  // chunk 0 now, the others as they arrive
                    quantize_rows(0, chunk_lo(1));
                    quantized = 1;
                    gphases = chunks;
                } else {
                    quantize_rows(0, n);
                    quantized = chunks;
                    gphases = gather_phases(c, n, 4 * (nd + 1), draws);
                }
            }
        }
        if (side_pre) CK(cudaStreamWaitEvent(s, c.join, 0));  // gather after the sampler
        const bool fused = fuse_try && head_on;
        if (fuse_try && !head_on) CK(launch_sampler(make_sa(), s, c.num_sms));  // unfused after all
        const bool share = share_try && head_on && gphases == 1;
        if (share_try && !share) CK(launch_sampler(make_sa(), s, c.num_sms));  // no head filter after all
        tm.mark(E_SAMPLED);
        GatherArgs ga{};
        ga.tp = tp;
        ga.sink = EdgeSink{c.keys.as<unsigned long long>(), edge_cap, &dc[C_EDGE_CURSOR], nb};
        ga.counters = dc;
        ga.n = n;
        ga.row_begin = rb;
        ga.row_end = re;
        ga.draws = (uint32_t)draws;
        ga.base = (uint32_t)base;
        ga.seed_mixed = seed_mixed;
        ga.force_mod = test_force_mod();
        ga.rows_per_block = (uint32_t)env_u64("SNGB_GATHER_RPB", 0);
        if (pre_partners && q8_on) CK(cudaStreamWaitEvent(gs, c.pev, 0));
        // dynamic row claiming (persistent grid): one zeroed counter per launch
        constexpr uint32_t kWorkSlots = 256;
        const bool dyn = ga.rows_per_block == 0 && env_u64("SNGB_GATHER_DYN", 1) == 1;
        uint32_t work_slot = 0;
        if (dyn || fused) {
            c.work.ensure(kWorkSlots * 8);
            CK(cudaMemsetAsync(c.work.p, 0, kWorkSlots * 8, s));
        }
        // SNGB_PRIO=1: gather on a high-priority stream, so the block scheduler
        // prefers its blocks and the (low-priority) sampler fills the gaps
        const bool prio = side && env_u64("SNGB_PRIO", 0) == 1;
        if (prio) {
            CK(cudaEventRecord(c.hi_fork, s));
            CK(cudaStreamWaitEvent(c.hi, c.hi_fork, 0));
            gs = c.hi;
        }
        // L2-blocked phases: each launch tests only partners in one slice of
        // the rows, small enough to stay L2-resident while every vertex's
        // draws are regenerated (cheap) and its query row streamed.
        auto part = [&](uint32_t ph) { return (uint32_t)(n * ph / gphases); };
        auto gather = [&](uint64_t qlo, uint64_t qhi, uint32_t plo, uint32_t phi) {
            ga.row_begin = std::max(rb, qlo);
            ga.row_end = std::min(re, qhi);
            ga.part_lo = plo;
            ga.part_hi = phi;
            if (ga.row_end <= ga.row_begin) return;
            ga.partners = nullptr;
            if (pre_partners && q8_on) {  // the launch's slices, if on bucket boundaries
                const uint32_t blo = (uint32_t)((uint64_t)plo * chunks / n);
                const uint32_t bhi = (uint32_t)((uint64_t)phi * chunks / n);
                if (chunk_lo(blo) == plo && chunk_lo(bhi) == phi) {
                    ga.partners = c.partners.as<uint32_t>();
                    ga.poff = c.poff.as<uint32_t>();
                    ga.partners_row0 = rb;
                    ga.nbuckets = chunks;
                    ga.blo = blo;
                    ga.bhi = bhi;
                }
            }
            ga.work = nullptr;
            if (dyn && work_slot < kWorkSlots) {
                ga.work = c.work.as<unsigned long long>() + work_slot++;
                // ~16 claims per resident warp, at most 32 rows per claim
                const uint64_t warps = (uint64_t)c.num_sms * 64;
                ga.grab = (uint32_t)std::max<uint64_t>(
                    1, std::min<uint64_t>(32, (ga.row_end - ga.row_begin) / (warps * 16)));
            }
            if (q8_on) CK(launch_gather_q8(ga, q8p.args, gs, c.num_sms));
            else if (head_on) CK(launch_gather_head(ga, hp.args, gs, c.num_sms));
            else if (metric != kMetricEuclid || d > 1024)
                CK(launch_gather_metric(ga, exhaustive, gs, c.num_sms));
            else CK(launch_gather(ga, exhaustive, gs, c.num_sms));
        };
        auto land_chunk = [&](uint32_t k) {  // chunk k uploaded, prepared, quantised
            if (k >= prepared) {
                CK(cudaStreamWaitEvent(gs, c.up_ev[k], 0));
                prepare_rows(chunk_lo(k), chunk_lo(k + 1));
            }
            if (q8_on && k >= quantized) quantize_rows(chunk_lo(k), chunk_lo(k + 1));
        };
        if (h_src && attempt == 0 && prepared < chunks && chunks == gphases && gphases > 1) {
            // triangular schedule over (query chunk, partner slice) blocks:
            // once chunk k is in, every block it completes can run -- queries
            // <= k against slice k, then chunk k against the earlier slices
            for (uint32_t k = 0; k < gphases; ++k) {
                land_chunk(k);
                gather(0, part(k + 1), part(k), part(k + 1));
                if (q8_on) {  // the 8-bit table is L2-resident whole: one launch for the rest
                    if (k > 0) gather(part(k), part(k + 1), 0, part(k));
                } else {      // fp32: one L2 slice of partners per launch
                    for (uint32_t j = 0; j < k; ++j) gather(part(k), part(k + 1), part(j), part(j + 1));
                }
            }
            prepared = quantized = chunks;
        } else {
            if (h_src && attempt == 0)
                for (uint32_t k = 0; k < chunks; ++k) land_chunk(k);
            prepared = quantized = chunks;
            ensure_norms();
            if (fused) {  // Floyd bookkeeping + head gather in one kernel
                ga.row_begin = rb;
                ga.row_end = re;
                ga.part_lo = 0;
                ga.part_hi = (uint32_t)n;
                ga.partners = nullptr;
                ga.work = c.work.as<unsigned long long>() + work_slot++;
                ++work_slot;  // k_duo's Floyd chunk counter (ga.work + 1)
                CK(launch_floyd_head(make_sa(), ga, hp.args, gs, c.num_sms));
            } else if (share) {
                // Row chunks through a bounded draw buffer: the gather of chunk k on this
                // stream writes buffer k & 1, the Floyd pass of chunk k on the side stream
                // reads it while the gather of chunk k + 1 runs (two buffers, events).
                const uint64_t rows = re - rb, per_row = draws * 4ull;
                size_t free_b = 0, total_b = 0;
                CK(cudaMemGetInfo(&free_b, &total_b));
                uint64_t budget = env_u64("SNGB_TBUF_MB", 4096) << 20;  // per buffer
                budget = std::min<uint64_t>(budget, (free_b + c.tbuf.bytes) / 4);
                uint64_t crow = std::max<uint64_t>(budget / per_row, 1024);
                crow = std::max<uint64_t>(crow, (rows + 199) / 200);  // <= 200 chunks (work slots)
                crow = std::min<uint64_t>(crow, rows);
                const uint64_t nchunks = (rows + crow - 1) / crow;
                const uint32_t nbuf = nchunks > 1 ? 2 : 1;
                c.tbuf.ensure(nbuf * crow * per_row);
                c.tflags.ensure(nbuf * crow);
                const bool serial = env_u64("SNGB_SHARE_SERIAL", 0) == 1;
                cudaStream_t fs = serial ? gs : c.side;
                for (uint64_t k = 0; k < nchunks; ++k) {
                    const uint32_t b = (uint32_t)(k & (nbuf - 1));
                    const uint64_t r0 = rb + k * crow, r1 = std::min<uint64_t>(re, r0 + crow);
                    if (k >= 2 && !serial) CK(cudaStreamWaitEvent(gs, c.sh_f[b], 0));
                    ga.tbuf = c.tbuf.as<uint32_t>() + (uint64_t)b * crow * draws;
                    ga.tflags = c.tflags.as<unsigned char>() + (uint64_t)b * crow;
                    ga.tbuf_row0 = r0;
                    gather(r0, r1, 0, (uint32_t)n);
                    SamplerArgs sa = make_sa();
                    sa.row_begin = r0;
                    sa.row_end = r1;
                    sa.tbuf = ga.tbuf;
                    sa.tflags = ga.tflags;
                    sa.tbuf_row0 = r0;
                    sa.rows_per_block = (uint32_t)env_u64("SNGB_SAMPLER_RPB", 16);
                    if (!serial) {
                        CK(cudaEventRecord(c.sh_g[b], gs));
                        CK(cudaStreamWaitEvent(fs, c.sh_g[b], 0));
                    }
                    if (k == 0 && !serial) {
                        tm.mark_on(E_SIDE0, fs);
                        tm.side = true;
                    }
                    CK(launch_sampler(sa, fs, c.num_sms));
                    if (!serial) CK(cudaEventRecord(c.sh_f[b], fs));
                }
                ga.tbuf = nullptr;
                ga.tflags = nullptr;
                if (!serial) {
                    tm.mark_on(E_SIDE1, fs);
                    CK(cudaEventRecord(c.join, fs));
                    CK(cudaStreamWaitEvent(s, c.join, 0));  // extras need every Floyd pass
                }
            } else {
                for (uint32_t ph = 0; ph < gphases; ++ph) gather(rb, re, part(ph), part(ph + 1));
            }
        }
        if (exhaustive && rb > 0 && !upper_only) {  // a row range: its rows' pairs with every v < rb too
            ga.exh_low = (uint32_t)rb;
            for (uint32_t ph = 0; ph < gphases; ++ph) gather(rb, re, part(ph), part(ph + 1));
            ga.exh_low = 0;
        }
        if (prio) {
            CK(cudaEventRecord(c.hi_join, c.hi));
            CK(cudaStreamWaitEvent(s, c.hi_join, 0));
            gs = s;
        }
        tm.mark(E_GATHERED);  // gather kernel(s) done (concurrent with the sampler)
        if (side) CK(cudaStreamWaitEvent(s, c.join, 0));  // extras need the sampler
        if (!exhaustive) {
            ExtrasArgs ea{};
            ea.tp = tp;
            ea.sink = ga.sink;
            ea.counters = dc;
            ea.extras = c.extras.as<unsigned long long>();
            ea.count_ptr = &dc[C_EXTRA_CURSOR];
            ea.capacity = extras_cap;
            if (q8_on) CK(launch_extras_q8(ea, q8p.args, s, c.num_sms));
            else if (metric != kMetricEuclid || d > 1024) CK(launch_extras_metric(ea, s, c.num_sms));
            else CK(launch_extras(ea, s, c.num_sms));
        }
        CK(launch_band(tp, ga.sink, dc, s, c.num_sms));  // the band pairs, decided exactly
        tm.mark(E_EXTRAS);
        CK(cudaMemcpyAsync(c.h_counters, dc, C_COUNT * sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (c.h_counters[C_NONFINITE]) return SNGB_ERR_NONFINITE;
        if (metric == kMetricCosine && n >= 2 && c.h_counters[C_ZERO_ROWS])
            return SNGB_ERR_ZERO_VECTOR;  // distance.hpp:96-97 (any zero row meets a pair)
        if (q8_pipe) {  // the plan came from chunk 0: does it cover every value?
            const double glo = ordered_value(~(uint32_t)c.h_counters[C_QMIN]);
            const double ghi = ordered_value((uint32_t)c.h_counters[C_QMAX]);
            q8_pipe = false;
            if (glo < q8p.lo || ghi > q8p.lo + 255.0 * q8p.s) {
                if (attempt == 3) {
                    g_detail = "8-bit plan retries exhausted";
                    throw CudaFail{cudaErrorUnknown};
                }
                q8_replan = true;  // redo with the global range (the data is resident)
                continue;
            }
        }
        const uint64_t need_e = c.h_counters[C_EDGE_CURSOR];
        const uint64_t need_x = c.h_counters[C_EXTRA_CURSOR];
        const uint64_t need_b = c.h_counters[C_BAND_CURSOR];
        const bool ok = need_e <= edge_cap && (exhaustive || need_x <= extras_cap) &&
                        need_b <= band_cap;
        if (ok) {
            gr.raw = need_e;
            c.edge_hint = std::max<uint64_t>(c.edge_hint, need_e);
            break;
        }
        if (attempt == 3) {
            g_detail = "edge buffer overflow after retries";
            throw CudaFail{cudaErrorMemoryAllocation};
        }
        if (need_b > band_cap) band_cap = need_b + need_b / 8 + 1024;
        c.band_hint = std::max<uint64_t>(c.band_hint, band_cap);
        if (need_e > edge_cap) edge_cap = need_e + need_e / 8 + 1024;
        if (need_x > extras_cap) extras_cap = need_x + need_x / 8 + 1024;
        c.edge_hint = std::max<uint64_t>(c.edge_hint, edge_cap);
    }

    // ---- symmetrise + dedup (graph.cpp:181-188, 34-40) ----
    c.keys_alt.ensure(std::max<uint64_t>(gr.raw, 1) * 8);
    const size_t tb = std::max(sort_unique_temp_bytes(std::max<uint64_t>(gr.raw, 1), nb),
                               cluster_temp_bytes(n));
    c.temp.ensure(tb);
    // the build's keys are canonical (a < b < n): 32-bit sort keys when they fit
    // (SNGB_SORT32=0 keeps the 64-bit sort)
    CK(sort_unique(c.keys.as<unsigned long long>(), c.keys_alt.as<unsigned long long>(), gr.raw,
                   nb, c.temp.p, c.temp.bytes, dc, &gr.ukeys, s,
                   env_u64("SNGB_SORT32", 1) ? n : 0));
    tm.mark(E_SORTED);
    return SNGB_OK;
}

void ensure_cluster_bufs(DevCtx& c, uint64_t n, ClusterBuffers& b) {
    c.deg.ensure(n * 4);
    c.core.ensure(n);
    c.parent.ensure(n * 4);
    c.broot.ensure(n * 4);
    c.first.ensure(n * 4);
    c.flags.ensure((n + 1) * 4);
    c.rank.ensure((n + 1) * 4);
    c.temp.ensure(cluster_temp_bytes(n));
    b.deg = c.deg.as<uint32_t>();
    b.core = c.core.as<uint8_t>();
    b.parent = c.parent.as<uint32_t>();
    b.broot = c.broot.as<uint32_t>();
    b.first = c.first.as<uint32_t>();
    b.flags = c.flags.as<uint32_t>();
    b.rank = c.rank.as<uint32_t>();
    b.temp = c.temp.p;
    b.temp_bytes = c.temp.bytes;
    c.rstart.ensure(n * 4);
    b.rstart = c.rstart.as<uint32_t>();
}

void fill_info(sngb_info* info, const unsigned long long* hc, uint64_t n, uint32_t d,
               const GraphResult& gr, uint64_t rows, Timer& tm, bool clustered, bool host) {
    if (!info) return;
    std::memset(info, 0, sizeof(*info));
    info->kernel_launches = sngb_t_launch_hand;
    info->library_launches = sngb_t_launch_lib;
    info->draws = gr.draws;
    info->distance_evals = gr.exhaustive ? rows * (n - 1) : rows * gr.draws;  // graph.cpp:153,179
    info->edges = hc[C_UNIQUE];
    info->graph_bytes = (n + 1) * 8 + 2 * info->edges * 4;  // graph.hpp:41-43
    info->collisions = hc[C_COLLISIONS];
    info->irregular_vertices = hc[C_IRREGULAR];
    info->pairs_evaluated = hc[C_PAIRS];
    info->band_rechecks = hc[C_BAND];
    info->band_1e6 = hc[C_BAND6];
    info->fp32_flips = hc[C_FLIPS];
    info->directed_accepts = hc[C_EDGE_CURSOR];
    info->gather_pairs = hc[C_GATHER_PAIRS];
    info->filter_bits = gr.q8 ? 8 : (gr.head ? 16 : 32);
    info->head_bytes = gr.head;
    if (gr.head)  // every pair reads its head, survivors their fp32 row
        info->gather_bytes = hc[C_GATHER_PAIRS] * gr.head + hc[C_TAIL_PAIRS] * 4ull * d;
    else if (gr.q8 && q8_split((d + 15) / 16))  // every pair reads its head, survivors the rest
        info->gather_bytes = hc[C_GATHER_PAIRS] * (kHeadVals + 4ull) +
                             hc[C_TAIL_PAIRS] * ((uint64_t)d - kHeadVals + 4);
    else
        info->gather_bytes = hc[C_GATHER_PAIRS] * (gr.q8 ? (uint64_t)d + 4 : 4ull * d);
    if (clustered) {
        info->cluster_count = (int32_t)hc[C_CLUSTERS];
        info->core_count = (uint32_t)hc[C_CORE];
        info->border_count = (uint32_t)hc[C_BORDER];
        info->noise_count = (uint32_t)hc[C_NOISE];
    }
    if (tm.on) {
        info->ms_upload = host ? tm.between(E_START, E_UPLOADED) : 0.f;
        info->ms_sample = tm.side ? tm.between(E_SIDE0, E_SIDE1) : tm.between(E_PREPARED, E_SAMPLED);
        info->ms_gather = tm.between(E_SAMPLED, E_GATHERED);
        info->ms_extras = tm.between(E_GATHERED, E_EXTRAS);
        info->ms_sort = tm.between(E_EXTRAS, E_SORTED);
        info->ms_cluster = clustered ? tm.between(E_SORTED, E_CLUSTERED) : 0.f;
        info->ms_download = host ? tm.between(E_CLUSTERED, E_DOWNLOADED) : 0.f;
        info->ms_total = tm.between(E_START, E_END);
    }
}

template <typename F>
int guarded(F&& f) {
    sngb_t_launch_hand = 0;
    sngb_t_launch_lib = 0;
    try {
        return f();
    } catch (const CudaFail&) {
        cudaGetLastError();
        return SNGB_ERR_CUDA;
    } catch (const std::bad_alloc&) {
        g_detail = "host allocation failed";
        return SNGB_ERR_CUDA;
    }
}

// Full pipeline on device buffers; labels/roles device pointers.
int dbscan_device(DevCtx& c, cudaStream_t s, Timer& tm, const float* d_pts, uint64_t n, uint32_t d,
                  double eps, int32_t min_pts, double rate, uint64_t seed, int32_t* d_labels,
                  uint8_t* d_roles, GraphResult& gr, const float* h_src = nullptr,
                  const double* d_pts64 = nullptr, int32_t metric = kMetricEuclid) {
    int rc = build_graph(c, s, tm, d_pts, n, d, eps, rate, seed, 0, n, gr, h_src, d_pts64, metric);
    if (rc) return rc;
    ClusterBuffers b{};
    ensure_cluster_bufs(c, n, b);
    unsigned long long* dc = c.counters.as<unsigned long long>();
    CK(cluster_unique_edges(gr.ukeys, &dc[C_UNIQUE], gr.raw, n, gr.nb, min_pts, b, dc, d_labels,
                            d_roles, s, c.num_sms));
    tm.mark(E_CLUSTERED);
    return SNGB_OK;
}

// ---- multi-GPU merge steps -----------------------------------
// Shared frame: device + context lock + zeroed counters; `f` enqueues on `s`;
// the counters come back synchronously and bad caller keys fail the call.
template <class F>
int merge_step(const sngb_opts* opts, uint64_t n, F&& f) {
    if (n == 0) return SNGB_ERR_EMPTY;
    if (n > 0x7fffffffull) return SNGB_ERR_TOO_LARGE;  // int32 vertex arrays
    if (!metric_flags_ok(opts)) return SNGB_ERR_ARG;
    if (device_count() == 0) return SNGB_ERR_NO_DEVICE;
    return guarded([&]() -> int {
        const int dev = resolve_device(opts);
        DeviceGuard dg(dev);
        DevCtx& c = get_ctx(dev);
        std::lock_guard<std::mutex> lk(c.mu);
        cudaStream_t s = (opts && opts->stream) ? (cudaStream_t)opts->stream : c.stream;
        sngb_t_launch_hand = 0;
        sngb_t_launch_lib = 0;
        c.counters.ensure(C_COUNT * 8);
        unsigned long long* dc = c.counters.as<unsigned long long>();
        CK(cudaMemsetAsync(dc, 0, C_COUNT * 8, s));
        CK(f(c, s, dc));
        CK(cudaMemcpyAsync(c.h_counters, dc, C_COUNT * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (c.h_counters[C_BADKEY]) return SNGB_ERR_ARG;
        return SNGB_OK;
    });
}

const unsigned long long* ull(const uint64_t* p) {
    return reinterpret_cast<const unsigned long long*>(p);
}

}  // namespace host
}  // namespace sngb

using namespace sngb::host;

extern "C" {

int sngb_abi_version(void) { return SNGB_ABI_VERSION; }

int sngb_device_count(void) { return device_count(); }

const char* sngb_last_error_detail(void) { return detail().c_str(); }

const char* sngb_strerror(int code) {
    switch (code) {
        case SNGB_OK: return "ok";
        case SNGB_ERR_EPS: return "eps must be > 0";
        case SNGB_ERR_MINPTS: return "min_pts must be >= 1";
        case SNGB_ERR_RATE: return "rate must lie in (0, 1]";
        case SNGB_ERR_EMPTY: return "dataset is empty";
        case SNGB_ERR_DIM: return "dataset dimension must be >= 1";
        case SNGB_ERR_NONFINITE: return "dataset contains a non-finite value";
        case SNGB_ERR_TOO_LARGE: return "dataset has too many points for u32 vertex ids";
        case SNGB_ERR_ARG: return "invalid argument (null pointer, bad row range or key)";
        case SNGB_ERR_NO_DEVICE: return "no CUDA device available (the GPU path has no CPU fallback)";
        case SNGB_ERR_CUDA: return "CUDA error";
        case SNGB_ERR_CAPACITY: return "output buffer too small";
        case SNGB_ERR_ZERO_VECTOR: return "cosine distance is undefined for zero vectors";
        default: return "unknown error";
    }
}

void sngb_release_pools(void) {
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    for (auto& c : g_ctx)
        if (c) {
            std::lock_guard<std::mutex> l2(c->mu);
            int prev = 0;
            cudaGetDevice(&prev);
            cudaSetDevice(c->dev);
            c->release();
            cudaSetDevice(prev);
        }
}

int sngb_dbscan_f32_device(const float* d_pts, uint64_t n, uint32_t d, double eps, int32_t min_pts,
                           double rate, uint64_t seed, const sngb_opts* opts, int32_t* d_labels,
                           uint8_t* d_roles, sngb_info* info) {
    int rc = validate(n, d, eps, min_pts, rate, true);
    if (rc) return rc;
    if (!d_pts || !d_labels || !d_roles) return SNGB_ERR_ARG;
    if (!metric_flags_ok(opts)) return SNGB_ERR_ARG;
    if (device_count() == 0) return SNGB_ERR_NO_DEVICE;
    std::vector<int> devs;
    const int w = multi_devices(opts, devs);
    if (w < 0) return SNGB_ERR_ARG;
    if (w > 1)
        return guarded([&]() -> int {
            if (opts->stream) {  // the caller's prior work on the points is complete
                DeviceGuard dg(devs[0]);
                CK(cudaStreamSynchronize((cudaStream_t)opts->stream));
            }
            return multi_dbscan(devs, 2, d_pts, n, d, eps, min_pts, rate, seed, metric_of(opts),
                                false, (opts->flags & SNGB_FLAG_TIMING) != 0, d_labels, d_roles,
                                info);
        });
    return guarded([&]() -> int {
        const int dev = resolve_device(opts);
        DeviceGuard dg(dev);
        DevCtx& c = get_ctx(dev);
        std::lock_guard<std::mutex> lk(c.mu);
        cudaStream_t s = (opts && opts->stream) ? (cudaStream_t)opts->stream : c.stream;
        Timer tm{c, s, opts && (opts->flags & SNGB_FLAG_TIMING)};
        tm.mark(E_START);
        tm.mark(E_UPLOADED);
        GraphResult gr;
        int r = dbscan_device(c, s, tm, d_pts, n, d, eps, min_pts, rate, seed, d_labels, d_roles, gr,
                              nullptr, nullptr, metric_of(opts));
        if (r) return r;
        tm.mark(E_DOWNLOADED);
        tm.mark(E_END);
        CK(cudaMemcpyAsync(c.h_counters, c.counters.p, C_COUNT * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        fill_info(info, c.h_counters, n, d, gr, n, tm, true, false);
        return SNGB_OK;
    });
}

static int dbscan_f32_host(int slot, const float* pts, uint64_t n, uint32_t d, double eps,
                           int32_t min_pts, double rate, uint64_t seed, const sngb_opts* opts,
                           int32_t* labels_out, uint8_t* roles_out, sngb_info* info) {
    int rc = validate(n, d, eps, min_pts, rate, true);
    if (rc) return rc;
    if (!pts || !labels_out || !roles_out) return SNGB_ERR_ARG;
    if (!metric_flags_ok(opts)) return SNGB_ERR_ARG;
    if (device_count() == 0) return SNGB_ERR_NO_DEVICE;
    return guarded([&]() -> int {
        const int dev = resolve_device(opts);
        DeviceGuard dg(dev);
        DevCtx& c = get_ctx(dev, slot);
        std::lock_guard<std::mutex> lk(c.mu);
        cudaStream_t s = (opts && opts->stream) ? (cudaStream_t)opts->stream : c.stream;
        Timer tm{c, s, opts && (opts->flags & SNGB_FLAG_TIMING)};
        tm.mark(E_START);
        c.upload.ensure(n * d * sizeof(float));
        c.labels.ensure(n * 4);
        c.roles.ensure(n);
        GraphResult gr;
        // the upload is chunked and overlapped inside build_graph
        int r = dbscan_device(c, s, tm, c.upload.as<float>(), n, d, eps, min_pts, rate, seed,
                              c.labels.as<int32_t>(), c.roles.as<uint8_t>(), gr, pts, nullptr,
                              metric_of(opts));
        if (r) return r;
        CK(cudaMemcpyAsync(labels_out, c.labels.p, n * 4, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(roles_out, c.roles.p, n, cudaMemcpyDeviceToHost, s));
        tm.mark(E_DOWNLOADED);
        tm.mark(E_END);
        CK(cudaMemcpyAsync(c.h_counters, c.counters.p, C_COUNT * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        fill_info(info, c.h_counters, n, d, gr, n, tm, true, true);
        return SNGB_OK;
    });
}

int sngb_dbscan_f32(const float* pts, uint64_t n, uint32_t d, double eps, int32_t min_pts,
                    double rate, uint64_t seed, const sngb_opts* opts, int32_t* labels_out,
                    uint8_t* roles_out, sngb_info* info) {
    std::vector<int> devs;
    if (opts && opts->num_gpus != 0 && opts->num_gpus != 1) {
        int rc = validate(n, d, eps, min_pts, rate, true);
        if (rc) return rc;
        if (!pts || !labels_out || !roles_out) return SNGB_ERR_ARG;
        if (!metric_flags_ok(opts)) return SNGB_ERR_ARG;
        if (device_count() == 0) return SNGB_ERR_NO_DEVICE;
    }
    const int w = multi_devices(opts, devs);
    if (w < 0) return SNGB_ERR_ARG;
    if (w > 1) {
        return guarded([&]() -> int {
            return multi_dbscan(devs, 0, pts, n, d, eps, min_pts, rate, seed, metric_of(opts),
                                false, (opts->flags & SNGB_FLAG_TIMING) != 0, labels_out,
                                roles_out, info);
        });
    }
    return dbscan_f32_host(0, pts, n, d, eps, min_pts, rate, seed, opts, labels_out, roles_out,
                           info);
}

// Many small problems (the theory lab's pattern, theory.cpp:239-256): up to
// SNGB_BATCH_SLOTS (default 8) host workers, each with its own device context
// and streams, run the problems concurrently so their launch latencies and
// host syncs overlap on the GPU.  Results as if each were a separate call.
int sngb_dbscan_batch_f32(sngb_problem* probs, uint64_t count, const sngb_opts* opts) {
    if (count && !probs) return SNGB_ERR_ARG;
    if (count == 0) return SNGB_OK;
    const uint64_t want = env_u64("SNGB_BATCH_SLOTS", 8);
    const int slots = (int)std::max<uint64_t>(1, std::min<uint64_t>({count, want, (uint64_t)kMaxSlots}));
    std::atomic<uint64_t> next{0};
    auto worker = [&](int slot) {
        for (;;) {
            const uint64_t i = next.fetch_add(1);
            if (i >= count) break;
            sngb_problem& p = probs[i];
            sngb_opts o = opts ? *opts : sngb_opts{-1, 0u, nullptr, 0, 0};
            o.stream = nullptr;  // each worker runs on its own context's stream
            o.flags = (o.flags & SNGB_FLAG_TIMING) | p.flags;
            p.status = dbscan_f32_host(slot, p.pts, p.n, p.d, p.eps, p.min_pts, p.rate, p.seed, &o,
                                       p.labels_out, p.roles_out, p.info_out);
        }
    };
    std::vector<std::thread> pool;
    for (int sl = 1; sl < slots; ++sl) pool.emplace_back(worker, sl);
    worker(0);
    for (auto& t : pool) t.join();
    for (uint64_t i = 0; i < count; ++i)
        if (probs[i].status != SNGB_OK) return probs[i].status;
    return SNGB_OK;
}

int sngb_sampled_edges_f32_device(const float* d_pts, uint64_t n, uint32_t d, double eps,
                                  double rate, uint64_t seed, const sngb_opts* opts,
                                  uint64_t* d_keys_out, uint64_t capacity, uint64_t* count_out,
                                  sngb_info* info) {
    int rc = validate(n, d, eps, 1, rate, false);
    if (rc) return rc;
    if (!d_pts || !count_out) return SNGB_ERR_ARG;
    const uint64_t rb = opts ? opts->row_begin : 0;
    const uint64_t re = (opts && opts->row_end) ? opts->row_end : n;
    if (rb > re || re > n) return SNGB_ERR_ARG;
    if (!metric_flags_ok(opts)) return SNGB_ERR_ARG;
    if (device_count() == 0) return SNGB_ERR_NO_DEVICE;
    return guarded([&]() -> int {
        const int dev = resolve_device(opts);
        DeviceGuard dg(dev);
        DevCtx& c = get_ctx(dev);
        std::lock_guard<std::mutex> lk(c.mu);
        cudaStream_t s = (opts && opts->stream) ? (cudaStream_t)opts->stream : c.stream;
        Timer tm{c, s, opts && (opts->flags & SNGB_FLAG_TIMING)};
        tm.mark(E_START);
        tm.mark(E_UPLOADED);
        GraphResult gr;
        int r = build_graph(c, s, tm, d_pts, n, d, eps, rate, seed, rb, re, gr, nullptr, nullptr,
                            metric_of(opts));
        if (r) return r;
        tm.mark(E_CLUSTERED);
        tm.mark(E_DOWNLOADED);
        tm.mark(E_END);
        unsigned long long* dc = c.counters.as<unsigned long long>();
        CK(cudaMemcpyAsync(c.h_counters, dc, C_COUNT * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        const uint64_t m = c.h_counters[C_UNIQUE];
        *count_out = m;
        fill_info(info, c.h_counters, n, d, gr, re - rb, tm, false, false);
        if (m > capacity) return SNGB_ERR_CAPACITY;
        if (m && !d_keys_out) return SNGB_ERR_ARG;
        CK(launch_convert_keys(gr.ukeys, reinterpret_cast<unsigned long long*>(d_keys_out), m,
                               gr.nb, false, n, dc, s, c.num_sms));
        CK(cudaStreamSynchronize(s));
        return SNGB_OK;
    });
}

int sngb_sampled_edges_f32(const float* pts, uint64_t n, uint32_t d, double eps, double rate,
                           uint64_t seed, const sngb_opts* opts, uint64_t* keys_out,
                           uint64_t capacity, uint64_t* count_out, sngb_info* info) {
    int rc = validate(n, d, eps, 1, rate, false);
    if (rc) return rc;
    if (!pts || !count_out) return SNGB_ERR_ARG;
    const uint64_t rb = opts ? opts->row_begin : 0;
    const uint64_t re = (opts && opts->row_end) ? opts->row_end : n;
    if (rb > re || re > n) return SNGB_ERR_ARG;
    if (!metric_flags_ok(opts)) return SNGB_ERR_ARG;
    if (device_count() == 0) return SNGB_ERR_NO_DEVICE;
    return guarded([&]() -> int {
        const int dev = resolve_device(opts);
        DeviceGuard dg(dev);
        DevCtx& c = get_ctx(dev);
        std::lock_guard<std::mutex> lk(c.mu);
        cudaStream_t s = (opts && opts->stream) ? (cudaStream_t)opts->stream : c.stream;
        Timer tm{c, s, opts && (opts->flags & SNGB_FLAG_TIMING)};
        tm.mark(E_START);
        c.upload.ensure(n * d * sizeof(float));
        GraphResult gr;
        int r = build_graph(c, s, tm, c.upload.as<float>(), n, d, eps, rate, seed, rb, re, gr,
                            pts, nullptr, metric_of(opts));
        if (r) return r;
        tm.mark(E_CLUSTERED);
        unsigned long long* dc = c.counters.as<unsigned long long>();
        CK(cudaMemcpyAsync(c.h_counters, dc, C_COUNT * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        const uint64_t m = c.h_counters[C_UNIQUE];
        *count_out = m;
        if (m > capacity) {
            fill_info(info, c.h_counters, n, d, gr, re - rb, tm, false, true);
            return SNGB_ERR_CAPACITY;
        }
        if (m && !keys_out) return SNGB_ERR_ARG;
        unsigned long long* conv = (gr.ukeys == c.keys.as<unsigned long long>())
                                       ? c.keys_alt.as<unsigned long long>()
                                       : c.keys.as<unsigned long long>();
        CK(launch_convert_keys(gr.ukeys, conv, m, gr.nb, false, n, dc, s, c.num_sms));
        if (m) CK(cudaMemcpyAsync(keys_out, conv, m * 8, cudaMemcpyDeviceToHost, s));
        tm.mark(E_DOWNLOADED);
        tm.mark(E_END);
        CK(cudaStreamSynchronize(s));
        fill_info(info, c.h_counters, n, d, gr, re - rb, tm, false, true);
        return SNGB_OK;
    });
}

int sngb_cluster_edges_device(const uint64_t* d_keys, uint64_t nkeys, uint64_t n, int32_t min_pts,
                              const sngb_opts* opts, int32_t* d_labels, uint8_t* d_roles,
                              sngb_info* info) {
    if (min_pts < 1) return SNGB_ERR_MINPTS;
    if (n == 0) return SNGB_ERR_EMPTY;
    if (n >= 0xffffff00ull) return SNGB_ERR_TOO_LARGE;
    if ((nkeys && !d_keys) || !d_labels || !d_roles) return SNGB_ERR_ARG;
    if (!metric_flags_ok(opts)) return SNGB_ERR_ARG;
    if (device_count() == 0) return SNGB_ERR_NO_DEVICE;
    return guarded([&]() -> int {
        const int dev = resolve_device(opts);
        DeviceGuard dg(dev);
        DevCtx& c = get_ctx(dev);
        std::lock_guard<std::mutex> lk(c.mu);
        cudaStream_t s = (opts && opts->stream) ? (cudaStream_t)opts->stream : c.stream;
        Timer tm{c, s, opts && (opts->flags & SNGB_FLAG_TIMING)};
        tm.mark(E_START);
        tm.mark(E_UPLOADED);
        tm.mark(E_PREPARED);
        tm.mark(E_SAMPLED);
        tm.mark(E_GATHERED);
        tm.mark(E_EXTRAS);
        c.counters.ensure(C_COUNT * 8);
        unsigned long long* dc = c.counters.as<unsigned long long>();
        CK(cudaMemsetAsync(dc, 0, C_COUNT * 8, s));
        const uint32_t nb = bits_for(n - 1);
        c.keys.ensure(std::max<uint64_t>(nkeys, 1) * 8);
        c.keys_alt.ensure(std::max<uint64_t>(nkeys, 1) * 8);
        CK(launch_convert_keys(reinterpret_cast<const unsigned long long*>(d_keys),
                               c.keys.as<unsigned long long>(), nkeys, nb, true, n, dc, s,
                               c.num_sms));
        c.temp.ensure(std::max(sort_unique_temp_bytes(std::max<uint64_t>(nkeys, 1), nb),
                               cluster_temp_bytes(n)));
        GraphResult gr;
        gr.nb = nb;
        gr.raw = nkeys;
        CK(sort_unique(c.keys.as<unsigned long long>(), c.keys_alt.as<unsigned long long>(), nkeys,
                       nb, c.temp.p, c.temp.bytes, dc, &gr.ukeys, s));
        tm.mark(E_SORTED);
        ClusterBuffers b{};
        ensure_cluster_bufs(c, n, b);
        CK(cluster_unique_edges(gr.ukeys, &dc[C_UNIQUE], nkeys, n, nb, min_pts, b, dc, d_labels,
                                d_roles, s, c.num_sms));
        tm.mark(E_CLUSTERED);
        tm.mark(E_DOWNLOADED);
        tm.mark(E_END);
        CK(cudaMemcpyAsync(c.h_counters, dc, C_COUNT * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (c.h_counters[C_BADKEY]) return SNGB_ERR_ARG;
        fill_info(info, c.h_counters, n, 0, gr, 0, tm, true, false);
        return SNGB_OK;
    });
}

// ---- fp64 input (the reference's Dataset is fp64, dataset.hpp:69-71) -------
int sngb_dbscan_f64_device(const double* d_pts, uint64_t n, uint32_t d, double eps,
                           int32_t min_pts, double rate, uint64_t seed, const sngb_opts* opts,
                           int32_t* d_labels, uint8_t* d_roles, sngb_info* info) {
    int rc = validate(n, d, eps, min_pts, rate, true);
    if (rc) return rc;
    if (!d_pts || !d_labels || !d_roles) return SNGB_ERR_ARG;
    if (!metric_flags_ok(opts)) return SNGB_ERR_ARG;
    if (device_count() == 0) return SNGB_ERR_NO_DEVICE;
    return guarded([&]() -> int {
        const int dev = resolve_device(opts);
        DeviceGuard dg(dev);
        DevCtx& c = get_ctx(dev);
        std::lock_guard<std::mutex> lk(c.mu);
        cudaStream_t s = (opts && opts->stream) ? (cudaStream_t)opts->stream : c.stream;
        Timer tm{c, s, opts && (opts->flags & SNGB_FLAG_TIMING)};
        tm.mark(E_START);
        tm.mark(E_UPLOADED);
        GraphResult gr;
        int r = dbscan_device(c, s, tm, nullptr, n, d, eps, min_pts, rate, seed, d_labels, d_roles,
                              gr, nullptr, d_pts, metric_of(opts));
        if (r) return r;
        tm.mark(E_DOWNLOADED);
        tm.mark(E_END);
        CK(cudaMemcpyAsync(c.h_counters, c.counters.p, C_COUNT * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        fill_info(info, c.h_counters, n, d, gr, n, tm, true, false);
        return SNGB_OK;
    });
}

int sngb_dbscan_f64(const double* pts, uint64_t n, uint32_t d, double eps, int32_t min_pts,
                    double rate, uint64_t seed, const sngb_opts* opts, int32_t* labels_out,
                    uint8_t* roles_out, sngb_info* info) {
    int rc = validate(n, d, eps, min_pts, rate, true);
    if (rc) return rc;
    if (!pts || !labels_out || !roles_out) return SNGB_ERR_ARG;
    if (!metric_flags_ok(opts)) return SNGB_ERR_ARG;
    if (device_count() == 0) return SNGB_ERR_NO_DEVICE;
    std::vector<int> devs;
    const int w = multi_devices(opts, devs);
    if (w < 0) return SNGB_ERR_ARG;
    if (w > 1)
        return guarded([&]() -> int {
            return multi_dbscan(devs, 1, pts, n, d, eps, min_pts, rate, seed, metric_of(opts),
                                false, (opts->flags & SNGB_FLAG_TIMING) != 0, labels_out,
                                roles_out, info);
        });
    return guarded([&]() -> int {
        const int dev = resolve_device(opts);
        DeviceGuard dg(dev);
        DevCtx& c = get_ctx(dev);
        std::lock_guard<std::mutex> lk(c.mu);
        cudaStream_t s = (opts && opts->stream) ? (cudaStream_t)opts->stream : c.stream;
        Timer tm{c, s, opts && (opts->flags & SNGB_FLAG_TIMING)};
        tm.mark(E_START);
        c.upload64.ensure(n * d * sizeof(double));
        CK(cudaMemcpyAsync(c.upload64.p, pts, n * d * sizeof(double), cudaMemcpyHostToDevice, s));
        tm.mark(E_UPLOADED);
        c.labels.ensure(n * 4);
        c.roles.ensure(n);
        GraphResult gr;
        int r = dbscan_device(c, s, tm, nullptr, n, d, eps, min_pts, rate, seed,
                              c.labels.as<int32_t>(), c.roles.as<uint8_t>(), gr, nullptr,
                              c.upload64.as<double>(), metric_of(opts));
        if (r) return r;
        CK(cudaMemcpyAsync(labels_out, c.labels.p, n * 4, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(roles_out, c.roles.p, n, cudaMemcpyDeviceToHost, s));
        tm.mark(E_DOWNLOADED);
        tm.mark(E_END);
        CK(cudaMemcpyAsync(c.h_counters, c.counters.p, C_COUNT * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        fill_info(info, c.h_counters, n, d, gr, n, tm, true, true);
        return SNGB_OK;
    });
}

int sngb_sampled_edges_f64(const double* pts, uint64_t n, uint32_t d, double eps, double rate,
                           uint64_t seed, const sngb_opts* opts, uint64_t* keys_out,
                           uint64_t capacity, uint64_t* count_out, sngb_info* info) {
    int rc = validate(n, d, eps, 1, rate, false);
    if (rc) return rc;
    if (!pts || !count_out) return SNGB_ERR_ARG;
    const uint64_t rb = opts ? opts->row_begin : 0;
    const uint64_t re = (opts && opts->row_end) ? opts->row_end : n;
    if (rb > re || re > n) return SNGB_ERR_ARG;
    if (!metric_flags_ok(opts)) return SNGB_ERR_ARG;
    if (device_count() == 0) return SNGB_ERR_NO_DEVICE;
    return guarded([&]() -> int {
        const int dev = resolve_device(opts);
        DeviceGuard dg(dev);
        DevCtx& c = get_ctx(dev);
        std::lock_guard<std::mutex> lk(c.mu);
        cudaStream_t s = (opts && opts->stream) ? (cudaStream_t)opts->stream : c.stream;
        Timer tm{c, s, opts && (opts->flags & SNGB_FLAG_TIMING)};
        tm.mark(E_START);
        c.upload64.ensure(n * d * sizeof(double));
        CK(cudaMemcpyAsync(c.upload64.p, pts, n * d * sizeof(double), cudaMemcpyHostToDevice, s));
        tm.mark(E_UPLOADED);
        GraphResult gr;
        int r = build_graph(c, s, tm, nullptr, n, d, eps, rate, seed, rb, re, gr, nullptr,
                            c.upload64.as<double>(), metric_of(opts));
        if (r) return r;
        tm.mark(E_CLUSTERED);
        unsigned long long* dc = c.counters.as<unsigned long long>();
        CK(cudaMemcpyAsync(c.h_counters, dc, C_COUNT * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        const uint64_t m = c.h_counters[C_UNIQUE];
        *count_out = m;
        if (m > capacity) {
            fill_info(info, c.h_counters, n, d, gr, re - rb, tm, false, true);
            return SNGB_ERR_CAPACITY;
        }
        if (m && !keys_out) return SNGB_ERR_ARG;
        unsigned long long* conv = (gr.ukeys == c.keys.as<unsigned long long>())
                                       ? c.keys_alt.as<unsigned long long>()
                                       : c.keys.as<unsigned long long>();
        CK(launch_convert_keys(gr.ukeys, conv, m, gr.nb, false, n, dc, s, c.num_sms));
        if (m) CK(cudaMemcpyAsync(keys_out, conv, m * 8, cudaMemcpyDeviceToHost, s));
        tm.mark(E_DOWNLOADED);
        tm.mark(E_END);
        CK(cudaStreamSynchronize(s));
        fill_info(info, c.h_counters, n, d, gr, re - rb, tm, false, true);
        return SNGB_OK;
    });
}

int sngb_unique_keys_device(const uint64_t* d_keys, uint64_t nkeys, uint64_t n,
                            const sngb_opts* opts, uint64_t* d_out, uint64_t* count_out) {
    if ((nkeys && (!d_keys || !d_out)) || !count_out) return SNGB_ERR_ARG;
    if (nkeys && d_keys == d_out) return SNGB_ERR_ARG;
    uint64_t count = 0;
    const int rc = merge_step(opts, n, [&](DevCtx& c, cudaStream_t s, unsigned long long* dc) {
        if (nkeys == 0) return cudaSuccess;
        const uint32_t nb = bits_for(n - 1);
        c.keys.ensure(nkeys * 8);
        c.keys_alt.ensure(nkeys * 8);
        cudaError_t e = launch_convert_keys(ull(d_keys), c.keys.as<unsigned long long>(), nkeys, nb,
                                            true, n, dc, s, c.num_sms);
        if (e != cudaSuccess) return e;
        c.temp.ensure(sort_unique_temp_bytes(nkeys, nb));
        unsigned long long* u = nullptr;
        e = sort_unique(c.keys.as<unsigned long long>(), c.keys_alt.as<unsigned long long>(), nkeys,
                        nb, c.temp.p, c.temp.bytes, dc, &u, s);
        if (e != cudaSuccess) return e;
        // back to a<<32|b; unique <= nkeys, the tail beyond the count is scratch
        e = launch_convert_keys(u, reinterpret_cast<unsigned long long*>(d_out), nkeys, nb, false,
                                n, dc, s, c.num_sms);
        if (e != cudaSuccess) return e;
        e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) return e;
        return cudaMemcpy(&count, &dc[C_UNIQUE], 8, cudaMemcpyDeviceToHost);
    });
    if (rc == SNGB_OK) *count_out = count;
    return rc;
}

int sngb_degrees_device(const uint64_t* d_keys, uint64_t nkeys, uint64_t n, const sngb_opts* opts,
                        int32_t* d_degree) {
    if ((nkeys && !d_keys) || !d_degree) return SNGB_ERR_ARG;
    return merge_step(opts, n, [&](DevCtx& c, cudaStream_t s, unsigned long long* dc) {
        cudaError_t e = merge_check_keys(ull(d_keys), nkeys, n, dc, s, c.num_sms);
        if (e != cudaSuccess) return e;
        // a bad key is counted before any write: skip the pass and fail below
        e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) return e;
        unsigned long long bad = 0;
        e = cudaMemcpy(&bad, &dc[C_BADKEY], 8, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess || bad) return e;
        return merge_degrees(ull(d_keys), nkeys, reinterpret_cast<uint32_t*>(d_degree), s,
                             c.num_sms);
    });
}

int sngb_components_device(const uint64_t* d_keys, uint64_t nkeys, uint64_t n,
                           const int32_t* d_degree, int32_t min_pts, const sngb_opts* opts,
                           int32_t* d_parent, uint64_t* changed_out) {
    if (min_pts < 1) return SNGB_ERR_MINPTS;
    if ((nkeys && !d_keys) || !d_degree || !d_parent) return SNGB_ERR_ARG;
    uint64_t changed = 0;
    const int rc = merge_step(opts, n, [&](DevCtx& c, cudaStream_t s, unsigned long long* dc) {
        cudaError_t e = merge_check_keys(ull(d_keys), nkeys, n, dc, s, c.num_sms);
        if (e != cudaSuccess) return e;
        e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) return e;
        unsigned long long bad = 0;
        e = cudaMemcpy(&bad, &dc[C_BADKEY], 8, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess || bad) return e;
        c.core.ensure(n);
        c.first.ensure(n * 4);  // snapshot of the incoming forest
        e = merge_components(ull(d_keys), nkeys, n, reinterpret_cast<const uint32_t*>(d_degree),
                             min_pts, reinterpret_cast<uint32_t*>(d_parent), c.core.as<uint8_t>(),
                             c.first.as<uint32_t>(), dc, s, c.num_sms);
        if (e != cudaSuccess) return e;
        e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) return e;
        return cudaMemcpy(&changed, &dc[C_CHANGED], 8, cudaMemcpyDeviceToHost);
    });
    if (rc == SNGB_OK && changed_out) *changed_out = changed;
    return rc;
}

int sngb_border_device(const uint64_t* d_keys, uint64_t nkeys, uint64_t n, const int32_t* d_degree,
                       int32_t min_pts, const int32_t* d_parent, const sngb_opts* opts,
                       int32_t* d_border) {
    if (min_pts < 1) return SNGB_ERR_MINPTS;
    if ((nkeys && !d_keys) || !d_degree || !d_parent || !d_border) return SNGB_ERR_ARG;
    return merge_step(opts, n, [&](DevCtx& c, cudaStream_t s, unsigned long long* dc) {
        cudaError_t e = merge_check_keys(ull(d_keys), nkeys, n, dc, s, c.num_sms);
        if (e != cudaSuccess) return e;
        e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) return e;
        unsigned long long bad = 0;
        e = cudaMemcpy(&bad, &dc[C_BADKEY], 8, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess || bad) return e;
        c.core.ensure(n);
        return merge_border(ull(d_keys), nkeys, n, reinterpret_cast<const uint32_t*>(d_degree),
                            min_pts, reinterpret_cast<const uint32_t*>(d_parent),
                            reinterpret_cast<uint32_t*>(d_border), c.core.as<uint8_t>(), s,
                            c.num_sms);
    });
}

int sngb_relabel_device(uint64_t n, const int32_t* d_degree, int32_t min_pts,
                        const int32_t* d_parent, const int32_t* d_border, const sngb_opts* opts,
                        int32_t* d_labels, uint8_t* d_roles, sngb_info* info) {
    if (min_pts < 1) return SNGB_ERR_MINPTS;
    if (!d_degree || !d_parent || !d_border || !d_labels || !d_roles) return SNGB_ERR_ARG;
    unsigned long long hc[C_COUNT] = {};
    const int rc = merge_step(opts, n, [&](DevCtx& c, cudaStream_t s, unsigned long long* dc) {
        ClusterBuffers b{};
        ensure_cluster_bufs(c, n, b);
        cudaError_t e = merge_relabel(n, reinterpret_cast<const uint32_t*>(d_degree), min_pts,
                                      reinterpret_cast<const uint32_t*>(d_parent),
                                      reinterpret_cast<const uint32_t*>(d_border), b, dc, d_labels,
                                      d_roles, s, c.num_sms);
        if (e != cudaSuccess) return e;
        e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) return e;
        return cudaMemcpy(hc, dc, sizeof(hc), cudaMemcpyDeviceToHost);
    });
    if (rc == SNGB_OK && info) {
        std::memset(info, 0, sizeof(*info));
        info->cluster_count = (int32_t)hc[C_CLUSTERS];
        info->core_count = (uint32_t)hc[C_CORE];
        info->border_count = (uint32_t)hc[C_BORDER];
        info->noise_count = (uint32_t)hc[C_NOISE];
        info->kernel_launches = sngb_t_launch_hand;
        info->library_launches = sngb_t_launch_lib;
    }
    return rc;
}


// ---- sng::dbscan_exact / build_full_graph (clusterer.cpp:67-79, graph.cpp:191-220) ----
// The exact eps-graph is the exhaustive branch of the graph build (every v > u
// tested once: the GPU path already evaluates each unordered pair once);
// dbscan_exact differs from sng_dbscan(rate = 1) only in its validation (no
// rate) and in counting n(n-1)/2 distance evaluations (graph.cpp:206-210).
}  // extern "C"

static int validate_exact(uint64_t n, uint32_t d, double eps, int32_t min_pts) {
    if (!(eps > 0.0)) return SNGB_ERR_EPS;      // clusterer.cpp:69
    if (min_pts < 1) return SNGB_ERR_MINPTS;    // clusterer.cpp:70
    if (n == 0) return SNGB_ERR_EMPTY;          // graph.cpp:18
    if (d == 0) return SNGB_ERR_DIM;            // dataset.hpp:22
    if (n >= 0xffffff00ull) return SNGB_ERR_TOO_LARGE;
    return SNGB_OK;
}

static void exact_info(sngb_info* info, uint64_t n) {
    if (!info) return;
    info->draws = n - 1;
    info->distance_evals = n * (n - 1) / 2;  // build_full_graph: v > u only
}

template <class Single>
static int exact_call(uint64_t n, uint32_t d, double eps, int32_t min_pts, const void* pts,
                      const void* labels, const void* roles, const sngb_opts* opts, int src_kind,
                      int32_t* lab, uint8_t* rol, sngb_info* info, Single&& single) {
    int rc = validate_exact(n, d, eps, min_pts);
    if (rc) return rc;
    if (!pts || !labels || !roles) return SNGB_ERR_ARG;
    if (!metric_flags_ok(opts)) return SNGB_ERR_ARG;
    if (device_count() == 0) return SNGB_ERR_NO_DEVICE;
    std::vector<int> devs;
    const int w = multi_devices(opts, devs);
    if (w < 0) return SNGB_ERR_ARG;
    if (w > 1) {
        rc = guarded([&]() -> int {
            if (src_kind == 2 && opts->stream) {
                DeviceGuard dg(devs[0]);
                CK(cudaStreamSynchronize((cudaStream_t)opts->stream));
            }
            return multi_dbscan(devs, src_kind, pts, n, d, eps, min_pts, 1.0, 0, metric_of(opts),
                                true, (opts->flags & SNGB_FLAG_TIMING) != 0, lab, rol, info);
        });
        return rc;
    }
    rc = single();
    if (rc == SNGB_OK) exact_info(info, n);
    return rc;
}

extern "C" {

int sngb_dbscan_exact_f32(const float* pts, uint64_t n, uint32_t d, double eps, int32_t min_pts,
                          const sngb_opts* opts, int32_t* labels_out, uint8_t* roles_out,
                          sngb_info* info) {
    return exact_call(n, d, eps, min_pts, pts, labels_out, roles_out, opts, 0, labels_out,
                      roles_out, info, [&]() {
                          return dbscan_f32_host(0, pts, n, d, eps, min_pts, 1.0, 0, opts,
                                                 labels_out, roles_out, info);
                      });
}

int sngb_dbscan_exact_f32_device(const float* d_pts, uint64_t n, uint32_t d, double eps,
                                 int32_t min_pts, const sngb_opts* opts, int32_t* d_labels,
                                 uint8_t* d_roles, sngb_info* info) {
    return exact_call(n, d, eps, min_pts, d_pts, d_labels, d_roles, opts, 2, d_labels, d_roles,
                      info, [&]() {
                          sngb_opts o = opts ? *opts : sngb_opts{-1, 0u, nullptr, 0, 0, 0, nullptr};
                          o.num_gpus = 0;
                          return sngb_dbscan_f32_device(d_pts, n, d, eps, min_pts, 1.0, 0, &o,
                                                        d_labels, d_roles, info);
                      });
}

int sngb_dbscan_exact_f64(const double* pts, uint64_t n, uint32_t d, double eps, int32_t min_pts,
                          const sngb_opts* opts, int32_t* labels_out, uint8_t* roles_out,
                          sngb_info* info) {
    return exact_call(n, d, eps, min_pts, pts, labels_out, roles_out, opts, 1, labels_out,
                      roles_out, info, [&]() {
                          sngb_opts o = opts ? *opts : sngb_opts{-1, 0u, nullptr, 0, 0, 0, nullptr};
                          o.num_gpus = 0;
                          return sngb_dbscan_f64(pts, n, d, eps, min_pts, 1.0, 0, &o, labels_out,
                                                 roles_out, info);
                      });
}

int sngb_full_edges_f32(const float* pts, uint64_t n, uint32_t d, double eps, const sngb_opts* opts,
                        uint64_t* keys_out, uint64_t capacity, uint64_t* count_out,
                        sngb_info* info) {
    sngb_opts o = opts ? *opts : sngb_opts{-1, 0u, nullptr, 0, 0, 0, nullptr};
    o.row_begin = 0;
    o.row_end = 0;
    o.num_gpus = 0;
    const int rc = sngb_sampled_edges_f32(pts, n, d, eps, 1.0, 0, &o, keys_out, capacity,
                                          count_out, info);
    if (rc == SNGB_OK || rc == SNGB_ERR_CAPACITY) exact_info(info, n);
    return rc;
}

}  // extern "C"
