// sngb_internal.cuh -- shared device types of libsngb (not part of the ABI).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

namespace sngb {

constexpr unsigned kFull = 0xffffffffu;
constexpr uint32_t kEmpty = 0xffffffffu;

// Slots of the device counter block (u64 each).
enum Counter : int {
    C_EDGE_CURSOR = 0,   // emitted directed-accept keys (may exceed capacity)
    C_EXTRA_CURSOR,      // sampler extras (collision replacements, irregular partners)
    C_PAIRS,             // pairs evaluated on the GPU
    C_BAND,              // fp32 sum inside guard band -> exact fp64 recheck
    C_BAND6,             // |s32 - eps2| <= 1e-6 eps2
    C_FLIPS,             // bare-fp32 decision would differ from the exact one
    C_COLLISIONS,        // Floyd replacements
    C_IRREGULAR,         // vertices with a Lemire reject pre-condition
    C_GATHER_PAIRS,      // pairs evaluated by the gather kernel
    C_NONFINITE,         // non-finite input values seen
    C_UNIQUE,            // unique undirected edges (DeviceSelect output)
    C_CORE,
    C_BORDER,
    C_NOISE,
    C_CLUSTERS,
    C_BADKEY,            // self loop / out-of-range endpoint in caller keys
    C_CHANGED,           // merge step: vertices whose component root moved
    C_ZERO_ROWS,         // cosine: rows whose fp64 norm is 0 (distance.hpp:97)
    C_BAND_CURSOR,       // band pairs appended (see TestParams::band)
    C_QMIN,              // max of ~ordered(value): the dataset minimum (8-bit filter scale)
    C_QMAX,              // max of ordered(value): the dataset maximum
    C_TAIL_PAIRS,        // 8-bit filter: pairs the head did not reject (read their tail)
    C_IRR_CURSOR,        // fused sampler: vertices listed for the exact sequential replay
    C_COUNT
};

// The eps-test: fp32 accumulate with a rigorous guard band, exact fp64
// recheck (distance.hpp:75-83 order) inside the band.
struct TestParams {
    const float* pts;  // device rows, `stride` floats each, zero padded past d
    uint32_t stride;   // 2 (d <= 2) or a multiple of 4
    uint32_t d;        // true dimension
    float lo_thr;      // s32 <  lo_thr  => exact s64 <= eps2 (accept)
    float hi_thr;      // s32 >  hi_thr  => exact s64 >  eps2 (reject)
    float eps2f;       // (float)eps2, for the bare-fp32 comparison statistics
    double eps2;       // eps * eps in fp64, as distance.hpp:82 computes it
    const double* pts64;  // fp64 input: the caller's rows (d per row) for the exact
                          // recheck; pts then holds them rounded to fp32.  null: fp32 input
    int32_t metric;       // kMetricEuclid / kMetricManhattan / kMetricCosine
    double eps;           // the metric's eps (Manhattan, cosine compare against it)
    const float* rnorm;   // cosine: fp32 |row| per row (sqrt of the fp32 sum of squares)
    // pairs whose filter value lands in the band: appended here by the filter
    // kernels, decided exactly (fp64, the reference's order) by k_band afterwards,
    // so the rare exact path costs the hot kernels no registers
    uint4* band;                      // {u, v, filter value bits, 0}
    unsigned long long* band_cursor;  // may exceed band_cap (the host retries)
    unsigned long long band_cap;
};
constexpr int32_t kMetricEuclid = 0, kMetricManhattan = 1, kMetricCosine = 2;

// Canonical undirected edge keys: (min << nb) | max with nb = bits(n-1).
struct EdgeSink {
    unsigned long long* keys;
    unsigned long long capacity;
    unsigned long long* cursor;
    uint32_t nb;
};

struct GatherArgs {
    TestParams tp;
    EdgeSink sink;
    unsigned long long* counters;
    uint64_t n;
    uint64_t row_begin, row_end;
    uint32_t draws;       // per-vertex draws (sampled mode)
    uint32_t base;        // pool - draws, pool = n - 1
    uint64_t seed_mixed;  // mix(seed + gamma)
    uint32_t force_mod;   // test hook (0 = off), see test_fire()
    uint32_t part_lo, part_hi;  // partner rows tested by this launch (L2-blocked phases)
    uint32_t rows_per_block;    // 0: persistent grid; else one block per this many rows
    uint32_t exh_low;           // exhaustive, nonzero: partners are v < exh_low (the rows below a
                                // row range: graph.cpp:157-159 pairs a row with every v != u)
    unsigned long long* work;   // non-null: warps claim `grab` rows at a time from *work (zeroed)
    uint32_t grab;
    // Bucketed partner lists (k_partners; 8-bit head/tail gather only): row u's
    // partners grouped by partner slice, slice b = [n*b/B, n*(b+1)/B), its list at
    // partners[(u - partners_row0) * draws + poff[(u - partners_row0) * (B + 1) + b]];
    // a launch reads slices [blo, bhi) instead of regenerating every draw.
    // Draws from an irregular vertex's first fired draw on are left out.
    const uint32_t* partners;
    const uint32_t* poff;
    uint64_t partners_row0;
    uint32_t nbuckets, blo, bhi;
    // Shared draws (head gather -> k_floyd_pipe; only in builds with -DSNGB_SHARE_DRAWS=1:
    // measured no faster, DESIGN 5b): the gather also writes every draw
    // value t_i of row u to tbuf[(u - tbuf_row0) * draws + i] and whether the row's
    // stream met the Lemire pre-condition to tflags[u - tbuf_row0], so the Floyd
    // bookkeeping reads them instead of regenerating each draw.  null: off
    uint32_t* tbuf;
    unsigned char* tflags;
    uint64_t tbuf_row0;
};

// Test hook (env SNGB_TEST_FORCE_IRREGULAR=m): pretend the Lemire reject
// pre-condition fired at draw draws/2 of every vertex u with u % m == 0, so
// the exact sequential replay of irregular vertices is exercised by the
// parity tests.  The pre-condition is a superset test, so forcing it never
// changes results -- only which path produces them.
__device__ __forceinline__ bool test_fire(uint32_t force_mod, uint64_t u, uint32_t i,
                                          uint32_t draws) {
    return force_mod != 0 && (u % force_mod) == 0 && i == draws / 2;
}

struct SamplerArgs {
    uint64_t n;
    uint64_t row_begin, row_end;
    uint32_t draws, base;
    uint64_t seed_mixed;
    uint32_t force_mod;        // test hook, see test_fire()
    uint32_t rows_per_block;   // 0: persistent grid; else one block per this many rows
    uint32_t hash_mask;        // slots - 1 (slots: power of two >= 1.6 * draws)
    uint32_t hash_shift;       // 32 - log2(slots)
    uint32_t col_words;        // u32 words of a draws-bit bitmap (multiple of 4)
    uint32_t key_bits;         // bits of a draw value t (fast path epoch tags)
    const uint32_t* tbuf;           // shared draws written by the head gather (see GatherArgs)
    const unsigned char* tflags;
    uint64_t tbuf_row0;
    unsigned long long* scratch64;  // global tables when they do not fit shared memory
    unsigned long long* extras;  // (u << 32) | v ordered pairs to evaluate
    unsigned long long extras_capacity;
    unsigned long long* counters;
};

struct ExtrasArgs {
    TestParams tp;
    EdgeSink sink;
    unsigned long long* counters;
    const unsigned long long* extras;
    const unsigned long long* count_ptr;  // device: number of extras written (may exceed capacity)
    unsigned long long capacity;
};

// Host-side launch accounting (thread-local; read back into sngb_info).
void note_launch(int hand_written, int library = 0);

// ---- launchers (sngb_kernels.cu) ----
cudaError_t launch_prepare_points(const float* src, float* dst, uint64_t n, uint32_t d,
                                  uint32_t stride, unsigned long long* counters, bool minmax,
                                  cudaStream_t s);
// fp64 input: round into the padded fp32 table, count non-finite values, and
// the exact fp64 min / max as ordered 64-bit keys in C_QMIN / C_QMAX
cudaError_t launch_prepare_points_f64(const double* src, float* dst, uint64_t n, uint32_t d,
                                      uint32_t stride, unsigned long long* counters,
                                      cudaStream_t s);
// float <-> unsigned key with the same order (min/max by integer atomics)
__host__ __device__ __forceinline__ uint32_t ordered_key(float f) {
    uint32_t u;
#ifdef __CUDA_ARCH__
    u = __float_as_uint(f);
#else
    std::memcpy(&u, &f, 4);
#endif
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__host__ __device__ __forceinline__ uint64_t ordered_key64(double f) {
    uint64_t u;
#ifdef __CUDA_ARCH__
    u = (uint64_t)__double_as_longlong(f);
#else
    std::memcpy(&u, &f, 8);
#endif
    return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}
__host__ __device__ __forceinline__ double ordered_value64(uint64_t k) {
    const uint64_t u = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
    double f;
#ifdef __CUDA_ARCH__
    f = __longlong_as_double((long long)u);
#else
    std::memcpy(&f, &u, 8);
#endif
    return f;
}
__host__ __device__ __forceinline__ float ordered_value(uint32_t k) {
    const uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
    float f;
#ifdef __CUDA_ARCH__
    f = __uint_as_float(u);
#else
    std::memcpy(&f, &u, 4);
#endif
    return f;
}
// sngb_sampler.cu
void floyd_geometry(uint32_t draws, uint32_t& slots, uint32_t& col_words);
size_t floyd_scratch_bytes(uint32_t draws, int num_sms, uint64_t rows);
cudaError_t launch_sampler(const SamplerArgs& a, cudaStream_t s, int num_sms);
// launch_sampler would pick k_floyd_pipe for this problem (it likes 64 rows per block)
bool sampler_uses_pipe(uint64_t n, uint32_t draws);
// the head gather can hand its draws to k_floyd_pipe through global memory (SNGB_SHARE_T)
bool share_eligible(uint64_t n, uint32_t draws);
cudaError_t launch_gather(const GatherArgs& a, bool exhaustive, cudaStream_t s, int num_sms);
// exact fp64 decision of the band pairs; accepted ones go to `sink`
cudaError_t launch_band(const TestParams& tp, const EdgeSink& sink, unsigned long long* counters,
                        cudaStream_t s, int num_sms);
// sngb_metric.cu: Manhattan / cosine (fp32 filter + the reference's fp64 recheck)
cudaError_t launch_row_norms(const TestParams& tp, uint64_t n, float* rnorm,
                             unsigned long long* counters, cudaStream_t s, int num_sms);
cudaError_t launch_gather_metric(const GatherArgs& a, bool exhaustive, cudaStream_t s,
                                 int num_sms);
cudaError_t launch_extras_metric(const ExtrasArgs& a, cudaStream_t s, int num_sms);
// sngb_quant.cu: the 8-bit filter for wide rows (exact via integer thresholds
// on Q2 = sum (qa - qb)^2 plus the fp64 recheck in the band)
// 8-bit row layout: chunk 0 = (N over the first kHeadVals values, N over the
// row, 0, 0), chunks 1..nd the bytes; the head is chunks [0, kHead)
constexpr uint32_t kHead = 16;  // half a warp per head in k_gather_q8s
constexpr uint32_t kHeadVals = 16 * (kHead - 1);
constexpr uint32_t kSplitMinRW = 40;  // rows this wide take the early-reject gather
struct Q8Args {
    const uint4* rows;   // n rows of nd + 1 16-byte chunks: norm chunk, bytes, zero pad
    uint32_t nd;         // data chunks per row = ceil(d / 16)
    int32_t accept_max;  // Q2 <= accept_max: the reference accepts
    int32_t reject_min;  // Q2 >  reject_min: the reference rejects (else exact recheck)
};
constexpr uint32_t kQ8MaxD = 1520;  // widest rows of the 8-bit filter (3 chunks per lane)
struct Q8Plan {
    double s, lo;  // scale (a power of two) and offset (a multiple of s)
    Q8Args args;
    const uint32_t* perm = nullptr;  // device: stored value k = column perm[k] (null: identity)
};
// per-column sums and sums of squares (stats[0..d) and stats[d..2d)), fp64
cudaError_t launch_colstats(const float* pts, uint32_t stride, uint64_t n, uint32_t d,
                            const double* pts64, double* stats, cudaStream_t s, int num_sms);
bool q8_plan(double lo, double hi, uint32_t d, double eps2, Q8Plan& p);
bool q8_split(uint32_t nd);  // rows of nd data chunks take the early-reject gather
cudaError_t launch_quantize(const float* pts, uint32_t stride, uint64_t n, uint32_t d,
                            const Q8Plan& p, uint4* out, cudaStream_t s, int num_sms,
                            const double* pts64 = nullptr);
cudaError_t launch_gather_q8(const GatherArgs& a, const Q8Args& q, cudaStream_t s, int num_sms);
// bucketed partner lists of rows [a.row_begin, a.row_end) (a.nbuckets slices);
// draws <= 1024; see GatherArgs::partners
cudaError_t launch_partners(const GatherArgs& a, uint32_t* lists, uint32_t* offsets, cudaStream_t s,
                            int num_sms);
cudaError_t launch_extras_q8(const ExtrasArgs& a, const Q8Args& q, cudaStream_t s, int num_sms);
cudaError_t launch_extras(const ExtrasArgs& a, cudaStream_t s, int num_sms);
// Head filter for narrow rows (sngb_head.cu): a few coordinates per row in a
// compact L2-resident table, exact early reject, survivors take the fp32 test.
constexpr int kHeadU16x2 = 0, kHeadU8x4 = 1, kHeadU8x2 = 2;  // head formats (4, 4, 2 bytes)
#ifndef SNGB_HEAD_DEFAULT4
#define SNGB_HEAD_DEFAULT4 0
#endif
constexpr int kHeadDefault4 = SNGB_HEAD_DEFAULT4;  // the 4-byte format auto picks
struct HeadArgs {
    const void* head;  // n head words: coordinate j in bits [j*b, (j+1)*b), b = 16 or 8
    float reject;      // head Q (q units^2) > reject: the reference rejects
    int32_t kind;      // kHead*
    uint32_t coords;   // coordinates in the head (2 or min(d, 4))
};
struct HeadPlan {
    double s, lo;  // scale (a power of two) and offset (a multiple of s)
    HeadArgs args;
};
bool head_plan(double lo, double hi, uint32_t d, double eps2, int kind, HeadPlan& p);
cudaError_t launch_head_quantize(const float* pts, uint32_t stride, uint64_t n, const HeadPlan& p,
                                 void* out, cudaStream_t s, int num_sms);
cudaError_t launch_gather_head(const GatherArgs& a, const HeadArgs& h, cudaStream_t s, int num_sms);
// sngb_fused.cu: Floyd bookkeeping + head gather in one pass (large n, narrow rows);
// a.work must point at a zeroed counter (dynamic vertex claiming)
bool fused_eligible(uint64_t n, uint32_t draws, uint32_t stride);
// global scratch of the fused kernel (per-warp draw / group lists, replay list)
size_t fused_scratch_bytes(uint32_t draws, uint64_t rows, int num_sms);
cudaError_t launch_floyd_head(const SamplerArgs& sa, const GatherArgs& ga, const HeadArgs& h,
                              cudaStream_t s, int num_sms);

// ---- cluster stage (sngb_cluster.cu) ----
struct ClusterBuffers {
    unsigned long long* keys;     // in: raw keys (count), sorted in place via alt
    unsigned long long* keys_alt; // scratch of the same size
    uint32_t* deg;                // n
    uint8_t* core;                // n
    uint32_t* parent;             // n
    uint32_t* broot;              // n
    uint32_t* first;              // n
    uint32_t* flags;              // n + 1
    uint32_t* rank;               // n + 1
    void* temp;
    size_t temp_bytes;
    uint32_t* rstart = nullptr;   // n: first key of each vertex's run (null: edge-based rounds)
};

// Sort + unique raw keys; returns pointer to the unique keys (one of the two
// buffers) and writes the unique count to counters[C_UNIQUE].
cudaError_t sort_unique(unsigned long long* keys, unsigned long long* alt, uint64_t count,
                        uint32_t nb, void* temp, size_t temp_bytes,
                        unsigned long long* counters, unsigned long long** unique_out,
                        cudaStream_t s, uint64_t tri_n = 0);  // tri_n: canonical keys of
                                                              // n = tri_n points, 32-bit sort
size_t sort_unique_temp_bytes(uint64_t count, uint32_t nb);
size_t cluster_temp_bytes(uint64_t n);

// m_ptr: device pointer to the unique count (DeviceSelect output); m_max bounds it.
cudaError_t cluster_unique_edges(const unsigned long long* ukeys, const unsigned long long* m_ptr,
                                 uint64_t m_max, uint64_t n,
                                 uint32_t nb, int32_t min_pts, const ClusterBuffers& b,
                                 unsigned long long* counters, int32_t* labels, uint8_t* roles,
                                 cudaStream_t s, int num_sms);

// multi-GPU merge steps (sngb_cluster.cu); keys are canonical a<<32|b
cudaError_t merge_check_keys(const unsigned long long* keys, uint64_t m, uint64_t n,
                             unsigned long long* counters, cudaStream_t s, int num_sms);
cudaError_t merge_degrees(const unsigned long long* keys, uint64_t m, uint32_t* deg, cudaStream_t s,
                          int num_sms);
cudaError_t merge_components(const unsigned long long* keys, uint64_t m, uint64_t n,
                             const uint32_t* deg, int32_t min_pts, uint32_t* parent, uint8_t* core,
                             uint32_t* before, unsigned long long* counters, cudaStream_t s,
                             int num_sms);
cudaError_t merge_border(const unsigned long long* keys, uint64_t m, uint64_t n, const uint32_t* deg,
                         int32_t min_pts, const uint32_t* parent, uint32_t* border, uint8_t* core,
                         cudaStream_t s, int num_sms);
cudaError_t merge_relabel(uint64_t n, const uint32_t* deg, int32_t min_pts, const uint32_t* parent,
                          const uint32_t* border, const ClusterBuffers& b,
                          unsigned long long* counters, int32_t* labels, uint8_t* roles,
                          cudaStream_t s, int num_sms);
cudaError_t launch_convert_keys(const unsigned long long* in, unsigned long long* out, uint64_t m,
                                uint32_t nb, bool to_compact, uint64_t n,
                                unsigned long long* counters, cudaStream_t s, int num_sms);

}  // namespace sngb
