// gather_ceiling.cu -- measured ceilings for the random-row gather at every
// BASELINE row shape and table size (the roofline denominators bench.py
// reports as l2_gather_peak / hbm_gather_peak).  Not part of the product.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather_ceiling tools/gather_ceiling.cu
//   tools/gather_ceiling > profiles/<round>_gather_ceilings.jsonl
//
// k_lean<G, V, UN>: a group of G lanes reads a random row of W float4 (lane q
// takes columns q, q+G, ...; V = ceil(W/G)), UN independent rows in flight per
// group per iteration.  Row indices are a hash of (group, iteration, k) -- no
// dependency chain -- and the loaded values feed one running sum so nothing is
// dead code.  A case may read only the first R chunks of each row (the
// 8-bit gather's head: k_gather_q8s reads 256 B of every 800-B row).  Every case is swept over UN and resident blocks per SM and the
// best rate is reported: an upper bound for a kernel that also has to do
// per-pair work, not an estimate of one.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                            \
    do {                                                                                 \
        cudaError_t e = (x);                                                             \
        if (e != cudaSuccess) {                                                          \
            fprintf(stderr, "%s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            return 1;                                                                    \
        }                                                                                \
    } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    return x;
}

template <int G, int V, int UN>
__global__ void __launch_bounds__(256) k_lean(const float4* __restrict__ tab, uint64_t rows,
                                              uint32_t W, uint32_t R, uint32_t iters, float* sink) {
    const int lane = threadIdx.x & 31, q = lane % G;
    const uint32_t grp = (blockIdx.x * blockDim.x + threadIdx.x) / G;
    float acc = 0.f;
    for (uint32_t it = 0; it < iters; ++it) {
        float4 v[UN][V];
#pragma unroll
        for (int k = 0; k < UN; ++k) {
            const uint32_t h = hash32(grp * 0x9E3779B1u + it * UN + k);
            const uint64_t r = ((uint64_t)h * rows) >> 32;
            const float4* row = tab + r * W + q;
#pragma unroll
            for (int c = 0; c < V; ++c)
                v[k][c] = (q + G * c < (int)R) ? __ldg(row + G * c) : make_float4(0, 0, 0, 0);
        }
#pragma unroll
        for (int k = 0; k < UN; ++k)
#pragma unroll
            for (int c = 0; c < V; ++c) acc += (v[k][c].x + v[k][c].y) + (v[k][c].z + v[k][c].w);
    }
    if (acc == 1234.5f) sink[0] = acc;
}

// 4- and 2-byte rows (the head tables of sngb_head.cu): one element per row per lane
template <int UN, typename T = uint32_t>
__global__ void __launch_bounds__(256) k_lean32(const T* __restrict__ tab, uint64_t rows,
                                                uint32_t iters, float* sink) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    for (uint32_t it = 0; it < iters; ++it) {
        uint32_t v[UN];
#pragma unroll
        for (int k = 0; k < UN; ++k) {
            const uint32_t h = hash32(t * 0x9E3779B1u + it * UN + k);
            v[k] = __ldg(tab + (((uint64_t)h * rows) >> 32));
        }
#pragma unroll
        for (int k = 0; k < UN; ++k) acc += v[k];
    }
    if (acc == 12345u) sink[0] = (float)acc;
}

template <class F>
float time_ms(F&& f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();  // warm-up
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(a);
        f();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    return best;
}

template <int UN, typename T = uint32_t>
double run32(size_t table_bytes, const float4* tab, float* sink, int sms, int bpsm) {
    const uint64_t rows = table_bytes / sizeof(T);
    const int blocks = sms * bpsm;
    const double threads = (double)blocks * 256;
    uint32_t iters = (uint32_t)(1e10 / (threads * UN * 32));
    if (iters < 4) iters = 4;
    const float ms = time_ms([&] {
        k_lean32<UN, T><<<blocks, 256>>>(reinterpret_cast<const T*>(tab), rows, iters, sink);
    });
    return threads * iters * UN / (ms * 1e-3);  // rows per second
}

struct Case {
    const char* name;
    size_t table_bytes;
    uint32_t row_bytes;  // stride in the padded device layout
    uint32_t read_bytes = 0;  // bytes read from the start of each row (0: all)
};

template <int G, int V, int UN>
double run(const Case& c, const float4* tab, float* sink, int sms, int bpsm) {
    const uint32_t W = c.row_bytes / 16;
    const uint32_t rb = c.read_bytes ? c.read_bytes : c.row_bytes, R = rb / 16;
    const uint64_t rows = c.table_bytes / c.row_bytes;
    const int blocks = sms * bpsm;
    const double groups = (double)blocks * 256 / G;
    // ~2 GB of rows per launch, at least 4 iterations
    uint32_t iters = (uint32_t)(2e9 / (groups * UN * rb));
    if (iters < 4) iters = 4;
    const float ms =
        time_ms([&] { k_lean<G, V, UN><<<blocks, 256>>>(tab, rows, W, R, iters, sink); });
    const double nrows = groups * iters * UN;
    return nrows * rb / (ms * 1e-3) / 1e9;  // GB/s of the bytes read
}

template <int G, int V>
void sweep(const Case& c, const float4* tab, float* sink, int sms) {
    double best = 0;
    int bu = 0, bb = 0;
    for (int bpsm : {2, 4, 8}) {
        const double r1 = run<G, V, 2>(c, tab, sink, sms, bpsm);
        const double r2 = run<G, V, 4>(c, tab, sink, sms, bpsm);
        const double r3 = run<G, V, 8>(c, tab, sink, sms, bpsm);
        if (r1 > best) best = r1, bu = 2, bb = bpsm;
        if (r2 > best) best = r2, bu = 4, bb = bpsm;
        if (r3 > best) best = r3, bu = 8, bb = bpsm;
    }
    const uint32_t rb = c.read_bytes ? c.read_bytes : c.row_bytes;
    printf("{\"bench\": \"ceiling_%s\", \"row_bytes\": %u, \"read_bytes\": %u, \"table_MB\": %.1f, "
           "\"GB_per_s\": %.1f, \"rows_per_s\": %.4g, \"best_rows_in_flight_per_group\": %d, "
           "\"best_blocks_per_sm\": %d}\n",
           c.name, c.row_bytes, rb, c.table_bytes / 1048576.0, best, best * 1e9 / rb, bu, bb);
    fflush(stdout);
}

int main(int argc, char** argv) {
    // any argument: just the newest cases ("q5": the cfg5 reduced-precision tables)
    const bool only_new = argc > 1;
    const bool q5 = argc > 1 && argv[1][0] == 'q';
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const size_t max_bytes = 2560ull << 20;
    float4* tab;
    float* sink;
    CK(cudaMalloc(&tab, max_bytes));
    CK(cudaMemset(tab, 0, max_bytes));
    CK(cudaMalloc(&sink, 64));
    // the configs' shapes: cfg1 8-B rows (float2, 0.16 MB) is covered by the
    // 16-B case on a small table; cfg4 pads 12-B rows to 16 B.
    const Case c1{"cfg1_row16B_0.3MB", 320ull << 10, 16};
    const Case c4{"cfg4_row16B_80MB", 80ull << 20, 16};
    const Case c3{"cfg3_row64B_64MB", 64ull << 20, 64};
    const Case c5{"cfg5_row128B_2560MB", 2560ull << 20, 128};
    const Case c2l2{"cfg2_row3136B_55MB_slice", 55ull << 20, 3136};
    const Case c2hbm{"cfg2_row3136B_220MB_full", 220ull << 20, 3136};
    const Case c2q8{"cfg2_q8_row800B_56MB", 56ull << 20, 800};
    if (!only_new) {
        sweep<1, 1>(c1, tab, sink, sms);
        sweep<1, 1>(c4, tab, sink, sms);
        sweep<4, 1>(c3, tab, sink, sms);
        sweep<8, 1>(c5, tab, sink, sms);
        sweep<32, 7>(c2l2, tab, sink, sms);
        sweep<32, 7>(c2hbm, tab, sink, sms);
        sweep<32, 2>(c2q8, tab, sink, sms);
    }
    if (q5) {
        // cfg5 (20 M rows, d = 32) as 8-bit (32-B rows, 640 MB), 16-bit (64 B, 1280 MB)
        // and 4-bit (16 B, 320 MB) tables: random rows from HBM at sector granularity
        const Case c5q8{"cfg5_q8_row32B_640MB", 640ull << 20, 32};
        const Case c5q16{"cfg5_q16_row64B_1280MB", 1280ull << 20, 64};
        const Case c5q4{"cfg5_q4_row16B_320MB", 320ull << 20, 16};
        sweep<1, 1>(c5q4, tab, sink, sms);
        sweep<2, 1>(c5q8, tab, sink, sms);
        sweep<4, 1>(c5q16, tab, sink, sms);
        // the head filter's tables: 4-byte rows for cfg3 (1 M rows, 4 MB), cfg4 (5 M,
        // 20 MB) and a 20 M-row 80 MB table; 2-byte rows for cfg5 (20 M rows, 40 MB)
        auto head_case = [&](size_t bytes, int eb, const char* tag) {
            double best = 0;
            int bu = 0, bb = 0;
            for (int bpsm : {2, 4, 8}) {
                double r[3];
                if (eb == 4) {
                    r[0] = run32<2>(bytes, tab, sink, sms, bpsm);
                    r[1] = run32<4>(bytes, tab, sink, sms, bpsm);
                    r[2] = run32<8>(bytes, tab, sink, sms, bpsm);
                } else {
                    r[0] = run32<2, unsigned short>(bytes, tab, sink, sms, bpsm);
                    r[1] = run32<4, unsigned short>(bytes, tab, sink, sms, bpsm);
                    r[2] = run32<8, unsigned short>(bytes, tab, sink, sms, bpsm);
                }
                for (int j = 0; j < 3; ++j)
                    if (r[j] > best) best = r[j], bu = 2 << j, bb = bpsm;
            }
            printf("{\"bench\": \"ceiling_%s\", \"row_bytes\": %d, \"read_bytes\": %d, "
                   "\"table_MB\": %zu, \"GB_per_s\": %.1f, \"rows_per_s\": %.4g, "
                   "\"best_rows_in_flight_per_group\": %d, \"best_blocks_per_sm\": %d}\n",
                   tag, eb, eb, bytes >> 20, best * eb / 1e9, best, bu, bb);
            fflush(stdout);
        };
        head_case(80ull << 20, 4, "head4B_80MB");
        head_case(4ull << 20, 4, "head4B_4MB");
        head_case(20ull << 20, 4, "head4B_20MB");
        head_case(40ull << 20, 2, "head2B_40MB");
        return 0;
    }
    const Case c2q8h{"cfg2_q8_head256B_of_row800B_56MB", 56ull << 20, 800, 256};
    sweep<16, 1>(c2q8h, tab, sink, sms);
    return 0;
}
