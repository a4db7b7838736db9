// tools/microbench.cu -- B200 measurements that set this project's rooflines
// and pick between sampler designs.  Not part of the product.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
//   tools/microbench            (one JSON object per line)
//
// 1. shared-memory op throughput (random addresses, per-warp private regions):
//    LDS.32, STS.32, ATOMS.CAS.32, ATOMS.CAS.64, ATOMS.OR.32, MATCH.ANY
// 2. the RNG draw (mix + Lemire) throughput
// 3. random row gather bandwidth (algorithmic bytes / s) from an L2-resident
//    table and from an HBM-resident table, for the row sizes of the workloads.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#include "../paper_2006_06743_b200/csrc/sngb_rng.cuh"

#define CK(x)                                                                                 \
    do {                                                                                      \
        cudaError_t e = (x);                                                                  \
        if (e != cudaSuccess) {                                                               \
            fprintf(stderr, "%s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);      \
            exit(1);                                                                          \
        }                                                                                     \
    } while (0)

__device__ __forceinline__ uint32_t xs32(uint32_t x) {
    x ^= x << 13;
    x ^= x >> 17;
    x ^= x << 5;
    return x;
}

constexpr int kOps = 4096;

// op: 0 LDS, 1 STS, 2 CAS32, 3 CAS64, 4 OR32, 5 MATCH
template <int OP>
__global__ void k_smem(unsigned long long* sink, uint32_t words_per_warp_log2) {
    extern __shared__ uint32_t sm[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t* base = sm + (w << words_per_warp_log2);
    const uint32_t mask = (1u << words_per_warp_log2) - 1;
    uint32_t x = 0x9e3779b9u * (threadIdx.x + 1) + blockIdx.x;
    uint32_t acc = 0;
    for (int i = lane; i < (1 << words_per_warp_log2); i += 32) base[i] = i;
    __syncwarp();
#pragma unroll 8
    for (int k = 0; k < kOps; ++k) {
        x = xs32(x);
        const uint32_t a = x & mask;
        if (OP == 0) acc += ((volatile uint32_t*)base)[a];
        if (OP == 1) ((volatile uint32_t*)base)[a] = x;
        if (OP == 2) acc += atomicCAS(&base[a], x, acc);
        if (OP == 3)
            acc += (uint32_t)atomicCAS(reinterpret_cast<unsigned long long*>(base) + (a >> 1),
                                       (unsigned long long)x, (unsigned long long)acc);
        if (OP == 4) acc += atomicOr(&base[a], x);
        if (OP == 5) acc += __match_any_sync(0xffffffffu, x & 0xffff);
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

// the product's draw: sngb::mix (sngb_rng.cuh; its 64-bit constant multiplies are one
// IMAD.WIDE and two chained IMADs since round 2)
using sngb::mix;

__global__ void k_rng(unsigned long long* sink, uint32_t draws) {
    const uint64_t key = mix(blockIdx.x * 1024ull + threadIdx.x);
    uint32_t acc = 0;
    for (uint32_t i = 0; i < draws; ++i) {
        const uint64_t x = mix(key + (uint64_t)(i + 1) * 0x9e3779b97f4a7c15ULL);
        const uint32_t b = 1000000u + i;
        const uint64_t p1 = (uint64_t)(uint32_t)x * b;
        const uint64_t s = (uint64_t)(uint32_t)(x >> 32) * b + (p1 >> 32);
        acc += (uint32_t)(s >> 32) + (((uint32_t)s == 0u) ? 1u : 0u);
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

// Random row gather: each group of G lanes reads one random row of `vec`
// float4s (row = vec*16 bytes) per iteration.
template <int G>
__global__ void k_gather_rows(const float4* __restrict__ tab, uint64_t rows, uint32_t vec,
                              uint32_t iters, unsigned long long* sink) {
    const int lane = threadIdx.x & 31, q = lane % G, g = lane / G;
    uint32_t x = 0x9e3779b9u * (blockIdx.x * blockDim.x + threadIdx.x / G * G + 1);
    float acc = 0.f;
    for (uint32_t it = 0; it < iters; ++it) {
        x = xs32(x + g);
        const uint64_t r = (uint64_t)x * rows >> 32;
        for (uint32_t c = q; c < vec; c += G) {
            const float4 v = __ldg(tab + r * vec + c);
            acc += v.x + v.y + v.z + v.w;
        }
    }
    if (acc == 1234.5f) sink[0] = 1;
}

// Lean random-row gather: 8 lanes per 128-byte row, UN rows in flight per
// group, minimal index math -- the random-row ceiling without our kernel's
// per-pair work.
template <int UN>
__global__ void k_gather_lean(const float4* __restrict__ tab, uint64_t rows, uint32_t iters,
                              unsigned long long* sink) {
    const int lane = threadIdx.x & 31, q = lane & 7, g = lane >> 3;
    uint32_t x = 0x9e3779b9u * (blockIdx.x * blockDim.x + (threadIdx.x & ~7) + 1);
    float acc = 0.f;
    for (uint32_t it = 0; it < iters; ++it) {
        float4 v[UN];
#pragma unroll
        for (int k = 0; k < UN; ++k) {
            x = xs32(x + g + k);
            const uint64_t r = (uint64_t)x * rows >> 32;
            v[k] = __ldg(tab + r * 8 + q);
        }
#pragma unroll
        for (int k = 0; k < UN; ++k) acc += v[k].x + v[k].y + v[k].z + v[k].w;
    }
    if (acc == 1234.5f) sink[0] = 1;
}

// Coalesced re-reads of an L2-resident buffer: `passes` sweeps, grid-stride.
__global__ void k_stream(const float4* __restrict__ tab, uint64_t n4, int passes,
                         unsigned long long* sink) {
    float acc = 0.f;
    for (int p = 0; p < passes; ++p)
        for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
             i += (uint64_t)gridDim.x * blockDim.x) {
            const float4 v = __ldg(tab + i);
            acc += v.x + v.y + v.z + v.w;
        }
    if (acc == 1234.5f) sink[0] = 1;
}

template <typename F>
float time_ms(F&& f, int reps = 5) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    f();
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        CK(cudaEventRecord(a));
        f();
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        if (ms < best) best = ms;
    }
    return best;
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    unsigned long long* sink;
    CK(cudaMalloc(&sink, 64));
    const int threads = 256, log2w = 11;  // 8 KB per warp -> 64 KB per block
    const size_t smem = (size_t)(threads / 32) << log2w << 2;
    const int blocks = sms * 3;
    const char* names[] = {"lds32", "sts32", "atoms_cas32", "atoms_cas64", "atoms_or32",
                           "match_any"};
    auto run_smem = [&](int op) {
        switch (op) {
#define CASE(K)                                                                                \
    case K:                                                                                    \
        CK(cudaFuncSetAttribute(k_smem<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,        \
                                (int)smem));                                                   \
        return time_ms([&] { k_smem<K><<<blocks, threads, smem>>>(sink, log2w); });
            CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5)
#undef CASE
        }
        return 0.f;
    };
    for (int op = 0; op < 6; ++op) {
        const float ms = run_smem(op);
        const double ops = (double)blocks * threads * kOps;
        const double per_sm_cycle = ops / (ms * 1e-3) / sms / 1.965e9;  // lane-ops / SM / cycle
        printf("{\"bench\": \"%s\", \"lane_ops_per_s\": %.4g, \"lane_ops_per_sm_cycle_at_1965\": %.3f}\n",
               names[op], ops / (ms * 1e-3), per_sm_cycle);
    }
    {
        const uint32_t draws = 4096;
        const int b = sms * 8;
        const float ms = time_ms([&] { k_rng<<<b, 256>>>(sink, draws); });
        const double n = (double)b * 256 * draws;
        printf("{\"bench\": \"rng_draw\", \"draws_per_s\": %.4g, \"draws_per_sm_cycle_at_1965\": %.3f}\n",
               n / (ms * 1e-3), n / (ms * 1e-3) / sms / 1.965e9);
    }
    // gathers
    struct Case {
        const char* name;
        size_t table_bytes;
        uint32_t vec;  // float4 per row
    } cases[] = {
        {"l2_row16B_60MB", 60ull << 20, 1},    {"l2_row16B_80MB", 80ull << 20, 1},
        {"l2_row64B_64MB", 64ull << 20, 4},    {"l2_row128B_64MB", 64ull << 20, 8},
        {"hbm_row16B_2GB", 2ull << 30, 1},     {"hbm_row128B_2.5GB", 2560ull << 20, 8},
        {"hbm_row3136B_2GB", 2ull << 30, 196}, {"mixed_row3136B_220MB", 220ull << 20, 196},
        {"l2_row3136B_55MB", 55ull << 20, 196}, {"l2_row3136B_32MB", 32ull << 20, 196},
    };
    float4* tab;
    CK(cudaMalloc(&tab, 2560ull << 20));
    CK(cudaMemset(tab, 0, 2560ull << 20));
    for (auto& c : cases) {
        const uint64_t rows = c.table_bytes / (16ull * c.vec);
        const int b = sms * 8;
        const uint32_t iters = c.vec >= 64 ? 64 : (c.vec >= 4 ? 256 : 1024);
        float ms;
        int G = c.vec == 1 ? 1 : (c.vec == 4 ? 4 : (c.vec == 8 ? 8 : 32));
        auto launch = [&] {
            if (G == 1) k_gather_rows<1><<<b, 256>>>(tab, rows, c.vec, iters, sink);
            else if (G == 4) k_gather_rows<4><<<b, 256>>>(tab, rows, c.vec, iters, sink);
            else if (G == 8) k_gather_rows<8><<<b, 256>>>(tab, rows, c.vec, iters, sink);
            else k_gather_rows<32><<<b, 256>>>(tab, rows, c.vec, iters, sink);
        };
        ms = time_ms(launch);
        const double nrows = (double)b * (256 / G) * iters;
        const double bytes = nrows * c.vec * 16;
        printf("{\"bench\": \"gather_%s\", \"rows_per_s\": %.4g, \"GB_per_s\": %.1f}\n", c.name,
               nrows / (ms * 1e-3), bytes / (ms * 1e-3) / 1e9);
    }
    {
        const uint64_t rows = (2560ull << 20) / 128;
        for (int bpsm : {4, 8}) {
            const int b = sms * bpsm;
            const uint32_t iters = 64;
            auto l8 = [&] { k_gather_lean<8><<<b, 256>>>(tab, rows, iters, sink); };
            auto l16 = [&] { k_gather_lean<16><<<b, 256>>>(tab, rows, iters, sink); };
            const float m8 = time_ms(l8), m16 = time_ms(l16);
            const double r8 = (double)b * 32 * iters * 8, r16 = (double)b * 32 * iters * 16;
            printf("{\"bench\": \"gather_hbm_row128B_lean_u8_b%d\", \"GB_per_s\": %.1f}\n", bpsm,
                   r8 * 128 / (m8 * 1e-3) / 1e9);
            printf("{\"bench\": \"gather_hbm_row128B_lean_u16_b%d\", \"GB_per_s\": %.1f}\n", bpsm,
                   r16 * 128 / (m16 * 1e-3) / 1e9);
        }
    }
    // L2 streaming read: every warp reads a 32 MB L2-resident buffer with
    // coalesced 16-byte loads (the L2 -> SM bandwidth ceiling)
    {
        const size_t bytes = 32ull << 20;
        const uint64_t n4 = bytes / 16;
        const int b = sms * 8;
        auto launch = [&] { k_stream<<<b, 256>>>(tab, n4, 8, sink); };
        const float ms = time_ms(launch);
        const double total = (double)b * 256 * 8 * (n4 / ((double)b * 256)) * 16;
        printf("{\"bench\": \"l2_stream_read_32MB\", \"GB_per_s\": %.1f}\n",
               (double)n4 * 16 * 8 / (ms * 1e-3) / 1e9);
        (void)total;
    }
    return 0;
}
