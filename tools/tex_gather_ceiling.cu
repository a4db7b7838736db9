// tex_gather_ceiling.cu -- do the texture units fetch random 2-/4-byte heads
// faster than LDG?  Not part of the product.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tex_gather_ceiling tools/tex_gather_ceiling.cu
//   tools/tex_gather_ceiling > profiles/<round>_tex_gather.jsonl
//
// The head-filter gather (sngb_head.cu) is bound by L1TEX: a divergent LDG whose
// 32 lanes hit 32 lines costs 32 wavefronts, about one per SM-cycle
// (profiles/r02_tma_gather.jsonl: 2.9e11 random heads/s).  tex1Dfetch on a
// linear texture takes the TEX path of the same unit; this times it against
// the LDG baseline on the same tables (u16 and u32 heads, 2 / 40 / 80 MB).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

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

template <typename T, int UN>
__global__ void __launch_bounds__(256) k_ldg(const T* __restrict__ tab, uint32_t rows,
                                             uint32_t iters, uint32_t* sink) {
    const uint32_t gid = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    for (uint32_t it = 0; it < iters; ++it) {
        T v[UN];
#pragma unroll
        for (int k = 0; k < UN; ++k) {
            const uint32_t h = hash32(gid * 0x9E3779B1u + it * UN + k);
            v[k] = __ldg(tab + (uint32_t)(((uint64_t)h * rows) >> 32));
        }
#pragma unroll
        for (int k = 0; k < UN; ++k) acc ^= (uint32_t)v[k];
    }
    if (acc == 0x7fffu && gid == 0u) sink[0] = acc;
}

template <typename T, int UN>
__global__ void __launch_bounds__(256) k_tex(cudaTextureObject_t tex, uint32_t rows, uint32_t iters,
                                             uint32_t* sink) {
    const uint32_t gid = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    for (uint32_t it = 0; it < iters; ++it) {
        T v[UN];
#pragma unroll
        for (int k = 0; k < UN; ++k) {
            const uint32_t h = hash32(gid * 0x9E3779B1u + it * UN + k);
            v[k] = tex1Dfetch<T>(tex, (int)(((uint64_t)h * rows) >> 32));
        }
#pragma unroll
        for (int k = 0; k < UN; ++k) acc ^= (uint32_t)v[k];
    }
    if (acc == 0x7fffu && gid == 0u) sink[0] = acc;
}

template <typename F>
static double time_ms(F launch) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(a);
        launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    return best;
}

template <typename T>
static int run(const char* name, int sms, int clk, uint32_t* sink) {
    for (uint64_t mb : {2ull, 40ull, 80ull}) {
        const uint32_t rows = (uint32_t)(mb * 1000000ull / sizeof(T));
        T* tab;
        CK(cudaMalloc(&tab, (size_t)rows * sizeof(T)));
        CK(cudaMemset(tab, 0x5a, (size_t)rows * sizeof(T)));
        cudaResourceDesc rd = {};
        rd.resType = cudaResourceTypeLinear;
        rd.res.linear.devPtr = tab;
        rd.res.linear.desc = cudaCreateChannelDesc<T>();
        rd.res.linear.sizeInBytes = (size_t)rows * sizeof(T);
        cudaTextureDesc td = {};
        td.readMode = cudaReadModeElementType;
        cudaTextureObject_t tex = 0;
        CK(cudaCreateTextureObject(&tex, &rd, &td, nullptr));
        for (int bpsm : {2, 4, 8}) {
            const int grid = sms * bpsm;
            const double threads = (double)grid * 256;
            const uint32_t it = 256;
            double ms = time_ms([&] { k_ldg<T, 8><<<grid, 256>>>(tab, rows, it, sink); });
            CK(cudaGetLastError());
            double rps = threads * it * 8.0 / (ms * 1e-3);
            printf("{\"case\": \"ldg_%s\", \"table_mb\": %llu, \"bpsm\": %d, \"rows_per_s\": %.4g, \"per_sm_cycle\": %.3f}\n",
                   name, (unsigned long long)mb, bpsm, rps, rps / (sms * (clk * 1e3)));
            ms = time_ms([&] { k_tex<T, 8><<<grid, 256>>>(tex, rows, it, sink); });
            CK(cudaGetLastError());
            rps = threads * it * 8.0 / (ms * 1e-3);
            printf("{\"case\": \"tex_%s\", \"table_mb\": %llu, \"bpsm\": %d, \"rows_per_s\": %.4g, \"per_sm_cycle\": %.3f}\n",
                   name, (unsigned long long)mb, bpsm, rps, rps / (sms * (clk * 1e3)));
            fflush(stdout);
        }
        CK(cudaDestroyTextureObject(tex));
        CK(cudaFree(tab));
    }
    return 0;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    uint32_t* sink;
    CK(cudaMalloc(&sink, 4));
    if (run<unsigned short>("u16", sms, clk, sink)) return 1;
    if (run<unsigned int>("u32", sms, clk, sink)) return 1;
    return 0;
}
