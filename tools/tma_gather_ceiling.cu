// tma_gather_ceiling.cu -- can the TMA unit fetch random small rows faster than
// LDG?  Not part of the product.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_gather_ceiling tools/tma_gather_ceiling.cu
//   tools/tma_gather_ceiling > profiles/<round>_tma_gather.jsonl
//
// A divergent LDG whose 32 lanes hit 32 different 128-B lines costs 32 L1TEX
// wavefronts, and L1TEX retires about one wavefront per SM-cycle
// (B300_MICROARCH.md "L1tex wavefront queue"): 148 SMs x 1.965 GHz = 2.9e11
// random rows/s, exactly the ceiling of the head-filter gather
// (profiles/r01_gather_ceilings.jsonl).  Three ways around L1TEX are timed
// against the LDG baseline on the same table (u16 heads, `rows16` 16-byte rows):
//
//   ldg      each lane LDG.U16 of UN random heads per iteration
//   g4       each lane issues one cp.async.bulk.tensor.2d ... tile::gather4 per
//            iteration: 4 random 16-B rows -> 64 B of shared memory, completion
//            on a per-warp mbarrier, S stages in flight
//   bulk     each lane issues UN cp.async.bulk (16 B, 1-D) per iteration
//
// Every fetched head feeds a running XOR, so nothing is dead code.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

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

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W;\n\t}" ::"r"(a),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void g4(uint32_t dst, const CUtensorMap* tm, uint32_t mbar, int c0,
                                   int r0, int r1, int r2, int r3) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst),
        "l"(tm), "r"(mbar), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
        : "memory");
}
__device__ __forceinline__ void bulk16(uint32_t dst, const void* src, uint32_t mbar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];" ::"r"(dst),
        "l"(src), "r"(mbar)
        : "memory");
}

template <int UN>
__global__ void __launch_bounds__(256) k_ldg(const uint16_t* __restrict__ tab, uint32_t rows,
                                             uint32_t iters, uint32_t* sink) {
    const uint32_t gid = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    for (uint32_t it = 0; it < iters; ++it) {
        uint16_t v[UN];
#pragma unroll
        for (int k = 0; k < UN; ++k) {
            const uint32_t h = hash32(gid * 0x9E3779B1u + it * UN + k);
            const uint32_t r = (uint32_t)(((uint64_t)h * rows) >> 32);
            v[k] = __ldg(tab + r);
        }
#pragma unroll
        for (int k = 0; k < UN; ++k) acc ^= v[k];
    }
    if (acc == 0x7fffu && gid == 0u) sink[0] = acc;
}

// S stages per warp; a stage = 32 lanes x 4 rows x 16 B = 2 KB
template <int S>
__global__ void __launch_bounds__(256) k_g4(const __grid_constant__ CUtensorMap tm, uint32_t rows16,
                                            uint32_t iters, uint32_t* sink) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) unsigned long long mb[8][S];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t gid = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned char* buf = sm + (size_t)w * S * 4096;
    if (lane == 0)
        for (int s = 0; s < S; ++s) mbar_init(smem_u32(&mb[w][s]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    uint32_t acc = 0;
    uint32_t sub[S];  // head within the 16-B row, 4 x 3 bits per stage
    auto issue = [&](uint32_t it, int s) {
        uint32_t r[4], sb = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t h = hash32(gid * 0x9E3779B1u + it * 4 + k);
            const uint32_t e = (uint32_t)(((uint64_t)h * (rows16 * 8ull)) >> 32);
            r[k] = e >> 3;
            sb |= (e & 7u) << (3 * k);
        }
        sub[s] = sb;
        const uint32_t mbar = smem_u32(&mb[w][s]);
        if (lane == 0) mbar_expect_tx(mbar, 2048);
        __syncwarp();
        g4(smem_u32(buf + s * 4096 + lane * 128), &tm, mbar, 0, r[0], r[1], r[2], r[3]);
    };
#pragma unroll
    for (int s = 0; s < S; ++s) issue(s, s);
    uint32_t ph = 0;
    for (uint32_t it = 0; it < iters; ++it) {
#pragma unroll
        for (int s = 0; s < S; ++s) {
            mbar_wait(smem_u32(&mb[w][s]), ph);
            const uint16_t* st = reinterpret_cast<const uint16_t*>(buf + s * 4096 + lane * 128);
#pragma unroll
            for (int k = 0; k < 4; ++k) acc ^= st[k * 8 + ((sub[s] >> (3 * k)) & 7u)];
            __syncwarp();
            issue((it + 1) * S + s, s);
        }
        ph ^= 1u;
    }
#pragma unroll
    for (int s = 0; s < S; ++s) mbar_wait(smem_u32(&mb[w][s]), ph);
    if (acc == 0x7fffu && gid == 0u) sink[0] = acc;
}

// 1-D bulk copies: each lane 4 x 16 B per stage
template <int S>
__global__ void __launch_bounds__(256) k_bulk(const uint16_t* __restrict__ tab, uint32_t rows16,
                                              uint32_t iters, uint32_t* sink) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) unsigned long long mb[8][S];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t gid = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned char* buf = sm + (size_t)w * S * 4096;
    if (lane == 0)
        for (int s = 0; s < S; ++s) mbar_init(smem_u32(&mb[w][s]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    uint32_t acc = 0;
    uint32_t sub[S];
    auto issue = [&](uint32_t it, int s) {
        uint32_t sb = 0;
        const uint32_t mbar = smem_u32(&mb[w][s]);
        if (lane == 0) mbar_expect_tx(mbar, 2048);
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t h = hash32(gid * 0x9E3779B1u + it * 4 + k);
            const uint32_t e = (uint32_t)(((uint64_t)h * (rows16 * 8ull)) >> 32);
            sb |= (e & 7u) << (3 * k);
            bulk16(smem_u32(buf + s * 4096 + lane * 128 + k * 16), tab + (size_t)(e >> 3) * 8, mbar);
        }
        sub[s] = sb;
    };
#pragma unroll
    for (int s = 0; s < S; ++s) issue(s, s);
    uint32_t ph = 0;
    for (uint32_t it = 0; it < iters; ++it) {
#pragma unroll
        for (int s = 0; s < S; ++s) {
            mbar_wait(smem_u32(&mb[w][s]), ph);
            const uint16_t* st = reinterpret_cast<const uint16_t*>(buf + s * 4096 + lane * 128);
#pragma unroll
            for (int k = 0; k < 4; ++k) acc ^= st[k * 8 + ((sub[s] >> (3 * k)) & 7u)];
            __syncwarp();
            issue((it + 1) * S + s, s);
        }
        ph ^= 1u;
    }
#pragma unroll
    for (int s = 0; s < S; ++s) mbar_wait(smem_u32(&mb[w][s]), ph);
    if (acc == 0x7fffu && gid == 0u) sink[0] = acc;
}


// Mixed: every lane keeps S gather4 stages in flight AND does UN LDG lookups per
// stage wait.  If the TMA unit's path to L2 were independent of the LSU / L1TEX tag
// stage the two rates would add (1.0 + 0.6 per SM-cycle).
template <int S, int UN>
__global__ void __launch_bounds__(256) k_mix(const __grid_constant__ CUtensorMap tm,
                                             const uint16_t* __restrict__ tab, uint32_t rows16,
                                             uint32_t iters, uint32_t* sink) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) unsigned long long mb[8][S];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t gid = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned char* buf = sm + (size_t)w * S * 4096;
    if (lane == 0)
        for (int s = 0; s < S; ++s) mbar_init(smem_u32(&mb[w][s]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    uint32_t acc = 0;
    uint32_t sub[S];
    auto issue = [&](uint32_t it, int s) {
        uint32_t r[4], sb = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t h = hash32(gid * 0x9E3779B1u + it * 4 + k);
            const uint32_t e = (uint32_t)(((uint64_t)h * (rows16 * 8ull)) >> 32);
            r[k] = e >> 3;
            sb |= (e & 7u) << (3 * k);
        }
        sub[s] = sb;
        const uint32_t mbar = smem_u32(&mb[w][s]);
        if (lane == 0) mbar_expect_tx(mbar, 2048);
        __syncwarp();
        g4(smem_u32(buf + s * 4096 + lane * 128), &tm, mbar, 0, r[0], r[1], r[2], r[3]);
    };
#pragma unroll
    for (int s = 0; s < S; ++s) issue(s, s);
    uint32_t ph = 0;
    for (uint32_t it = 0; it < iters; ++it) {
#pragma unroll
        for (int s = 0; s < S; ++s) {
            uint16_t v[UN];
#pragma unroll
            for (int k = 0; k < UN; ++k) {  // the LDG lookups ride on the stage's latency
                const uint32_t h = hash32(~gid * 0x85EBCA6Bu + (it * S + s) * UN + k);
                v[k] = __ldg(tab + (uint32_t)(((uint64_t)h * (rows16 * 8ull)) >> 32));
            }
            mbar_wait(smem_u32(&mb[w][s]), ph);
            const uint16_t* st = reinterpret_cast<const uint16_t*>(buf + s * 4096 + lane * 128);
#pragma unroll
            for (int k = 0; k < 4; ++k) acc ^= st[k * 8 + ((sub[s] >> (3 * k)) & 7u)];
#pragma unroll
            for (int k = 0; k < UN; ++k) acc ^= v[k];
            __syncwarp();
            issue((it + 1) * S + s, s);
        }
        ph ^= 1u;
    }
#pragma unroll
    for (int s = 0; s < S; ++s) mbar_wait(smem_u32(&mb[w][s]), ph);
    if (acc == 0x7fffu && gid == 0u) sink[0] = acc;
}


// Wide rows (the 8-bit gather's heads: the first 256 B of random 800-B rows,
// cfg2's 56 MB table).  ldg: half a warp per row (16 lanes x 16 B), UN rows
// in flight per half warp.  g4w: lanes 0..7 each issue one gather4 (4 rows x
// 256 B) per stage, so a stage is 32 rows = 8 KB; the warp then reads them
// back from shared memory (16 B per lane per row).
template <int UN>
__global__ void __launch_bounds__(256) k_ldg_wide(const uint4* __restrict__ tab, uint32_t rows,
                                                  uint32_t row16, uint32_t iters, uint32_t* sink) {
    const uint32_t gid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t half = gid >> 4, q = threadIdx.x & 15;
    uint32_t acc = 0;
    for (uint32_t it = 0; it < iters; ++it) {
        uint4 v[UN];
#pragma unroll
        for (int k = 0; k < UN; ++k) {
            const uint32_t h = hash32(half * 0x9E3779B1u + it * UN + k);
            const uint32_t r = (uint32_t)(((uint64_t)h * rows) >> 32);
            v[k] = __ldg(tab + (size_t)r * row16 + q);
        }
#pragma unroll
        for (int k = 0; k < UN; ++k) acc ^= v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
    }
    if (acc == 0x7fffu && gid == 0u) sink[0] = acc;
}

template <int S>
__global__ void __launch_bounds__(128) k_g4_wide(const __grid_constant__ CUtensorMap tm, uint32_t rows,
                                                 uint32_t iters, uint32_t* sink) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) unsigned long long mb[4][S];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t gid = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned char* buf = sm + (size_t)w * S * 8192;
    if (lane == 0)
        for (int s = 0; s < S; ++s) mbar_init(smem_u32(&mb[w][s]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    uint32_t acc = 0;
    auto issue = [&](uint32_t it, int s) {
        const uint32_t mbar = smem_u32(&mb[w][s]);
        if (lane == 0) mbar_expect_tx(mbar, 8192);
        __syncwarp();
        if (lane < 8) {
            uint32_t r[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t h = hash32(gid * 0x9E3779B1u + it * 4 + k);
                r[k] = (uint32_t)(((uint64_t)h * rows) >> 32);
            }
            g4(smem_u32(buf + s * 8192 + lane * 1024), &tm, mbar, 0, r[0], r[1], r[2], r[3]);
        }
    };
#pragma unroll
    for (int s = 0; s < S; ++s) issue(s, s);
    uint32_t ph = 0;
    for (uint32_t it = 0; it < iters; ++it) {
#pragma unroll
        for (int s = 0; s < S; ++s) {
            mbar_wait(smem_u32(&mb[w][s]), ph);
            const uint4* st = reinterpret_cast<const uint4*>(buf + s * 8192);
#pragma unroll 4
            for (int k = 0; k < 16; ++k) {
                const uint4 v = st[k * 32 + lane];
                acc ^= v.x ^ v.y ^ v.z ^ v.w;
            }
            __syncwarp();
            issue((it + 1) * S + s, s);
        }
        ph ^= 1u;
    }
#pragma unroll
    for (int s = 0; s < S; ++s) mbar_wait(smem_u32(&mb[w][s]), ph);
    if (acc == 0x7fffu && gid == 0u) sink[0] = acc;
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
        return nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

template <class F>
static double time_ms(F launch, int reps = 5) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
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

static int wide(int sms, int clk, PFN_cuTensorMapEncodeTiled_v12000 encode, uint32_t* sink) {
    const uint32_t rows = 70000, row_bytes = 800;
    unsigned char* tab;
    CK(cudaMalloc(&tab, (size_t)rows * row_bytes));
    CK(cudaMemset(tab, 0x5a, (size_t)rows * row_bytes));
    CUtensorMap tm;
    cuuint64_t gdim[2] = {row_bytes, rows};
    cuuint64_t gstr[1] = {row_bytes};
    cuuint32_t box[2] = {256, 1};
    cuuint32_t es[2] = {1, 1};
    if (encode(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, tab, gdim, gstr, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        fprintf(stderr, "encode (wide) failed\n");
        return 1;
    }
    for (int bpsm : {2, 4, 8}) {
        const int grid = sms * bpsm;
        const uint32_t it = 64;
        double ms = time_ms([&] { k_ldg_wide<4><<<grid, 256>>>(reinterpret_cast<const uint4*>(tab), rows, row_bytes / 16, it, sink); });
        CK(cudaGetLastError());
        double rps = (double)grid * 16 * it * 4 / (ms * 1e-3);
        printf("{\"case\": \"ldg_wide256\", \"table_mb\": 56, \"bpsm\": %d, \"rows_per_s\": %.4g, \"per_sm_cycle\": %.3f}\n",
               bpsm, rps, rps / (sms * (clk * 1e3)));
        for (int S : {1, 2}) {
            const size_t smem = (size_t)4 * S * 8192;
            const int g2 = sms * bpsm * 2;
            if (S == 1) {
                cudaFuncSetAttribute(k_g4_wide<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                ms = time_ms([&] { k_g4_wide<1><<<g2, 128, smem>>>(tm, rows, it, sink); });
            } else {
                cudaFuncSetAttribute(k_g4_wide<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                ms = time_ms([&] { k_g4_wide<2><<<g2, 128, smem>>>(tm, rows, it, sink); });
            }
            CK(cudaGetLastError());
            rps = (double)g2 * 4 * 32 * it * S / (ms * 1e-3);
            printf("{\"case\": \"tma_gather4_wide256\", \"table_mb\": 56, \"bpsm\": %d, \"stages\": %d, \"rows_per_s\": %.4g, \"per_sm_cycle\": %.3f}\n",
                   bpsm * 2, S, rps, rps / (sms * (clk * 1e3)));
            fflush(stdout);
        }
    }
    cudaFree(tab);
    return 0;
}

template <int S, int UN>
static int run_mix(const CUtensorMap& tm, const uint16_t* tab, uint32_t rows16, int sms, int clk,
                   unsigned long long mb, uint32_t* sink) {
    for (int bpsm : {2, 4, 8}) {
        const int grid = sms * bpsm;
        const double threads = (double)grid * 256;
        const size_t smem = (size_t)8 * S * 4096;
        const uint32_t it = 64;
        cudaFuncSetAttribute(k_mix<S, UN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        double ms = time_ms([&] { k_mix<S, UN><<<grid, 256, smem>>>(tm, tab, rows16, it, sink); });
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) {
            printf("{\"case\": \"mix\", \"error\": \"%s\"}\n", cudaGetErrorString(e));
            return 1;
        }
        const double rps = threads * (double)it * S * (4.0 + UN) / (ms * 1e-3);
        printf("{\"case\": \"mix_g4_ldg\", \"table_mb\": %llu, \"bpsm\": %d, \"stages\": %d, \"ldg_per_stage\": %d, \"rows_per_s\": %.4g, \"per_sm_cycle\": %.3f}\n",
               mb, bpsm, S, UN, rps, rps / (sms * (clk * 1e3)));
        fflush(stdout);
    }
    return 0;
}

int main(int argc, char** argv) {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    auto encode = get_encode();
    if (!encode) {
        fprintf(stderr, "no cuTensorMapEncodeTiled\n");
        return 1;
    }
    uint32_t* sink;
    CK(cudaMalloc(&sink, 4));
    if (argc > 1 && argv[1][0] == 'w') return wide(sms, clk, encode, sink);
    const bool mixed = argc > 1 && argv[1][0] == 'm';
    for (uint64_t mb : {2ull, 40ull, 80ull, 400ull}) {
        const uint64_t heads = mb * 1000000ull / 2;  // u16 heads
        const uint32_t rows16 = (uint32_t)(heads / 8);
        uint16_t* tab;
        CK(cudaMalloc(&tab, rows16 * 16ull));
        CK(cudaMemset(tab, 0x5a, rows16 * 16ull));
        CUtensorMap tm;
        cuuint64_t gdim[2] = {8, rows16};
        cuuint64_t gstr[1] = {16};
        cuuint32_t box[2] = {8, 1};
        cuuint32_t es[2] = {1, 1};
        CUresult cr = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, tab, gdim, gstr, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (cr != CUDA_SUCCESS) {
            fprintf(stderr, "encode failed %d\n", (int)cr);
            return 1;
        }
        if (mixed) {
            if (run_mix<2, 4>(tm, tab, rows16, sms, clk, mb, sink)) return 1;
            if (run_mix<2, 8>(tm, tab, rows16, sms, clk, mb, sink)) return 1;
            if (run_mix<2, 16>(tm, tab, rows16, sms, clk, mb, sink)) return 1;
            if (run_mix<4, 4>(tm, tab, rows16, sms, clk, mb, sink)) return 1;
            if (run_mix<4, 8>(tm, tab, rows16, sms, clk, mb, sink)) return 1;
            CK(cudaFree(tab));
            continue;
        }
        for (int bpsm : {2, 4, 8}) {
            const int grid = sms * bpsm;
            const uint64_t threads = (uint64_t)grid * 256;
            {
                const uint32_t it = 256;
                double ms = time_ms([&] { k_ldg<8><<<grid, 256>>>(tab, rows16 * 8, it, sink); });
                CK(cudaGetLastError());
                const double rps = threads * it * 8.0 / (ms * 1e-3);
                printf("{\"case\": \"ldg_u16\", \"table_mb\": %llu, \"bpsm\": %d, \"rows_per_s\": %.4g, \"per_sm_cycle\": %.3f}\n",
                       (unsigned long long)mb, bpsm, rps, rps / (sms * (clk * 1e3)));
            }
            for (int S : {2, 4}) {
                const size_t smem = (size_t)8 * S * 4096;
                const uint32_t it = 64;
                double ms;
                if (S == 2) {
                    cudaFuncSetAttribute(k_g4<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                    ms = time_ms([&] { k_g4<2><<<grid, 256, smem>>>(tm, rows16, it, sink); });
                } else {
                    cudaFuncSetAttribute(k_g4<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                    ms = time_ms([&] { k_g4<4><<<grid, 256, smem>>>(tm, rows16, it, sink); });
                }
                cudaError_t e = cudaGetLastError();
                if (e != cudaSuccess) {
                    printf("{\"case\": \"g4\", \"S\": %d, \"bpsm\": %d, \"error\": \"%s\"}\n", S, bpsm,
                           cudaGetErrorString(e));
                    return 1;
                }
                const double rps = threads * (double)it * S * 4.0 / (ms * 1e-3);
                printf("{\"case\": \"tma_gather4\", \"table_mb\": %llu, \"bpsm\": %d, \"stages\": %d, \"rows_per_s\": %.4g, \"per_sm_cycle\": %.3f}\n",
                       (unsigned long long)mb, bpsm, S, rps, rps / (sms * (clk * 1e3)));
                if (S == 2) {
                    cudaFuncSetAttribute(k_bulk<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                    ms = time_ms([&] { k_bulk<2><<<grid, 256, smem>>>(tab, rows16, it, sink); });
                } else {
                    cudaFuncSetAttribute(k_bulk<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                    ms = time_ms([&] { k_bulk<4><<<grid, 256, smem>>>(tab, rows16, it, sink); });
                }
                CK(cudaGetLastError());
                const double rps2 = threads * (double)it * S * 4.0 / (ms * 1e-3);
                printf("{\"case\": \"bulk16\", \"table_mb\": %llu, \"bpsm\": %d, \"stages\": %d, \"rows_per_s\": %.4g, \"per_sm_cycle\": %.3f}\n",
                       (unsigned long long)mb, bpsm, S, rps2, rps2 / (sms * (clk * 1e3)));
                fflush(stdout);
            }
        }
        cudaFree(tab);
    }
    return 0;
}
