// sngb_device.cuh -- warp-level helpers shared by the kernels.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "sngb_internal.cuh"

namespace sngb {

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

// Per-warp shared-memory staging of 64-bit records with batched flushes
// (one global atomic per flush instead of one per record).
template <int STAGE>
struct WarpStage {
    unsigned long long* buf;
    int count;

    __device__ __forceinline__ void flush(const EdgeSink& s, int lane) {
        __syncwarp();
        if (count == 0) return;
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(s.cursor, (unsigned long long)count);
        base = __shfl_sync(kFull, base, 0);
        for (int j = lane; j < count; j += 32)
            if (base + j < s.capacity) s.keys[base + j] = buf[j];
        __syncwarp();
        count = 0;
    }

    __device__ __forceinline__ void push(bool has, unsigned long long rec, const EdgeSink& s,
                                         int lane) {
        const unsigned m = __ballot_sync(kFull, has);
        if (!m) return;
        if (has) buf[count + __popc(m & lanemask_lt())] = rec;
        count += __popc(m);
        if (count > STAGE - 32) flush(s, lane);
    }
};

constexpr int kStage = 128;
constexpr int kWarpsPerBlock = 8;

__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}

}  // namespace sngb
