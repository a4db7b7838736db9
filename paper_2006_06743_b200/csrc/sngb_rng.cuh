// sngb_rng.cuh -- device restatement of the reference's counter-based RNG.
//
// Bit-exact with proj/include/sng/rng.hpp:
//   mix                 rng.hpp:9-13   (SplitMix64 finalizer)
//   Stream key          rng.hpp:23-24  key = mix(seed + gamma) ^ mix(id * C1 + C2)
//   next()              rng.hpp:26     mix(key + (++counter) * gamma)
//   next_below(bound)   rng.hpp:35-48  Lemire multiply-reject
//
// Data-parallel form: while no Lemire rejection has
// happened, draw i of a stream uses counter i+1, so every draw is computable
// independently.  `fire` flags the (necessary) pre-condition of a rejection,
// lo < bound; a vertex with any fired draw is resolved by the exact
// sequential path (sampler kernel), so the fast paths never need to know how
// many extra counters a rejection consumed.
#pragma once
#include <cstdint>

namespace sngb {

constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ULL;
constexpr uint64_t kIdMul = 0xda942042e4dd58b5ULL;
constexpr uint64_t kIdAdd = 0x8bb84b93962eacc9ULL;

// z * C mod 2^64.  On the device: one IMAD.WIDE and two IMADs chained through the
// high word (ptxas compiles the plain product to two parallel IMADs, an IMAD.WIDE
// and an add: one more instruction, and mix() is ~2/3 of every draw).
__host__ __device__ __forceinline__ uint64_t mul64c(uint64_t z, uint64_t C) {
#ifdef __CUDA_ARCH__
    const uint32_t zl = (uint32_t)z, zh = (uint32_t)(z >> 32);
    const uint32_t cl = (uint32_t)C, ch = (uint32_t)(C >> 32);
    uint64_t p, r;
    uint32_t lo, hi;
    asm("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(zl), "r"(cl));
    asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "l"(p));
    asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(hi) : "r"(zl), "r"(ch));
    asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(hi) : "r"(zh), "r"(cl));
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(lo), "r"(hi));
    return r;
#else
    return z * C;
#endif
}

__host__ __device__ __forceinline__ uint64_t mix(uint64_t z) {
    z = mul64c(z ^ (z >> 30), 0xbf58476d1ce4e5b9ULL);
    z = mul64c(z ^ (z >> 27), 0x94d049bb133111ebULL);
    return z ^ (z >> 31);
}

// mix(seed + gamma): the seed half of every vertex key, computed once on the host.
__host__ __device__ __forceinline__ uint64_t seed_part(uint64_t seed) { return mix(seed + kGamma); }

__host__ __device__ __forceinline__ uint64_t vertex_key(uint64_t seed_mixed, uint64_t u) {
    return seed_mixed ^ mix(u * kIdMul + kIdAdd);
}

// Output of the counter-th next() (counter >= 1) of a stream with `key`.
__device__ __forceinline__ uint64_t stream_at(uint64_t key, uint64_t counter) {
    return mix(key + counter * kGamma);
}

// Lemire step for a 32-bit bound: t = floor(x * b / 2^64); fire = (lo < b)
// where lo = x * b mod 2^64.  Two 32x32->64 products instead of a 64x64 high
// multiply (b < 2^32 because b <= n-1 and vertex ids are u32).
__device__ __forceinline__ uint32_t lemire32(uint64_t x, uint32_t b, bool& fire) {
    const uint64_t p1 = (uint64_t)(uint32_t)x * b;
    const uint64_t s = (uint64_t)(uint32_t)(x >> 32) * b + (p1 >> 32);
    // lo = (s << 32) | (uint32)p1  <  b  (< 2^32)  <=>  (uint32)s == 0 && (uint32)p1 < b
    fire = ((uint32_t)s == 0u) && ((uint32_t)p1 < b);
    return (uint32_t)(s >> 32);
}

// Same, returning the low word of s instead of the pre-condition: a draw can
// fire only if slo == 0, so a running minimum of slo over many draws is a one-
// instruction superset test (the exact test is redone on the rare hit).
__device__ __forceinline__ uint32_t lemire32_slo(uint64_t x, uint32_t b, uint32_t& slo) {
    const uint64_t p1 = (uint64_t)(uint32_t)x * b;
    const uint64_t s = (uint64_t)(uint32_t)(x >> 32) * b + (p1 >> 32);
    slo = (uint32_t)s;
    return (uint32_t)(s >> 32);
}

// Exact sequential Stream (rng.hpp:21-48) for the rare irregular vertices.
struct SeqStream {
    uint64_t key;
    uint64_t counter;
    __device__ __forceinline__ uint64_t next() { return mix(key + (++counter) * kGamma); }
    __device__ uint64_t next_below(uint64_t bound) {
        uint64_t x = next();
        uint64_t hi = __umul64hi(x, bound);
        uint64_t lo = x * bound;
        if (lo < bound) {
            const uint64_t threshold = (0 - bound) % bound;
            while (lo < threshold) {
                x = next();
                hi = __umul64hi(x, bound);
                lo = x * bound;
            }
        }
        return hi;
    }
};

}  // namespace sngb
