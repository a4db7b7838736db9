// sngb_cluster.cu -- symmetrise/dedup, degrees, core mask, union-find,
// border attachment and canonical relabelling on the device.
//
// Reference being replaced:
//   csr_from_pairs / SampledGraph::from_edges   graph.cpp:34-40, 67-102
//   core mask                                   clusterer.cpp:12-13
//   connected_components + UnionFind            graph.cpp:222-247, union_find.hpp
//   core / border / noise                       clusterer.cpp:17-39
//   relabel by smallest member                  clusterer.cpp:41-51
//
// Order-equivalences that make the edge-centric GPU form exact:
//   * Union-find always hooks the larger root under the smaller one, so every
//     component's final root is its smallest core vertex.  The reference
//     numbers components by first appearance of the root in vertex order,
//     i.e. by smallest member -- the same order as our roots.
//   * "smallest component id over core neighbours" (clusterer.cpp:31-35) is
//     therefore "smallest root", an atomicMin over incident core edges.
//   * relabel by smallest member: first[r] = atomicMin over members; the
//     vertices that are some cluster's first member, in vertex order, are the
//     clusters in the reference's final order -> exclusive scan of flags.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "sngb_internal.cuh"

namespace sngb {

namespace {

constexpr uint32_t kNone = 0xffffffffu;

__device__ __forceinline__ void decode(unsigned long long k, uint32_t nb, uint32_t& a, uint32_t& b) {
    a = (uint32_t)(k >> nb);
    b = (uint32_t)(k & ((1ull << nb) - 1));
}

// Edge-centric kernels read the edge count from the device (m_ptr: the
// DeviceSelect output, no host round trip) or, when m_ptr is null, take m_host.
// Sorted keys come in runs of equal smaller endpoint a (~E/n long), so the
// edge kernels give each thread kRun consecutive keys: one atomic per run of a
// for the degree, and union-find keeps a's root across the run.
constexpr int kRun = 8;

// rstart (optional): the index of each vertex's first key (the start of its
// run), for the vertex-parallel Afforest rounds of k_union_nth.
__global__ void k_degrees(const unsigned long long* __restrict__ keys, const unsigned long long* m_ptr,
                          uint64_t m_host, uint32_t nb, uint32_t* deg, uint32_t* rstart = nullptr) {
    const uint64_t m = m_ptr ? *m_ptr : m_host;
    for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c * kRun < m;
         c += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t e1 = (c + 1) * kRun < m ? (c + 1) * kRun : m;
        uint32_t run_a = 0xffffffffu, run = 0;
        if (rstart && c > 0) run_a = (uint32_t)(keys[c * kRun - 1] >> nb);  // previous key's a
        for (uint64_t e = c * kRun; e < e1; ++e) {
            uint32_t a, b;
            decode(keys[e], nb, a, b);
            if (a != run_a) {
                if (run) atomicAdd(&deg[run_a], run);
                if (rstart) rstart[a] = (uint32_t)e;  // a run starts here
                run_a = a;
                run = 0;
            }
            ++run;
            atomicAdd(&deg[b], 1u);
        }
        if (run) atomicAdd(&deg[run_a], run);
    }
}

// core mask (clusterer.cpp:12-13) + union-find init + border init.
__global__ void k_init(const uint32_t* __restrict__ deg, uint64_t n, uint32_t min_pts, uint8_t* core,
                       uint32_t* parent, uint32_t* broot, uint32_t* first) {
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x) {
        core[v] = deg[v] >= min_pts ? 1 : 0;
        parent[v] = (uint32_t)v;
        broot[v] = kNone;
        first[v] = kNone;
    }
}

__device__ __forceinline__ uint32_t uf_find(uint32_t* parent, uint32_t x) {
    // pointer jumping with path halving; parent[x] <= x always, so the
    // benign races only ever shorten paths.
    uint32_t p = parent[x];
    while (p != x) {
        const uint32_t gp = parent[p];
        if (gp != p) parent[x] = gp;
        x = p;
        p = gp;
    }
    return x;
}

// union over core-core edges (graph.cpp:228-235): hook larger root under smaller.
__global__ void k_union(const unsigned long long* __restrict__ keys, const unsigned long long* m_ptr,
                        uint64_t m_host, uint32_t nb, const uint8_t* __restrict__ core,
                        uint32_t* parent) {
    const uint64_t m = m_ptr ? *m_ptr : m_host;
    for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c * kRun < m;
         c += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t e1 = (c + 1) * kRun < m ? (c + 1) * kRun : m;
        uint32_t run_a = 0xffffffffu, ra = 0;
        for (uint64_t e = c * kRun; e < e1; ++e) {
            uint32_t a, b;
            decode(keys[e], nb, a, b);
            if (!core[a] || !core[b]) continue;
            if (a != run_a) {
                run_a = a;
                ra = uf_find(parent, a);
            }
            if (parent[b] == ra) continue;  // b already hangs off a's root
            for (;;) {
                // ra is in a's tree; walk up if another thread hooked it meanwhile
                for (uint32_t p = parent[ra]; p != ra; p = parent[ra]) ra = p;
                const uint32_t rb = uf_find(parent, b);
                if (ra == rb) break;
                const uint32_t lo = ra < rb ? ra : rb, hi = ra < rb ? rb : ra;
                if (atomicCAS(&parent[hi], hi, lo) == hi) {
                    ra = lo;  // the merged root (a's side may just have been hooked)
                    break;
                }
            }
        }
    }
}

// Afforest-style first round: union each vertex with the first neighbour of its
// run of keys only (one edge per vertex), so that after a compression most
// core vertices already point at their component's root and the full pass can
// dismiss an edge with two loads (parent[a] == parent[b]) instead of two finds.
__global__ void k_union_first(const unsigned long long* __restrict__ keys,
                              const unsigned long long* m_ptr, uint64_t m_host, uint32_t nb,
                              const uint8_t* __restrict__ core, uint32_t* parent, uint32_t nth) {
    const uint64_t m = m_ptr ? *m_ptr : m_host;
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
         e += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t a, b;
        decode(keys[e], nb, a, b);
        // only the nth key of a run (Afforest round nth: each vertex's nth neighbour)
        if (e < nth || (uint32_t)(keys[e - nth] >> nb) != a) continue;
        if (e > nth && (uint32_t)(keys[e - nth - 1] >> nb) == a) continue;
        if (!core[a] || !core[b]) continue;
        for (;;) {
            const uint32_t ra = uf_find(parent, a), rb = uf_find(parent, b);
            if (ra == rb) break;
            const uint32_t lo = ra < rb ? ra : rb, hi = ra < rb ? rb : ra;
            if (atomicCAS(&parent[hi], hi, lo) == hi) break;
        }
    }
}

// The same Afforest round, vertex-parallel: vertex v's nth neighbour is the key
// at rstart[v] + nth when it still belongs to v's run (n threads instead of m).
__global__ void k_union_nth(const unsigned long long* __restrict__ keys,
                            const unsigned long long* m_ptr, uint64_t n, uint32_t nb,
                            const uint32_t* __restrict__ rstart, const uint8_t* __restrict__ core,
                            uint32_t* parent, uint32_t nth) {
    const uint64_t m = *m_ptr;
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t s0 = rstart[v];
        if (s0 == 0xffffffffu || !core[v]) continue;
        const uint64_t e = (uint64_t)s0 + nth;
        if (e >= m) continue;
        uint32_t a, b;
        decode(keys[e], nb, a, b);
        if (a != (uint32_t)v || !core[b]) continue;
        for (;;) {
            const uint32_t ra = uf_find(parent, a), rb = uf_find(parent, b);
            if (ra == rb) break;
            const uint32_t lo = ra < rb ? ra : rb, hi = ra < rb ? rb : ra;
            if (atomicCAS(&parent[hi], hi, lo) == hi) break;
        }
    }
}

__global__ void k_compress(uint64_t n, const uint8_t* __restrict__ core, uint32_t* parent) {
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x) {
        if (!core[v]) continue;
        uint32_t r = (uint32_t)v;
        while (parent[r] != r) r = parent[r];
        parent[v] = r;
    }
}

// border: non-core endpoint adjacent to a core vertex takes the minimum root.
__global__ void k_border(const unsigned long long* __restrict__ keys, const unsigned long long* m_ptr,
                         uint64_t m_host, uint32_t nb, const uint8_t* __restrict__ core,
                         const uint32_t* __restrict__ parent, uint32_t* broot) {
    const uint64_t m = m_ptr ? *m_ptr : m_host;
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
         e += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t a, b;
        decode(keys[e], nb, a, b);
        const bool ca = core[a], cb = core[b];
        if (ca && !cb) atomicMin(&broot[b], parent[a]);
        else if (cb && !ca) atomicMin(&broot[a], parent[b]);
    }
}

__device__ __forceinline__ uint32_t cluster_root(uint64_t v, const uint8_t* core,
                                                 const uint32_t* parent, const uint32_t* broot) {
    return core[v] ? parent[v] : broot[v];
}

// first member of each cluster (clusterer.cpp:41-51: clusters are numbered by
// their smallest member).  A component's root is its smallest core vertex
// (hooking keeps parent[v] <= v), so among core members only the root itself
// is a candidate: core non-roots skip the atomic (cfg2: all 70 k vertices are
// core and hammered 10 addresses before), border vertices compete with it.
__global__ void k_first(uint64_t n, const uint8_t* __restrict__ core,
                        const uint32_t* __restrict__ parent, const uint32_t* __restrict__ broot,
                        uint32_t* first) {
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x) {
        if (core[v]) {
            if (parent[v] == (uint32_t)v) atomicMin(&first[v], (uint32_t)v);
        } else {
            // first[r] only decreases, so a (possibly stale) value <= v means the atomic
            // could not change it: on cfg5 a cluster's hundreds of thousands of border
            // vertices otherwise queue on one address (k_first 1.4 ms)
            const uint32_t r = broot[v];
            if (r != kNone && *(volatile uint32_t*)&first[r] > (uint32_t)v)
                atomicMin(&first[r], (uint32_t)v);
        }
    }
}

__global__ void k_flags(uint64_t n, const uint8_t* __restrict__ core,
                        const uint32_t* __restrict__ parent, const uint32_t* __restrict__ broot,
                        const uint32_t* __restrict__ first, uint32_t* flags) {
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v <= n;
         v += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t f = 0;
        if (v < n) {
            const uint32_t r = cluster_root(v, core, parent, broot);
            f = (r != kNone && first[r] == (uint32_t)v) ? 1u : 0u;
        }
        flags[v] = f;
    }
}

__global__ void k_labels(uint64_t n, const uint8_t* __restrict__ core,
                         const uint32_t* __restrict__ parent, const uint32_t* __restrict__ broot,
                         const uint32_t* __restrict__ first, const uint32_t* __restrict__ rank,
                         int32_t* labels, uint8_t* roles, unsigned long long* counters) {
    unsigned nc = 0, nbd = 0, nn = 0;
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x) {
        const bool c = core[v];
        const uint32_t r = c ? parent[v] : broot[v];
        if (r == kNone) {
            labels[v] = -1;  // kNoiseLabel (dataset.hpp:13)
            roles[v] = 2;    // PointRole::Noise
            ++nn;
        } else {
            labels[v] = (int32_t)rank[first[r]];
            roles[v] = c ? 0 : 1;  // Core / Border
            if (c) ++nc; else ++nbd;
        }
    }
    nc = __reduce_add_sync(kFull, nc);
    nbd = __reduce_add_sync(kFull, nbd);
    nn = __reduce_add_sync(kFull, nn);
    if ((threadIdx.x & 31) == 0) {
        if (nc) atomicAdd(&counters[C_CORE], (unsigned long long)nc);
        if (nbd) atomicAdd(&counters[C_BORDER], (unsigned long long)nbd);
        if (nn) atomicAdd(&counters[C_NOISE], (unsigned long long)nn);
    }
}

__global__ void k_store_clusters(const uint32_t* rank, uint64_t n, unsigned long long* counters) {
    counters[C_CLUSTERS] = rank[n];
}

__global__ void k_convert(const unsigned long long* __restrict__ in, unsigned long long* out,
                          uint64_t m, uint32_t nb, bool to_compact, uint64_t n,
                          unsigned long long* counters) {
    const unsigned long long mask = (1ull << nb) - 1;
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const unsigned long long k = in[e];
        if (to_compact) {
            uint64_t a = k >> 32, b = k & 0xffffffffull;
            if (a > b) {
                const uint64_t t = a;
                a = b;
                b = t;
            }
            // self loops / out-of-range endpoints are rejected like graph.cpp:78-80
            if (a == b || b >= n) atomicAdd(&counters[C_BADKEY], 1ull);
            out[e] = (a << nb) | b;
        } else {
            out[e] = ((k >> nb) << 32) | (k & mask);
        }
    }
}

// ---------------------------------------------------------------------------
// Multi-GPU merge steps.  Every rank owns the canonical keys
// (a<<32 | b, a < b) whose smaller endpoint lies in its row shard; vertex
// arrays are full length, int32 on the caller side so NCCL can SUM / MIN-
// reduce them; "no core neighbour" in the border array is INT32_MAX.
// ---------------------------------------------------------------------------
constexpr uint32_t kNoneI32 = 0x7fffffffu;

__global__ void k_check_keys(const unsigned long long* __restrict__ keys, uint64_t m, uint64_t n,
                             unsigned long long* counters) {
    unsigned bad = 0;
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const unsigned long long k = keys[e];
        const uint64_t a = k >> 32, b = k & 0xffffffffull;
        bad += (a >= b || b >= n) ? 1u : 0u;
    }
    bad = __reduce_add_sync(kFull, bad);
    if ((threadIdx.x & 31) == 0 && bad) atomicAdd(&counters[C_BADKEY], (unsigned long long)bad);
}

__global__ void k_coremask(const uint32_t* __restrict__ deg, uint64_t n, uint32_t min_pts,
                           uint8_t* core) {
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x)
        core[v] = deg[v] >= min_pts ? 1 : 0;
}

__global__ void k_count_changed(uint64_t n, const uint32_t* __restrict__ now,
                                const uint32_t* __restrict__ before, unsigned long long* counters) {
    unsigned c = 0;
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x)
        c += now[v] != before[v] ? 1u : 0u;
    c = __reduce_add_sync(kFull, c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(&counters[C_CHANGED], (unsigned long long)c);
}

// relabel inputs from the merged arrays: core mask, border roots (INT32_MAX ->
// kNone), first-member init.
__global__ void k_import(const uint32_t* __restrict__ deg, const uint32_t* __restrict__ border,
                         uint64_t n, uint32_t min_pts, uint8_t* core, uint32_t* broot,
                         uint32_t* first) {
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x) {
        core[v] = deg[v] >= min_pts ? 1 : 0;
        const uint32_t r = border[v];
        broot[v] = r == kNoneI32 ? kNone : r;
        first[v] = kNone;
    }
}

// 32-bit sort keys for small n (n(n-1)/2 <= 2^32: n <= 92 682, cfg1 and cfg2):
// the canonical pair (a, b), a < b, as its upper-triangular index
//     k = T(a) + (b - a - 1),  T(a) = a*n - a(a+1)/2,
// which sorts exactly like (a << nb) | b, so the radix sort moves half the
// bytes with one pass fewer (cfg2: 32 bits instead of 34 in u64 keys).
__global__ void k_to_tri(const unsigned long long* __restrict__ in, uint32_t* __restrict__ out,
                         uint64_t count, uint32_t nb, uint64_t n) {
    const unsigned long long mask = (1ull << nb) - 1;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const unsigned long long k = in[i];
        const uint64_t a = k >> nb, b = k & mask;
        out[i] = (uint32_t)(a * n - a * (a + 1) / 2 + (b - a - 1));
    }
}
__global__ void k_from_tri(const uint32_t* __restrict__ in, unsigned long long* __restrict__ out,
                           const unsigned long long* __restrict__ m_ptr, uint32_t nb, uint64_t n) {
    const uint64_t m = *m_ptr;
    const double c = 2.0 * (double)n - 1.0;
    auto T = [&](uint64_t a) { return a * n - a * (a + 1) / 2; };
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t k = in[i];
        // a = floor((c - sqrt(c^2 - 8k)) / 2), then exact integer fix-ups
        int64_t a = (int64_t)floor((c - sqrt(c * c - 8.0 * (double)k)) * 0.5);
        if (a < 0) a = 0;
        while (a > 0 && T((uint64_t)a) > k) --a;
        while ((uint64_t)a + 1 < n && T((uint64_t)a + 1) <= k) ++a;
        const uint64_t b = k - T((uint64_t)a) + (uint64_t)a + 1;
        out[i] = ((unsigned long long)a << nb) | b;
    }
}

unsigned grid_for(uint64_t items, int num_sms) {
    uint64_t b = (items + 255) / 256;
    const uint64_t cap = (uint64_t)num_sms * 8;
    if (b > cap) b = cap;
    return (unsigned)(b ? b : 1);
}

}  // namespace

size_t sort_unique_temp_bytes(uint64_t count, uint32_t nb) {
    size_t a = 0, b = 0, a32 = 0, b32 = 0;
    cub::DoubleBuffer<unsigned long long> db(nullptr, nullptr);
    cub::DeviceRadixSort::SortKeys(nullptr, a, db, (int64_t)count, 0, (int)(2 * nb));
    cub::DeviceSelect::Unique(nullptr, b, (unsigned long long*)nullptr,
                              (unsigned long long*)nullptr, (unsigned long long*)nullptr,
                              (int64_t)count);
    cub::DoubleBuffer<uint32_t> d32(nullptr, nullptr);
    cub::DeviceRadixSort::SortKeys(nullptr, a32, d32, (int64_t)count, 0, 32);
    cub::DeviceSelect::Unique(nullptr, b32, (uint32_t*)nullptr, (uint32_t*)nullptr,
                              (unsigned long long*)nullptr, (int64_t)count);
    size_t m = a > b ? a : b;
    m = m > a32 ? m : a32;
    m = m > b32 ? m : b32;
    return m + 256;
}

size_t cluster_temp_bytes(uint64_t n) {
    size_t a = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, a, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (int64_t)(n + 1));
    return a + 256;
}

cudaError_t sort_unique(unsigned long long* keys, unsigned long long* alt, uint64_t count,
                        uint32_t nb, void* temp, size_t temp_bytes, unsigned long long* counters,
                        unsigned long long** unique_out, cudaStream_t s, uint64_t tri_n) {
    if (count == 0) {
        *unique_out = keys;
        return cudaMemsetAsync(&counters[C_UNIQUE], 0, sizeof(unsigned long long), s);
    }
    if (tri_n >= 2 && tri_n * (tri_n - 1) / 2 <= (1ull << 32)) {
        // 32-bit triangular keys: keys -> alt (two u32 halves), sort, unique, decode -> keys
        uint32_t* h0 = reinterpret_cast<uint32_t*>(alt);
        uint32_t* h1 = h0 + count;
        const unsigned g = grid_for(count, 148);
        k_to_tri<<<g, 256, 0, s>>>(keys, h0, count, nb, tri_n);
        const uint64_t kmax = tri_n * (tri_n - 1) / 2 - 1;
        int bits = 1;
        while (bits < 32 && (kmax >> bits) != 0) ++bits;
        cub::DoubleBuffer<uint32_t> d32(h0, h1);
        size_t tb = temp_bytes;
        cudaError_t e = cub::DeviceRadixSort::SortKeys(temp, tb, d32, (int64_t)count, 0, bits, s);
        if (e != cudaSuccess) return e;
        uint32_t* sorted = d32.Current();
        uint32_t* uq = (sorted == h0) ? h1 : h0;
        tb = temp_bytes;
        e = cub::DeviceSelect::Unique(temp, tb, sorted, uq, &counters[C_UNIQUE], (int64_t)count, s);
        if (e != cudaSuccess) return e;
        k_from_tri<<<g, 256, 0, s>>>(uq, keys, &counters[C_UNIQUE], nb, tri_n);
        note_launch(2, 2 + (bits + 7) / 8 + 2);
        *unique_out = keys;
        return cudaGetLastError();
    }
    cub::DoubleBuffer<unsigned long long> db(keys, alt);
    size_t tb = temp_bytes;
    cudaError_t e =
        cub::DeviceRadixSort::SortKeys(temp, tb, db, (int64_t)count, 0, (int)(2 * nb), s);
    if (e != cudaSuccess) return e;
    unsigned long long* sorted = db.Current();
    unsigned long long* out = (sorted == keys) ? alt : keys;
    tb = temp_bytes;
    e = cub::DeviceSelect::Unique(temp, tb, sorted, out, &counters[C_UNIQUE], (int64_t)count, s);
    // onesweep: 1 histogram + 1 exclusive-sum + ceil(bits/8) passes; select: init + sweep
    note_launch(0, 2 + (int)((2 * nb + 7) / 8) + 2);
    *unique_out = out;
    return e;
}

cudaError_t launch_convert_keys(const unsigned long long* in, unsigned long long* out, uint64_t m,
                                uint32_t nb, bool to_compact, uint64_t n,
                                unsigned long long* counters, cudaStream_t s, int num_sms) {
    if (m == 0) return cudaSuccess;
    k_convert<<<grid_for(m, num_sms), 256, 0, s>>>(in, out, m, nb, to_compact, n, counters);
    note_launch(1);
    return cudaGetLastError();
}

cudaError_t cluster_unique_edges(const unsigned long long* ukeys, const unsigned long long* m_ptr,
                                 uint64_t m, uint64_t n,
                                 uint32_t nb, int32_t min_pts, const ClusterBuffers& b,
                                 unsigned long long* counters, int32_t* labels, uint8_t* roles,
                                 cudaStream_t s, int num_sms) {
    cudaError_t e = cudaMemsetAsync(b.deg, 0, n * sizeof(uint32_t), s);
    if (e != cudaSuccess) return e;
    const unsigned ge = grid_for(m, num_sms), gn = grid_for(n + 1, num_sms);
    if (b.rstart && m) {
        e = cudaMemsetAsync(b.rstart, 0xff, n * sizeof(uint32_t), s);
        if (e != cudaSuccess) return e;
    }
    if (m) k_degrees<<<ge, 256, 0, s>>>(ukeys, m_ptr, 0, nb, b.deg, b.rstart);
    k_init<<<gn, 256, 0, s>>>(b.deg, n, (uint32_t)min_pts, b.core, b.parent, b.broot, b.first);
    if (m) {
        // Afforest-style sampling rounds, each vertex's first then second
        // neighbour (SNGB_AFFOREST_ROUNDS; measured 0/1/2/3 rounds: union +
        // compress 282/121/116/133 us on cfg2, 186/114/103/110 us on cfg1)
        static const int rounds = [] {
            const char* e = std::getenv("SNGB_AFFOREST_ROUNDS");
            return e ? std::max(0, std::atoi(e)) : 2;
        }();
        for (int r = 0; r < rounds; ++r) {
            if (b.rstart && m_ptr)
                k_union_nth<<<gn, 256, 0, s>>>(ukeys, m_ptr, n, nb, b.rstart, b.core, b.parent,
                                               (uint32_t)r);
            else
                k_union_first<<<ge, 256, 0, s>>>(ukeys, m_ptr, 0, nb, b.core, b.parent, (uint32_t)r);
            k_compress<<<gn, 256, 0, s>>>(n, b.core, b.parent);
        }
        k_union<<<ge, 256, 0, s>>>(ukeys, m_ptr, 0, nb, b.core, b.parent);
    }
    k_compress<<<gn, 256, 0, s>>>(n, b.core, b.parent);
    if (m) k_border<<<ge, 256, 0, s>>>(ukeys, m_ptr, 0, nb, b.core, b.parent, b.broot);
    k_first<<<gn, 256, 0, s>>>(n, b.core, b.parent, b.broot, b.first);
    k_flags<<<gn, 256, 0, s>>>(n, b.core, b.parent, b.broot, b.first, b.flags);
    size_t tb = b.temp_bytes;
    e = cub::DeviceScan::ExclusiveSum(b.temp, tb, b.flags, b.rank, (int64_t)(n + 1), s);
    if (e != cudaSuccess) return e;
    k_labels<<<gn, 256, 0, s>>>(n, b.core, b.parent, b.broot, b.first, b.rank, labels, roles,
                                counters);
    k_store_clusters<<<1, 1, 0, s>>>(b.rank, n, counters);
    note_launch(m ? 11 : 6, 2);  // + CUB scan (init + sweep)
    return cudaGetLastError();
}

cudaError_t merge_check_keys(const unsigned long long* keys, uint64_t m, uint64_t n,
                             unsigned long long* counters, cudaStream_t s, int num_sms) {
    if (m == 0) return cudaSuccess;
    k_check_keys<<<grid_for(m, num_sms), 256, 0, s>>>(keys, m, n, counters);
    note_launch(1);
    return cudaGetLastError();
}

cudaError_t merge_degrees(const unsigned long long* keys, uint64_t m, uint32_t* deg, cudaStream_t s,
                          int num_sms) {
    if (m == 0) return cudaSuccess;
    k_degrees<<<grid_for(m, num_sms), 256, 0, s>>>(keys, nullptr, m, 32, deg);
    note_launch(1);
    return cudaGetLastError();
}

cudaError_t merge_components(const unsigned long long* keys, uint64_t m, uint64_t n,
                             const uint32_t* deg, int32_t min_pts, uint32_t* parent, uint8_t* core,
                             uint32_t* before, unsigned long long* counters, cudaStream_t s,
                             int num_sms) {
    const unsigned gn = grid_for(n, num_sms);
    k_coremask<<<gn, 256, 0, s>>>(deg, n, (uint32_t)min_pts, core);
    cudaError_t e = cudaMemcpyAsync(before, parent, n * 4, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return e;
    if (m) k_union<<<grid_for(m, num_sms), 256, 0, s>>>(keys, nullptr, m, 32, core, parent);
    k_compress<<<gn, 256, 0, s>>>(n, core, parent);
    k_count_changed<<<gn, 256, 0, s>>>(n, parent, before, counters);
    note_launch(m ? 4 : 3);
    return cudaGetLastError();
}

cudaError_t merge_border(const unsigned long long* keys, uint64_t m, uint64_t n, const uint32_t* deg,
                         int32_t min_pts, const uint32_t* parent, uint32_t* border, uint8_t* core,
                         cudaStream_t s, int num_sms) {
    k_coremask<<<grid_for(n, num_sms), 256, 0, s>>>(deg, n, (uint32_t)min_pts, core);
    if (m) k_border<<<grid_for(m, num_sms), 256, 0, s>>>(keys, nullptr, m, 32, core, parent, border);
    note_launch(m ? 2 : 1);
    return cudaGetLastError();
}

cudaError_t merge_relabel(uint64_t n, const uint32_t* deg, int32_t min_pts, const uint32_t* parent,
                          const uint32_t* border, const ClusterBuffers& b,
                          unsigned long long* counters, int32_t* labels, uint8_t* roles,
                          cudaStream_t s, int num_sms) {
    const unsigned gn = grid_for(n + 1, num_sms);
    k_import<<<gn, 256, 0, s>>>(deg, border, n, (uint32_t)min_pts, b.core, b.broot, b.first);
    k_first<<<gn, 256, 0, s>>>(n, b.core, parent, b.broot, b.first);
    k_flags<<<gn, 256, 0, s>>>(n, b.core, parent, b.broot, b.first, b.flags);
    size_t tb = b.temp_bytes;
    cudaError_t e = cub::DeviceScan::ExclusiveSum(b.temp, tb, b.flags, b.rank, (int64_t)(n + 1), s);
    if (e != cudaSuccess) return e;
    k_labels<<<gn, 256, 0, s>>>(n, b.core, parent, b.broot, b.first, b.rank, labels, roles,
                                counters);
    k_store_clusters<<<1, 1, 0, s>>>(b.rank, n, counters);
    note_launch(5, 2);
    return cudaGetLastError();
}

}  // namespace sngb
