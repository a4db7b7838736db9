// sngb_multi.cu -- sng::sng_dbscan / dbscan_exact over several GPUs of ONE
// process (sngb_opts.num_gpus > 1; include/sngb.h ABI 4).
//
// The reference's only parallelism is parallel_over_vertices (graph.cpp:45-63):
// contiguous row chunks whose per-vertex work is independent.  Here the chunks
// are GPUs, one host thread per shard:
//
//   1. replica   shard r uploads rows [rb_r, re_r) from the caller's buffer over
//                its own PCIe link, then pulls every other shard from its peer
//                over NVLink (cudaMemcpyPeerAsync) -- the all-gather;
//   2. build     build_graph on rows [rb_r, re_r) against the whole replica: the
//                hot path, no communication (sorted unique canonical keys);
//   3. route     every key a<<32|b goes to the shard owning its smaller endpoint a
//                (keys are sorted: one contiguous run per destination, pulled by
//                the owner with a peer copy); a mutual draw split over two shards
//                meets its twin there and is deduplicated (graph.cpp:34-40);
//   4. degrees   per-shard incidence counts, SUM all-reduce -> sampled degree and
//                core mask everywhere (graph.hpp:28, clusterer.cpp:12-13);
//   5. union     local union-find over owned core-core keys (graph.cpp:222-235),
//                then MIN all-reduce of the parent array + local re-union until
//                no shard changes an entry: the forest rooted at each component's
//                smallest core vertex, on every shard;
//   6. border    atomicMin of neighbour roots, MIN all-reduce (clusterer.cpp:26-37);
//   7. relabel   on shard 0 (clusterer.cpp:41-51) -> labels, roles.
//
// The collectives are this file's own: each shard's reduce kernel reads every
// peer's int32[n] array directly over NVLink (P2P loads) after a cross-device
// event fence; key runs and shards move with peer copies.  Results are the
// single-GPU call's, bit for bit (tests/test_gpu_multi.py, incl. several shards
// on one GPU: a repeated ordinal in sngb_opts.devices).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "sngb.h"
#include "sngb_host.cuh"
#include "sngb_internal.cuh"

namespace sngb {
namespace host {

namespace {

constexpr int kMaxRanks = 16;

struct PeerArrays {
    const int32_t* p[kMaxRanks];
};

// dst[v] = reduce_q src_q[v] (op 0: sum, 1: min), int4 vectors + a scalar tail;
// the sources live on the peers (NVLink loads) or on this GPU
__global__ void k_allreduce_i32(int32_t* __restrict__ dst, const PeerArrays src, int w, uint64_t n,
                                int op) {
    const uint64_t n4 = n / 4;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
        int4 a = reinterpret_cast<const int4*>(src.p[0])[i];
        for (int q = 1; q < w; ++q) {
            const int4 b = reinterpret_cast<const int4*>(src.p[q])[i];
            if (op == 0) {
                a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
            } else {
                a.x = min(a.x, b.x); a.y = min(a.y, b.y); a.z = min(a.z, b.z); a.w = min(a.w, b.w);
            }
        }
        reinterpret_cast<int4*>(dst)[i] = a;
    }
    for (uint64_t v = n4 * 4 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride) {
        int32_t a = src.p[0][v];
        for (int q = 1; q < w; ++q) a = op == 0 ? a + src.p[q][v] : min(a, src.p[q][v]);
        dst[v] = a;
    }
}

__global__ void k_fill_i32(int32_t* __restrict__ p, uint64_t n, int32_t v, int iota) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        p[i] = iota ? (int32_t)i : v;
}

// cuts[q] = first index of a sorted key array whose key >= bounds[q] (lower_bound)
__global__ void k_cuts(const unsigned long long* __restrict__ keys, uint64_t m,
                       const unsigned long long* __restrict__ bounds, int nb,
                       unsigned long long* __restrict__ cuts) {
    const int q = threadIdx.x;
    if (q >= nb) return;
    const unsigned long long b = bounds[q];
    uint64_t lo = 0, hi = m;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) / 2;
        if (keys[mid] < b) lo = mid + 1;
        else hi = mid;
    }
    cuts[q] = lo;
}

unsigned grid_n(uint64_t n, int sms) {
    uint64_t b = (n + 1023) / 1024;
    b = std::min<uint64_t>(std::max<uint64_t>(b, 1), (uint64_t)sms * 8);
    return (unsigned)b;
}

// A host barrier that any shard can abort (a failing shard releases the others).
struct Barrier {
    std::mutex mu;
    std::condition_variable cv;
    int w = 0, count = 0;
    uint64_t gen = 0;
    bool aborted = false;
    bool wait() {
        std::unique_lock<std::mutex> lk(mu);
        if (aborted) return false;
        const uint64_t g = gen;
        if (++count == w) {
            count = 0;
            ++gen;
            cv.notify_all();
            return true;
        }
        cv.wait(lk, [&] { return gen != g || aborted; });
        return !aborted;
    }
    void abort() {
        std::lock_guard<std::mutex> lk(mu);
        aborted = true;
        cv.notify_all();
    }
};

struct Aborted {};

enum class Src { HostF32, HostF64, DevF32 };

struct Job {
    // problem
    Src src;
    const void* pts;  // host rows, or device rows on devs[0]
    uint64_t n;
    uint32_t d;
    double eps, rate;
    int32_t min_pts;
    uint64_t seed;
    int32_t metric;
    bool exact;
    // outputs: host (HostF*) or device on devs[0] (DevF32)
    int32_t* labels;
    uint8_t* roles;
    // shards
    int W = 0;
    std::vector<int> devs, slots;
    std::vector<DevCtx*> ctx;
    Barrier bar;
    std::vector<int> status;
    // per-shard buffers published to the peers
    std::vector<void*> replica;
    std::vector<unsigned long long*> keys64;
    std::vector<std::vector<uint64_t>> cuts;
    std::vector<int32_t*> deg, degsum, pa, pb, bord, bordred;
    std::vector<uint64_t> changed, owned;
    std::vector<sngb_info> part;  // each shard's build counters
    std::vector<uint64_t> launches, lib_launches;
    uint64_t routed = 0;
    uint32_t rounds = 0;
    unsigned long long relabel_hc[C_COUNT] = {};
    float ms_total = 0.f, ms_merge = 0.f;
    bool timing = false;
};

size_t elem_bytes(const Job& j) { return j.src == Src::HostF64 ? 8 : 4; }

uint64_t shard_lo(const Job& j, int r) {  // graph.cpp:52-56 chunking, by shard
    const uint64_t chunk = (j.n + j.W - 1) / j.W;
    return std::min<uint64_t>(j.n, (uint64_t)r * chunk);
}

// every shard's work enqueued so far is complete before shard r continues on its stream
void fence(Job& j, int r, cudaStream_t s) {
    DevCtx& c = *j.ctx[r];
    CK(cudaEventRecord(c.mg_ev, s));
    if (!j.bar.wait()) throw Aborted{};
    for (int q = 0; q < j.W; ++q)
        if (q != r) CK(cudaStreamWaitEvent(s, j.ctx[q]->mg_ev, 0));
    if (!j.bar.wait()) throw Aborted{};  // nobody re-records an event before all waits exist
}

void allreduce(Job& j, int r, cudaStream_t s, const std::vector<int32_t*>& src, int32_t* dst,
               int op) {
    fence(j, r, s);  // every source written
    PeerArrays pa{};
    for (int q = 0; q < j.W; ++q) pa.p[q] = src[q];
    k_allreduce_i32<<<grid_n(j.n, j.ctx[r]->num_sms), 256, 0, s>>>(dst, pa, j.W, j.n, op);
    note_launch(1);
    CK(cudaGetLastError());
    fence(j, r, s);  // every source read before anyone writes it again
}

void rank_main(Job& j, int r) {
    const int dev = j.devs[r];
    DeviceGuard dg(dev);
    DevCtx& c = *j.ctx[r];
    cudaStream_t s = c.stream;
    reset_launches();
    const uint64_t n = j.n;
    const uint32_t d = j.d;
    const size_t eb = elem_bytes(j);
    const uint64_t rb = shard_lo(j, r), re = shard_lo(j, r + 1);
    if (j.timing && r == 0) CK(cudaEventRecord(c.ev[E_START], s));

    // ---- 1. replica ----
    void* rep = nullptr;
    if (j.src == Src::DevF32 && r == 0) {
        rep = const_cast<void*>(j.pts);
    } else {
        Buf& b = eb == 8 ? c.upload64 : c.upload;
        b.ensure(n * d * eb);
        rep = b.p;
    }
    j.replica[r] = rep;
    if (j.src != Src::DevF32 && re > rb)
        CK(cudaMemcpyAsync(static_cast<char*>(rep) + rb * d * eb,
                           static_cast<const char*>(j.pts) + rb * d * eb, (re - rb) * d * eb,
                           cudaMemcpyHostToDevice, s));
    fence(j, r, s);
    if (j.src == Src::DevF32) {
        if (r != 0)
            CK(cudaMemcpyPeerAsync(rep, dev, j.replica[0], j.devs[0], n * d * eb, s));
    } else {
        for (int q = 0; q < j.W; ++q) {
            const uint64_t lo = shard_lo(j, q), hi = shard_lo(j, q + 1);
            if (q == r || hi <= lo) continue;
            CK(cudaMemcpyPeerAsync(static_cast<char*>(rep) + lo * d * eb, dev,
                                   static_cast<const char*>(j.replica[q]) + lo * d * eb, j.devs[q],
                                   (hi - lo) * d * eb, s));
        }
    }

    // ---- 2. build the edges of rows [rb, re) ----
    Timer tm{c, s, false};
    GraphResult gr;
    const double rate = j.exact ? 1.0 : j.rate;
    const int rc = build_graph(c, s, tm, eb == 4 ? static_cast<const float*>(rep) : nullptr, n, d,
                               j.eps, rate, j.seed, rb, re, gr, nullptr,
                               eb == 8 ? static_cast<const double*>(rep) : nullptr, j.metric,
                               j.exact);
    if (rc) {  // the same validation result on every shard (each checked the whole replica)
        j.status[r] = rc;
        throw Aborted{};
    }
    unsigned long long* dc = c.counters.as<unsigned long long>();
    fill_info(&j.part[r], c.h_counters, n, d, gr, re - rb, tm, false, false);
    uint64_t m = 0;
    CK(cudaMemcpyAsync(&c.h_counters[C_UNIQUE], &dc[C_UNIQUE], 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    m = c.h_counters[C_UNIQUE];
    if (j.timing && r == 0) CK(cudaEventRecord(c.ev[E_SORTED], s));
    // canonical a<<32|b keys, sorted (the compact order is the same order)
    c.mg_k64.ensure(std::max<uint64_t>(m, 1) * 8);
    unsigned long long* k64 = c.mg_k64.as<unsigned long long>();
    CK(launch_convert_keys(gr.ukeys, k64, m, gr.nb, false, n, dc, s, c.num_sms));
    j.keys64[r] = k64;

    // ---- 3. route keys to the owner of their smaller endpoint ----
    c.mg_cuts.ensure(2 * (kMaxRanks + 1) * 8);
    unsigned long long* bounds = c.mg_cuts.as<unsigned long long>();
    unsigned long long hb[kMaxRanks + 1];
    for (int q = 0; q <= j.W; ++q) hb[q] = (unsigned long long)shard_lo(j, q) << 32;
    hb[j.W] = ~0ull;
    CK(cudaMemcpyAsync(bounds, hb, (j.W + 1) * 8, cudaMemcpyHostToDevice, s));
    k_cuts<<<1, 32, 0, s>>>(k64, m, bounds, j.W + 1, bounds + kMaxRanks + 1);
    note_launch(1);
    CK(cudaGetLastError());
    unsigned long long hcut[kMaxRanks + 1];
    CK(cudaMemcpyAsync(hcut, bounds + kMaxRanks + 1, (j.W + 1) * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    j.cuts[r].assign(hcut, hcut + j.W + 1);
    fence(j, r, s);  // every shard's keys and cuts published
    uint64_t total = 0;
    for (int q = 0; q < j.W; ++q) total += j.cuts[q][r + 1] - j.cuts[q][r];
    c.mg_recv.ensure(std::max<uint64_t>(total, 1) * 8);
    unsigned long long* recv = c.mg_recv.as<unsigned long long>();
    uint64_t off = 0;
    for (int q = 0; q < j.W; ++q) {
        const uint64_t cnt = j.cuts[q][r + 1] - j.cuts[q][r];
        if (cnt)
            CK(cudaMemcpyPeerAsync(recv + off, dev, j.keys64[q] + j.cuts[q][r], j.devs[q], cnt * 8,
                                   s));
        off += cnt;
    }
    if (r == 0) {
        uint64_t moved = 0;
        for (int q = 0; q < j.W; ++q)
            for (int t = 0; t < j.W; ++t)
                if (t != q) moved += j.cuts[q][t + 1] - j.cuts[q][t];
        j.routed = moved;
    }
    fence(j, r, s);  // all runs pulled before any key buffer is reused

    // ---- unique owned keys (graph.cpp:34-40) ----
    const uint32_t nb = bits_for(n - 1);
    c.keys.ensure(std::max<uint64_t>(total, 1) * 8);
    c.keys_alt.ensure(std::max<uint64_t>(total, 1) * 8);
    CK(cudaMemsetAsync(&dc[C_UNIQUE], 0, 8, s));
    CK(launch_convert_keys(recv, c.keys.as<unsigned long long>(), total, nb, true, n, dc, s,
                           c.num_sms));
    c.temp.ensure(std::max(sort_unique_temp_bytes(std::max<uint64_t>(total, 1), nb),
                           cluster_temp_bytes(n)));
    unsigned long long* u = nullptr;
    CK(sort_unique(c.keys.as<unsigned long long>(), c.keys_alt.as<unsigned long long>(), total, nb,
                   c.temp.p, c.temp.bytes, dc, &u, s));
    CK(cudaMemcpyAsync(&c.h_counters[C_UNIQUE], &dc[C_UNIQUE], 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const uint64_t mo = total ? c.h_counters[C_UNIQUE] : 0;
    j.owned[r] = mo;
    c.mg_owned.ensure(std::max<uint64_t>(mo, 1) * 8);
    unsigned long long* owned = c.mg_owned.as<unsigned long long>();
    CK(launch_convert_keys(u, owned, mo, nb, false, n, dc, s, c.num_sms));

    // ---- 4. degrees: SUM all-reduce ----
    c.mg_deg.ensure(n * 4);
    c.mg_degsum.ensure(n * 4);
    c.mg_pa.ensure(n * 4);
    c.mg_pb.ensure(n * 4);
    c.mg_bord.ensure(n * 4);
    c.mg_bordred.ensure(n * 4);
    j.deg[r] = c.mg_deg.as<int32_t>();
    j.degsum[r] = c.mg_degsum.as<int32_t>();
    j.pa[r] = c.mg_pa.as<int32_t>();
    j.pb[r] = c.mg_pb.as<int32_t>();
    j.bord[r] = c.mg_bord.as<int32_t>();
    j.bordred[r] = c.mg_bordred.as<int32_t>();
    const unsigned gn = grid_n(n, c.num_sms);
    CK(cudaMemsetAsync(j.deg[r], 0, n * 4, s));
    CK(merge_degrees(owned, mo, reinterpret_cast<uint32_t*>(j.deg[r]), s, c.num_sms));
    allreduce(j, r, s, j.deg, j.degsum[r], 0);
    const uint32_t* degsum = reinterpret_cast<const uint32_t*>(j.degsum[r]);

    // ---- 5. union-find, merged to a fixed point by MIN all-reduces ----
    c.core.ensure(n);
    c.first.ensure(n * 4);
    k_fill_i32<<<gn, 256, 0, s>>>(j.pa[r], n, 0, 1);  // parent = identity
    note_launch(1);
    auto components = [&](int32_t* parent) -> uint64_t {
        CK(cudaMemsetAsync(&dc[C_CHANGED], 0, 8, s));
        CK(merge_components(owned, mo, n, degsum, j.min_pts, reinterpret_cast<uint32_t*>(parent),
                            c.core.as<uint8_t>(), c.first.as<uint32_t>(), dc, s, c.num_sms));
        CK(cudaMemcpyAsync(&c.h_counters[C_CHANGED], &dc[C_CHANGED], 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        return c.h_counters[C_CHANGED];
    };
    components(j.pa[r]);
    bool in_b = false;  // which of the two forests holds the current result
    uint32_t rounds = 0;
    for (;;) {
        const std::vector<int32_t*>& srcv = in_b ? j.pb : j.pa;
        int32_t* dst = in_b ? j.pa[r] : j.pb[r];
        allreduce(j, r, s, srcv, dst, 1);
        in_b = !in_b;
        j.changed[r] = components(dst);
        ++rounds;
        if (!j.bar.wait()) throw Aborted{};
        uint64_t ch = 0;
        for (int q = 0; q < j.W; ++q) ch += j.changed[q];
        if (!j.bar.wait()) throw Aborted{};  // everyone read the flags before the next round
        if (ch == 0) break;
        if (rounds >= 64) {
            detail() = "multi-GPU union-find merge did not converge in 64 rounds";
            throw CudaFail{cudaErrorUnknown};
        }
    }
    if (r == 0) j.rounds = rounds;
    int32_t* parent = in_b ? j.pb[r] : j.pa[r];

    // ---- 6. border roots: MIN all-reduce ----
    k_fill_i32<<<gn, 256, 0, s>>>(j.bord[r], n, INT_MAX, 0);
    note_launch(1);
    CK(merge_border(owned, mo, n, degsum, j.min_pts, reinterpret_cast<const uint32_t*>(parent),
                    reinterpret_cast<uint32_t*>(j.bord[r]), c.core.as<uint8_t>(), s, c.num_sms));
    allreduce(j, r, s, j.bord, j.bordred[r], 1);
    if (j.timing && r == 0) CK(cudaEventRecord(c.ev[E_CLUSTERED], s));

    // ---- 7. relabel on shard 0 ----
    if (r == 0) {
        ClusterBuffers b{};
        ensure_cluster_bufs(c, n, b);
        CK(cudaMemsetAsync(dc, 0, C_COUNT * 8, s));
        int32_t* lab = j.labels;
        uint8_t* rol = j.roles;
        if (j.src != Src::DevF32) {
            c.labels.ensure(n * 4);
            c.roles.ensure(n);
            lab = c.labels.as<int32_t>();
            rol = c.roles.as<uint8_t>();
        }
        CK(merge_relabel(n, degsum, j.min_pts, reinterpret_cast<const uint32_t*>(parent),
                         reinterpret_cast<const uint32_t*>(j.bordred[r]), b, dc, lab, rol, s,
                         c.num_sms));
        if (j.src != Src::DevF32) {
            CK(cudaMemcpyAsync(j.labels, lab, n * 4, cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(j.roles, rol, n, cudaMemcpyDeviceToHost, s));
        }
        CK(cudaMemcpyAsync(j.relabel_hc, dc, C_COUNT * 8, cudaMemcpyDeviceToHost, s));
        if (j.timing) CK(cudaEventRecord(c.ev[E_END], s));
        CK(cudaStreamSynchronize(s));
        if (j.timing) {
            cudaEventElapsedTime(&j.ms_total, c.ev[E_START], c.ev[E_END]);
            cudaEventElapsedTime(&j.ms_merge, c.ev[E_SORTED], c.ev[E_CLUSTERED]);
        }
    }
    j.launches[r] = hand_launches();
    j.lib_launches[r] = lib_launches();
    if (!j.bar.wait()) throw Aborted{};  // shard 0 done with every peer's arrays
}

std::mutex g_multi_mu;  // one multi-GPU call at a time (it holds several contexts)

}  // namespace

// Resolve opts -> the device list of a multi-GPU call; returns 0 for a
// single-GPU call (num_gpus 0 / 1, or -1 on a one-GPU host), -1 for bad options.
int multi_devices(const sngb_opts* o, std::vector<int>& devs) {
    if (!o || o->num_gpus == 0 || o->num_gpus == 1) return 0;
    const int avail = device_count();
    int w = o->num_gpus;
    if (w == -1) w = avail;
    if (w < 1 || w > kMaxRanks) return -1;
    if (w == 1 && !o->devices) return 0;
    devs.resize(w);
    for (int r = 0; r < w; ++r) {
        devs[r] = o->devices ? o->devices[r] : (o->device >= 0 ? o->device + r : r);
        if (devs[r] < 0 || devs[r] >= avail) return -1;
    }
    return w > 1 ? w : 0;
}

// The multi-GPU call; validation has been done by the entry point.
int multi_dbscan(const std::vector<int>& devs, int src_kind, const void* pts, uint64_t n,
                 uint32_t d, double eps, int32_t min_pts, double rate, uint64_t seed,
                 int32_t metric, bool exact, bool timing, int32_t* labels, uint8_t* roles,
                 sngb_info* info) {
    std::lock_guard<std::mutex> glk(g_multi_mu);
    Job j;
    j.src = static_cast<Src>(src_kind);
    j.pts = pts;
    j.n = n;
    j.d = d;
    j.eps = eps;
    j.rate = rate;
    j.min_pts = min_pts;
    j.seed = seed;
    j.metric = metric;
    j.exact = exact;
    j.labels = labels;
    j.roles = roles;
    j.timing = timing;
    j.W = (int)devs.size();
    j.devs = devs;
    j.bar.w = j.W;
    const int W = j.W;
    j.slots.resize(W);
    for (int r = 0; r < W; ++r) {  // a repeated ordinal takes the next context slot
        int k = 0;
        for (int q = 0; q < r; ++q) k += devs[q] == devs[r];
        if (k >= kMaxSlots) return SNGB_ERR_ARG;
        j.slots[r] = k;
    }
    // peer access between the distinct devices (NVLink / NVSwitch)
    for (int a : devs)
        for (int b : devs) {
            if (a == b) continue;
            int ok = 0;
            CK(cudaDeviceCanAccessPeer(&ok, a, b));
            if (!ok) {
                detail() = "multi-GPU call: devices " + std::to_string(a) + " and " +
                           std::to_string(b) + " have no peer access";
                return SNGB_ERR_CUDA;
            }
            DeviceGuard dg(a);
            const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
            else CK(e);
        }
    j.ctx.resize(W);
    std::vector<std::unique_lock<std::mutex>> locks;
    for (int r = 0; r < W; ++r) {
        DeviceGuard dg(devs[r]);
        j.ctx[r] = &get_ctx(devs[r], j.slots[r]);
        if (!j.ctx[r]->mg_ev) CK(cudaEventCreateWithFlags(&j.ctx[r]->mg_ev, cudaEventDisableTiming));
    }
    {  // lock the contexts in a fixed order (no lock-order inversion with other calls)
        std::vector<int> order(W);
        for (int r = 0; r < W; ++r) order[r] = r;
        std::sort(order.begin(), order.end(), [&](int x, int y) {
            return std::make_pair(devs[x], j.slots[x]) < std::make_pair(devs[y], j.slots[y]);
        });
        for (int r : order) locks.emplace_back(j.ctx[r]->mu);
    }
    j.status.assign(W, SNGB_OK);
    j.replica.assign(W, nullptr);
    j.keys64.assign(W, nullptr);
    j.cuts.assign(W, {});
    for (auto* v : {&j.deg, &j.degsum, &j.pa, &j.pb, &j.bord, &j.bordred}) v->assign(W, nullptr);
    j.changed.assign(W, 0);
    j.owned.assign(W, 0);
    j.part.assign(W, sngb_info{});
    j.launches.assign(W, 0);
    j.lib_launches.assign(W, 0);
    std::vector<std::string> details(W);
    auto body = [&](int r) {
        try {
            rank_main(j, r);
        } catch (const CudaFail&) {
            cudaGetLastError();
            j.status[r] = SNGB_ERR_CUDA;
            details[r] = detail();
            j.bar.abort();
        } catch (const Aborted&) {
            j.bar.abort();
        } catch (const std::bad_alloc&) {
            j.status[r] = SNGB_ERR_CUDA;
            details[r] = "host allocation failed";
            j.bar.abort();
        }
    };
    std::vector<std::thread> th;
    for (int r = 1; r < W; ++r) th.emplace_back(body, r);
    body(0);
    for (auto& t : th) t.join();
    for (int r = 0; r < W; ++r)
        if (j.status[r] != SNGB_OK) {
            if (j.status[r] == SNGB_ERR_CUDA) detail() = details[r];
            // a CUDA error may have left work in flight on the other shards
            for (int q = 0; q < W; ++q) {
                DeviceGuard dg(devs[q]);
                cudaStreamSynchronize(j.ctx[q]->stream);
                cudaGetLastError();
            }
            return j.status[r];
        }
    if (info) {
        std::memset(info, 0, sizeof(*info));
        uint64_t draws = exact ? n - 1 : draws_for(n, rate);
        info->draws = draws;
        info->distance_evals = exact ? n * (n - 1) / 2 : (draws >= n - 1 ? n * (n - 1) : n * draws);
        uint64_t edges = 0;
        for (int r = 0; r < W; ++r) edges += j.owned[r];
        info->edges = edges;
        info->graph_bytes = (n + 1) * 8 + 2 * edges * 4;
        for (const sngb_info& p : j.part) {
            info->collisions += p.collisions;
            info->irregular_vertices += p.irregular_vertices;
            info->pairs_evaluated += p.pairs_evaluated;
            info->band_rechecks += p.band_rechecks;
            info->band_1e6 += p.band_1e6;
            info->fp32_flips += p.fp32_flips;
            info->directed_accepts += p.directed_accepts;
            info->gather_pairs += p.gather_pairs;
            info->gather_bytes += p.gather_bytes;
        }
        info->filter_bits = j.part[0].filter_bits;
        info->head_bytes = j.part[0].head_bytes;
        info->cluster_count = (int32_t)j.relabel_hc[C_CLUSTERS];
        info->core_count = (uint32_t)j.relabel_hc[C_CORE];
        info->border_count = (uint32_t)j.relabel_hc[C_BORDER];
        info->noise_count = (uint32_t)j.relabel_hc[C_NOISE];
        for (int r = 0; r < W; ++r) {
            info->kernel_launches += j.launches[r];
            info->library_launches += j.lib_launches[r];
        }
        info->num_gpus = (uint32_t)W;
        info->merge_rounds = j.rounds;
        info->routed_keys = j.routed;
        info->ms_total = j.ms_total;
        info->ms_merge = j.ms_merge;
    }
    return SNGB_OK;
}

}  // namespace host
}  // namespace sngb
