// sngb_host.cuh -- host-side internals of libsngb shared by the C-ABI entry
// points (sngb_api.cu) and the single-process multi-GPU driver (sngb_multi.cu).
// Not part of the ABI.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "sngb.h"
#include "sngb_internal.cuh"

namespace sngb {
namespace host {

// thread-local detail of the last SNGB_ERR_CUDA (sngb_last_error_detail)
std::string& detail();

struct CudaFail {
    cudaError_t err;
};

#define CK(expr)                                                                      \
    do {                                                                              \
        cudaError_t _e = (expr);                                                      \
        if (_e != cudaSuccess) {                                                      \
            char _b[512];                                                             \
            snprintf(_b, sizeof(_b), "%s at %s:%d (%s)", cudaGetErrorString(_e),      \
                     __FILE__, __LINE__, #expr);                                      \
            detail() = _b;                                                            \
            throw CudaFail{_e};                                                       \
        }                                                                             \
    } while (0)

struct Buf {
    void* p = nullptr;
    size_t bytes = 0;
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
    void ensure(size_t want) {
        if (want == 0) want = 16;
        if (bytes >= want) return;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        CK(cudaMalloc(&p, want));
        bytes = want;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
};

struct DevCtx {
    int dev = 0;
    int num_sms = 148;
    uint64_t l2_bytes = 126ull << 20;
    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr;          // sampler runs here, concurrently with the gather
    cudaStream_t hi = nullptr;            // high-priority stream for the gather (SNGB_PRIO)
    cudaEvent_t hi_fork = nullptr, hi_join = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
    // host-buffer calls: the points are uploaded in row chunks on `copy`,
    // chunk k's arrival is up_ev[k]; compute starts on the first chunk
    static constexpr int kMaxChunks = 16;
    cudaStream_t copy = nullptr;
    cudaEvent_t up_start = nullptr;
    cudaEvent_t up_ev[kMaxChunks] = {};
    std::mutex mu;
    Buf pts, upload, keys, keys_alt, extras, scratch, counters, deg, core, parent, broot, first,
        flags, rank, temp, labels, roles, work, q8, upload64, rnorm, band, partners, poff, rstart,
        colstats, perm, tbuf, tflags;
    cudaEvent_t sh_g[2] = {}, sh_f[2] = {};  // shared draws: chunk gathered / chunk's Floyd pass done
    cudaEvent_t qev = nullptr;  // min/max of the points copied to the host (8-bit filter)
    cudaEvent_t pev = nullptr;  // bucketed partner lists ready (host-upload 8-bit schedule)
    unsigned long long* h_counters = nullptr;  // pinned mirror of the counter block
    double* h_colstats = nullptr;  // pinned: per-column sums (8-bit filter column order)
    uint32_t* h_perm = nullptr;    // pinned: that column order, uploaded per call
    cudaEvent_t ev[12] = {};
    uint64_t edge_hint = 0;  // last needed edge capacity for this context
    uint64_t band_hint = 0;  // last needed band-list capacity

    // multi-GPU shard buffers (sngb_multi.cu) and its cross-device fence event
    Buf mg_k64, mg_cuts, mg_recv, mg_owned, mg_deg, mg_degsum, mg_pa, mg_pb, mg_bord, mg_bordred;
    cudaEvent_t mg_ev = nullptr;

    void release() {
        for (Buf* b : {&mg_k64, &mg_cuts, &mg_recv, &mg_owned, &mg_deg, &mg_degsum, &mg_pa, &mg_pb,
                       &mg_bord, &mg_bordred})
            b->release();
        for (Buf* b : {&pts, &upload, &keys, &keys_alt, &extras, &scratch, &counters, &deg, &core,
                       &parent, &broot, &first, &flags, &rank, &temp, &labels, &roles, &work, &q8, &upload64, &rnorm, &band, &partners, &poff, &rstart, &colstats, &perm, &tbuf, &tflags})
            b->release();
    }
};

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) CK(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

int device_count();
// One context per (device, slot): slot 0 serves the single-problem calls,
// slots 1.. the concurrent workers of sngb_dbscan_batch_f32 and the extra
// shards a multi-GPU call places on a repeated device ordinal.
constexpr int kMaxSlots = 16;
DevCtx& get_ctx(int dev, int slot = 0);
uint64_t env_u64(const char* name, uint64_t dflt);
uint32_t bits_for(uint64_t x);
uint64_t draws_for(uint64_t n, double rate);
int32_t metric_of(const sngb_opts* o);
bool metric_flags_ok(const sngb_opts* o);
// std::invalid_argument checks in the reference's order; exact: dbscan_exact
// (clusterer.cpp:67-70 + graph.cpp:17-21, no rate)
int validate(uint64_t n, uint32_t d, double eps, int32_t min_pts, double rate, bool need_minpts);

struct Timer {
    DevCtx& c;
    cudaStream_t s;
    bool on;
    int next = 0;
    void mark(int i) {
        if (on) CK(cudaEventRecord(c.ev[i], s));
    }
    void mark_on(int i, cudaStream_t st) {
        if (on) CK(cudaEventRecord(c.ev[i], st));
    }
    bool side = false;  // the sampler ran on the side stream (E_SIDE0..E_SIDE1)
    float between(int a, int b) {
        if (!on) return 0.f;
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, c.ev[a], c.ev[b]) != cudaSuccess) {
            cudaGetLastError();
            return 0.f;
        }
        return ms;
    }
};

enum Ev { E_START = 0, E_UPLOADED, E_PREPARED, E_SAMPLED, E_GATHERED, E_EXTRAS, E_SORTED,
          E_CLUSTERED, E_DOWNLOADED, E_END, E_SIDE0, E_SIDE1 };

struct GraphResult {
    unsigned long long* ukeys = nullptr;  // device, compact keys
    uint64_t m = 0;                       // unique count (valid after sync)
    uint32_t nb = 1;
    uint64_t draws = 0;
    bool exhaustive = false;
    uint64_t raw = 0;
    bool q8 = false;  // the gather ran the 8-bit filter
    uint32_t head = 0;  // the gather ran the head filter (sngb_head.cu): its bytes per row
};

// Graph build for query rows [rb, re) (see sngb_api.cu).  upper_only: in the
// exhaustive branch pair each row only with v > u (build_full_graph,
// graph.cpp:191-220: every unordered pair once over a row split)
int build_graph(DevCtx& c, cudaStream_t s, Timer& tm, const float* d_pts, uint64_t n, uint32_t d,
                double eps, double rate, uint64_t seed, uint64_t rb, uint64_t re,
                GraphResult& gr, const float* h_src = nullptr, const double* d_pts64 = nullptr,
                int32_t metric = kMetricEuclid, bool upper_only = false);
void ensure_cluster_bufs(DevCtx& c, uint64_t n, ClusterBuffers& b);
void fill_info(sngb_info* info, const unsigned long long* hc, uint64_t n, uint32_t d,
               const GraphResult& gr, uint64_t rows, Timer& tm, bool clustered, bool host);
// multi-GPU calls (sngb_multi.cu): the device list of opts (0: a single-GPU
// call, -1: bad options), and the call itself.  src_kind: 0 host fp32 rows,
// 1 host fp64 rows, 2 device fp32 rows on devs[0] (labels / roles there too).
int multi_devices(const sngb_opts* o, std::vector<int>& devs);
int multi_dbscan(const std::vector<int>& devs, int src_kind, const void* pts, uint64_t n,
                 uint32_t d, double eps, int32_t min_pts, double rate, uint64_t seed,
                 int32_t metric, bool exact, bool timing, int32_t* labels, uint8_t* roles,
                 sngb_info* info);
// launch accounting of the calling thread (sngb_info.kernel_launches / library_launches)
void reset_launches();
uint64_t hand_launches();
uint64_t lib_launches();

}  // namespace host
}  // namespace sngb
