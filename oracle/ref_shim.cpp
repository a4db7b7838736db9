// ref_shim.cpp -- extern "C" shim over the UNMODIFIED reference sources.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file together with
// /root/reference/proj/src/{graph,clusterer}.cpp (in place, read-only) into
// oracle/_ref/libsngref.so.  It is used to (a) pin the C restatement in
// oracle/sng_oracle.c, (b) generate tests/golden/ fixtures, and (c) time the
// reference CPU path for bench.py's cpu_baseline / --impl reference legs.
// Nothing in the product library links or loads it.
//
// Entry points wrap, without changing semantics:
//   sng::sng_dbscan            clusterer.hpp:42 / clusterer.cpp:54-65
//   sng::build_sampled_graph   graph.hpp:65-66 / graph.cpp:133-189
//   sng::rng::Stream           rng.hpp:21-72
//   oracle::reference_dbscan   tests/oracles.hpp:87-132 (s = 1 oracle)
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "sng/clusterer.hpp"
#include "sng/graph.hpp"
#include "sng/rng.hpp"
#include "oracles.hpp"

namespace {
thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    return -1;
}
}  // namespace

extern "C" {

const char* sngref_last_error() { return g_err.c_str(); }

unsigned sngref_hw_threads() { return std::thread::hardware_concurrency(); }

void sngref_stream_next(uint64_t seed, uint64_t id, uint64_t count, uint64_t* out) {
    sng::rng::Stream s = sng::rng::substream(seed, id);
    for (uint64_t i = 0; i < count; ++i) out[i] = s.next();
}

void sngref_stream_next_below(uint64_t seed, uint64_t id, uint64_t bound, uint64_t count,
                              uint64_t* out) {
    sng::rng::Stream s = sng::rng::substream(seed, id);
    for (uint64_t i = 0; i < count; ++i) out[i] = s.next_below(bound);
}

// Widening fp32 -> fp64 happens here, outside any timed region.
void* sngref_dataset_create(const float* pts, uint64_t n, uint32_t d) {
    try {
        std::vector<double> v(pts, pts + n * d);
        return new sng::Dataset(std::move(v), d);
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

void* sngref_dataset_create_f64(const double* pts, uint64_t n, uint32_t d) {
    try {
        std::vector<double> v(pts, pts + n * d);
        return new sng::Dataset(std::move(v), d);
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

void sngref_dataset_free(void* ds) { delete static_cast<sng::Dataset*>(ds); }

// info[0]=distance_evals info[1]=edges info[2]=graph_bytes info[3]=cluster_count
// *ms = wall time of the sng_dbscan call alone.
// metric for the calls below (test infrastructure): 0 Euclidean, 1 Manhattan, 2 cosine
static thread_local int g_metric = 0;
void sngref_set_metric(int m) { g_metric = m; }
static sng::Distance metric_dist() {
    return g_metric == 1 ? sng::Distance::manhattan()
                         : (g_metric == 2 ? sng::Distance::cosine() : sng::Distance::euclidean());
}

int sngref_dbscan(void* ds, double eps, int32_t min_pts, double rate, uint64_t seed, int threads,
                  int32_t* labels, uint8_t* roles, uint64_t* info, double* ms) {
    try {
        const auto& data = *static_cast<sng::Dataset*>(ds);
        sng::SngParams p;
        p.eps = eps;
        p.min_pts = min_pts;
        p.rate = rate;
        p.seed = seed;
        p.threads = threads;
        p.dist = metric_dist();
        sng::ClusterRunInfo ri;
        auto t0 = std::chrono::steady_clock::now();
        sng::Clustering c = sng::sng_dbscan(data, p, &ri);
        auto t1 = std::chrono::steady_clock::now();
        if (ms) *ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        for (size_t i = 0; i < c.size(); ++i) {
            labels[i] = c.assignment[i];
            roles[i] = static_cast<uint8_t>(c.role[i]);
        }
        if (info) {
            info[0] = ri.distance_evals;
            info[1] = ri.edges;
            info[2] = ri.graph_bytes;
            info[3] = static_cast<uint64_t>(c.cluster_count);
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Canonical edge list (SampledGraph::edges(), graph.cpp:104-111) as u<<32|v keys.
int sngref_sampled_edges(void* ds, double eps, double rate, uint64_t seed, int threads,
                         uint64_t** keys, uint64_t* nkeys, uint64_t* evals, double* ms) {
    try {
        const auto& data = *static_cast<sng::Dataset*>(ds);
        sng::BuildStats st;
        auto t0 = std::chrono::steady_clock::now();
        sng::SampledGraph g = sng::build_sampled_graph(data, eps, rate, metric_dist(), seed,
                                                       threads, &st);
        auto t1 = std::chrono::steady_clock::now();
        if (ms) *ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        auto e = g.edges();
        auto* out = static_cast<uint64_t*>(std::malloc((e.size() ? e.size() : 1) * sizeof(uint64_t)));
        for (size_t i = 0; i < e.size(); ++i)
            out[i] = (static_cast<uint64_t>(e[i].first) << 32) | e[i].second;
        *keys = out;
        *nkeys = e.size();
        if (evals) *evals = st.distance_evals;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// One build_sampled_graph (graph.cpp:133-189) then cluster_graph
// (clusterer.cpp:7-52) -- exactly what sng_dbscan (clusterer.cpp:54-65) does,
// but also returning the canonical edge list, so full-size fixtures need one
// (long) graph build instead of two.  *keys is malloc'ed (sngref_free).
int sngref_full_run(void* ds, double eps, int32_t min_pts, double rate, uint64_t seed,
                    int threads, int32_t* labels, uint8_t* roles, uint64_t* info,
                    uint64_t** keys, uint64_t* nkeys, double* ms) {
    try {
        const auto& data = *static_cast<sng::Dataset*>(ds);
        sng::SngParams p;
        p.eps = eps;
        p.min_pts = min_pts;
        p.rate = rate;
        p.seed = seed;
        p.threads = threads;
        p.dist = metric_dist();
        p.validate();
        sng::BuildStats st;
        auto t0 = std::chrono::steady_clock::now();
        sng::SampledGraph g = sng::build_sampled_graph(data, p.eps, p.rate, p.dist, p.seed,
                                                       p.threads, &st);
        sng::Clustering c = sng::cluster_graph(g, p.min_pts);
        auto t1 = std::chrono::steady_clock::now();
        if (ms) *ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        for (size_t i = 0; i < c.size(); ++i) {
            labels[i] = c.assignment[i];
            roles[i] = static_cast<uint8_t>(c.role[i]);
        }
        info[0] = st.distance_evals;
        info[1] = g.edge_count();
        info[2] = g.storage_bytes();
        info[3] = static_cast<uint64_t>(c.cluster_count);
        auto e = g.edges();
        auto* out = static_cast<uint64_t*>(std::malloc((e.size() ? e.size() : 1) * sizeof(uint64_t)));
        for (size_t i = 0; i < e.size(); ++i)
            out[i] = (static_cast<uint64_t>(e[i].first) << 32) | e[i].second;
        *keys = out;
        *nkeys = e.size();
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// sng::dbscan_exact (clusterer.hpp:46-48, clusterer.cpp:67-79) over
// build_full_graph (graph.cpp:191-220); also returns its canonical edges.
int sngref_dbscan_exact(void* ds, double eps, int32_t min_pts, int threads, int32_t* labels,
                        uint8_t* roles, uint64_t* info, uint64_t** keys, uint64_t* nkeys,
                        double* ms) {
    try {
        const auto& data = *static_cast<sng::Dataset*>(ds);
        sng::ClusterRunInfo ri;
        auto t0 = std::chrono::steady_clock::now();
        sng::Clustering c = sng::dbscan_exact(data, eps, min_pts, metric_dist(), threads, &ri);
        auto t1 = std::chrono::steady_clock::now();
        if (ms) *ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        for (size_t i = 0; i < c.size(); ++i) {
            labels[i] = c.assignment[i];
            roles[i] = static_cast<uint8_t>(c.role[i]);
        }
        info[0] = ri.distance_evals;
        info[1] = ri.edges;
        info[2] = ri.graph_bytes;
        info[3] = static_cast<uint64_t>(c.cluster_count);
        if (keys) {
            sng::BuildStats st;
            sng::SampledGraph g = sng::build_full_graph(data, eps, metric_dist(), threads, &st);
            auto e = g.edges();
            auto* out = static_cast<uint64_t*>(
                std::malloc((e.size() ? e.size() : 1) * sizeof(uint64_t)));
            for (size_t i = 0; i < e.size(); ++i)
                out[i] = (static_cast<uint64_t>(e[i].first) << 32) | e[i].second;
            *keys = out;
            *nkeys = e.size();
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// tests/oracles.hpp:87-132: classical expand-cluster DBSCAN (the s=1 oracle).
int sngref_reference_dbscan(void* ds, double eps, int32_t min_pts, int32_t* labels,
                            uint8_t* core) {
    try {
        const auto& data = *static_cast<sng::Dataset*>(ds);
        auto r = oracle::reference_dbscan(data, eps, min_pts);
        for (size_t i = 0; i < r.assignment.size(); ++i) {
            labels[i] = r.assignment[i];
            core[i] = r.core[i] ? 1 : 0;
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

void sngref_free(void* p) { std::free(p); }

}  // extern "C"
