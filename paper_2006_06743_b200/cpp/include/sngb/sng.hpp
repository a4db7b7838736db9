// sngb/sng.hpp -- header-only C++ mirror of the reference's SNG-DBSCAN entry
// point, implemented over the C ABI (include/sngb.h, libsngb.so).
//
// Same names, argument meaning and error behaviour as the reference:
//   sng::Dataset         proj/include/sng/dataset.hpp:16-71   (fp64 rows: kept
//                        as fp32 when exact, else as fp64 for the fp64 entry points)
//   sng::Distance        proj/include/sng/distance.hpp:13-43 (euclidean, manhattan,
//                        cosine; no custom callbacks on the GPU path)
//   sng::SngParams       proj/include/sng/clusterer.hpp:11-24
//   sng::ClusterRunInfo  proj/include/sng/clusterer.hpp:27-31
//   sng::Clustering      proj/include/sng/dataset.hpp:78-91
//   sng::sng_dbscan      proj/include/sng/clusterer.hpp:42
// std::invalid_argument carries the reference's messages; CUDA failures and a
// missing GPU throw std::runtime_error (there is no CPU fallback).
//
// A reference user switches by replacing #include "sng/clusterer.hpp" with
// #include "sngb/sng.hpp" and linking -lsngb.
#pragma once

#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "sngb.h"

namespace sng {

inline constexpr std::int32_t kNoiseLabel = -1;

enum class PointRole : std::uint8_t { Core, Border, Noise };

class Dataset {
public:
    Dataset() = default;
    Dataset(std::vector<double> values, std::size_t dim) : dim_(dim) {
        if (dim_ == 0) throw std::invalid_argument("dataset dimension must be >= 1");
        if (values.empty() || values.size() % dim_ != 0)
            throw std::invalid_argument("dataset values do not form n x dim rows");
        values_.resize(values.size());
        bool exact = true;
        for (std::size_t i = 0; i < values.size(); ++i) {
            if (!std::isfinite(values[i]))
                throw std::invalid_argument("dataset contains a non-finite value");
            values_[i] = static_cast<float>(values[i]);
            exact = exact && static_cast<double>(values_[i]) == values[i];
        }
        if (!exact) values64_ = std::move(values);  // fp32 cannot hold them: the fp64 path
    }
    Dataset(std::vector<float> values, std::size_t dim) : values_(std::move(values)), dim_(dim) {
        if (dim_ == 0) throw std::invalid_argument("dataset dimension must be >= 1");
        if (values_.empty() || values_.size() % dim_ != 0)
            throw std::invalid_argument("dataset values do not form n x dim rows");
        for (float v : values_)
            if (!std::isfinite(v)) throw std::invalid_argument("dataset contains a non-finite value");
    }
    std::size_t size() const { return dim_ == 0 ? 0 : values_.size() / dim_; }
    std::size_t dim() const { return dim_; }
    bool empty() const { return values_.empty(); }
    const std::vector<float>& values_f32() const { return values_; }
    bool is_fp64() const { return !values64_.empty(); }
    const std::vector<double>& values_f64() const { return values64_; }
    // the reference's accessor (dataset.hpp:69-71): the rows as fp64
    std::vector<double> values() const {
        return is_fp64() ? values64_ : std::vector<double>(values_.begin(), values_.end());
    }

private:
    std::vector<float> values_;
    std::vector<double> values64_;
    std::size_t dim_ = 0;
};

enum class Metric { Euclidean, Manhattan, Cosine, Custom };

class Distance {
public:
    static Distance euclidean() { return Distance(Metric::Euclidean); }
    static Distance manhattan() { return Distance(Metric::Manhattan); }
    static Distance cosine() { return Distance(Metric::Cosine); }
    static Distance parse(const std::string& name) {
        if (name == "euclidean") return euclidean();
        if (name == "manhattan") return manhattan();
        if (name == "cosine") return cosine();
        throw std::invalid_argument("unknown distance '" + name +
                                    "' (expected euclidean, manhattan, or cosine)");
    }
    Metric kind() const { return kind_; }
    std::uint32_t flags() const {
        return kind_ == Metric::Manhattan ? SNGB_FLAG_MANHATTAN
                                          : (kind_ == Metric::Cosine ? SNGB_FLAG_COSINE : 0u);
    }

private:
    explicit Distance(Metric k) : kind_(k) {}
    Metric kind_;
};

struct SngParams {
    double eps = 0.0;
    int min_pts = 1;
    double rate = 1.0;
    std::uint64_t seed = 0;
    Distance dist = Distance::euclidean();
    int threads = 0;  // CPU workers in the reference; unused by the GPU path
    int device = -1;  // CUDA ordinal (-1 = current)
    // extension (ABI 4): shard the rows over several GPUs of this process --
    // 0/1: one GPU, N: N GPUs, -1: every visible GPU; `devices` optionally lists
    // the ordinals (a repeated ordinal runs several shards on one GPU)
    int num_gpus = 0;
    std::vector<std::int32_t> devices;

    void validate() const {
        if (!(eps > 0.0)) throw std::invalid_argument("eps must be > 0");
        if (min_pts < 1) throw std::invalid_argument("min_pts must be >= 1");
        if (!(rate > 0.0) || rate > 1.0) throw std::invalid_argument("rate must lie in (0, 1]");
    }
};

struct ClusterRunInfo {
    std::uint64_t distance_evals = 0;
    std::size_t edges = 0;
    std::size_t graph_bytes = 0;
    sngb_info gpu{};  // extension: GPU counters and stage times
};

struct Clustering {
    std::vector<std::int32_t> assignment;
    std::vector<PointRole> role;
    std::int32_t cluster_count = 0;
    std::size_t size() const { return assignment.size(); }
    std::size_t count_role(PointRole r) const {
        std::size_t c = 0;
        for (PointRole x : role) c += (x == r);
        return c;
    }
};

namespace detail {
inline void check(int rc) {
    if (rc == SNGB_OK) return;
    if (rc >= SNGB_ERR_EPS && rc <= SNGB_ERR_ARG) throw std::invalid_argument(sngb_strerror(rc));
    std::string m = sngb_strerror(rc);
    if (rc == SNGB_ERR_CUDA) m += std::string(": ") + sngb_last_error_detail();
    throw std::runtime_error(m);
}
inline sngb_opts opts(int device, std::uint32_t flags, int num_gpus,
                      const std::vector<std::int32_t>& devices) {
    sngb_opts o{};
    o.device = device;
    o.flags = flags;
    o.num_gpus = devices.empty() ? num_gpus
                                 : (num_gpus == 0 || num_gpus == 1
                                        ? static_cast<int>(devices.size())
                                        : num_gpus);
    o.devices = devices.empty() ? nullptr : devices.data();
    return o;
}

inline Clustering to_clustering(std::vector<std::int32_t>&& labels,
                                const std::vector<std::uint8_t>& roles, const sngb_info& gi) {
    Clustering c;
    const std::size_t n = labels.size();
    c.assignment = std::move(labels);
    c.role.resize(n);
    for (std::size_t i = 0; i < n; ++i) c.role[i] = static_cast<PointRole>(roles[i]);
    c.cluster_count = gi.cluster_count;
    return c;
}

inline void to_info(ClusterRunInfo* info, const sngb_info& gi) {
    if (!info) return;
    info->distance_evals = gi.distance_evals;
    info->edges = gi.edges;
    info->graph_bytes = gi.graph_bytes;
    info->gpu = gi;
}
}  // namespace detail

inline Clustering sng_dbscan(const Dataset& data, const SngParams& params,
                             ClusterRunInfo* info = nullptr) {
    params.validate();
    if (data.empty()) throw std::invalid_argument("dataset is empty");
    const std::size_t n = data.size();
    std::vector<std::int32_t> labels(n);
    std::vector<std::uint8_t> roles(n);
    sngb_opts o = detail::opts(params.device, params.dist.flags(), params.num_gpus,
                               params.devices);
    sngb_info gi{};
    const auto d = static_cast<std::uint32_t>(data.dim());
    detail::check(data.is_fp64()
                      ? sngb_dbscan_f64(data.values_f64().data(), n, d, params.eps, params.min_pts,
                                        params.rate, params.seed, &o, labels.data(), roles.data(),
                                        &gi)
                      : sngb_dbscan_f32(data.values_f32().data(), n, d, params.eps, params.min_pts,
                                        params.rate, params.seed, &o, labels.data(), roles.data(),
                                        &gi));
    Clustering c;
    c.assignment = std::move(labels);
    c.role.resize(n);
    for (std::size_t i = 0; i < n; ++i) c.role[i] = static_cast<PointRole>(roles[i]);
    c.cluster_count = gi.cluster_count;
    if (info) {
        info->distance_evals = gi.distance_evals;
        info->edges = gi.edges;
        info->graph_bytes = gi.graph_bytes;
        info->gpu = gi;
    }
    return c;
}

// Classical DBSCAN on the exact eps-graph (clusterer.hpp:46-48,
// clusterer.cpp:67-79): distance_evals = n(n-1)/2.
inline Clustering dbscan_exact(const Dataset& data, double eps, int min_pts,
                               const Distance& dist = Distance::euclidean(), int threads = 0,
                               ClusterRunInfo* info = nullptr, int device = -1,
                               int num_gpus = 0,
                               const std::vector<std::int32_t>& devices = {}) {
    (void)threads;
    if (!(eps > 0.0)) throw std::invalid_argument("eps must be > 0");
    if (min_pts < 1) throw std::invalid_argument("min_pts must be >= 1");
    if (data.empty()) throw std::invalid_argument("dataset is empty");
    const std::size_t n = data.size();
    std::vector<std::int32_t> labels(n);
    std::vector<std::uint8_t> roles(n);
    sngb_opts o = detail::opts(device, dist.flags(), num_gpus, devices);
    sngb_info gi{};
    const auto d = static_cast<std::uint32_t>(data.dim());
    detail::check(data.is_fp64()
                      ? sngb_dbscan_exact_f64(data.values_f64().data(), n, d, eps, min_pts, &o,
                                              labels.data(), roles.data(), &gi)
                      : sngb_dbscan_exact_f32(data.values_f32().data(), n, d, eps, min_pts, &o,
                                              labels.data(), roles.data(), &gi));
    detail::to_info(info, gi);
    return detail::to_clustering(std::move(labels), roles, gi);
}

// The canonical edge list of build_full_graph (graph.hpp:69-70, SampledGraph::edges():
// u < v, sorted) for fp32-exact data.
inline std::vector<std::pair<std::uint32_t, std::uint32_t>> full_graph_edges(
    const Dataset& data, double eps, const Distance& dist = Distance::euclidean(),
    std::uint64_t* distance_evals = nullptr, int device = -1) {
    if (data.empty()) throw std::invalid_argument("dataset is empty");
    if (data.is_fp64())
        throw std::invalid_argument("full_graph_edges: fp32-exact data only (use dbscan_exact)");
    sngb_opts o = detail::opts(device, dist.flags(), 0, {});
    sngb_info gi{};
    std::uint64_t cap = 1u << 20, cnt = 0;
    std::vector<std::uint64_t> keys;
    for (;;) {
        keys.resize(cap);
        const int rc = sngb_full_edges_f32(data.values_f32().data(), data.size(),
                                           static_cast<std::uint32_t>(data.dim()), eps, &o,
                                           keys.data(), cap, &cnt, &gi);
        if (rc == SNGB_ERR_CAPACITY) {
            cap = cnt;
            continue;
        }
        detail::check(rc);
        break;
    }
    if (distance_evals) *distance_evals = gi.distance_evals;
    std::vector<std::pair<std::uint32_t, std::uint32_t>> e(cnt);
    for (std::uint64_t i = 0; i < cnt; ++i)
        e[i] = {static_cast<std::uint32_t>(keys[i] >> 32), static_cast<std::uint32_t>(keys[i])};
    return e;
}

}  // namespace sng
