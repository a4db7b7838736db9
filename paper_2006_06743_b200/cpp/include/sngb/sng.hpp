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
}  // namespace detail

inline Clustering sng_dbscan(const Dataset& data, const SngParams& params,
                             ClusterRunInfo* info = nullptr) {
    params.validate();
    if (data.empty()) throw std::invalid_argument("dataset is empty");
    const std::size_t n = data.size();
    std::vector<std::int32_t> labels(n);
    std::vector<std::uint8_t> roles(n);
    sngb_opts o{params.device, params.dist.flags(), nullptr, 0, 0};
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

}  // namespace sng
