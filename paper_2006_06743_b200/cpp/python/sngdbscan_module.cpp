// sngdbscan_module.cpp -- the `sngdbscan` Python module the reference planned
// (proj/CMakeLists.txt:11, module sngdbscan via pybind11; proj/python/
// CMakeLists.txt:1 is a placeholder), over libsngb.so (include/sngb.h).
//
//   sngdbscan.sng_dbscan(points, eps, min_pts, rate=1.0, seed=0, num_gpus=None,
//                        dist="euclidean", devices=None) -> (labels, roles, info)
//   sngdbscan.dbscan_exact(points, eps, min_pts, num_gpus=None, dist="euclidean",
//                          devices=None) -> (labels, roles, info)
//
// points: a C-contiguous float32 or float64 [n, d] array (float64 values that
// fp32 holds exactly take the fp32 entry points, bit-identical either way);
// labels int32[n] (cluster id or -1), roles uint8[n] (0 Core, 1 Border, 2 Noise),
// info: ClusterRunInfo's fields plus the GPU counters.  The GIL is released for
// the call.  std::invalid_argument's messages (the reference's) become
// ValueError, CUDA failures / no GPU RuntimeError.  There is no CPU fallback.
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <cmath>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "sngb.h"

namespace py = pybind11;

namespace {

uint32_t metric_flags(const std::string& dist) {  // distance.hpp:37-43
    if (dist == "euclidean") return 0u;
    if (dist == "manhattan") return SNGB_FLAG_MANHATTAN;
    if (dist == "cosine") return SNGB_FLAG_COSINE;
    throw py::value_error("unknown distance '" + dist +
                          "' (expected euclidean, manhattan, or cosine)");
}

void check(int rc) {
    if (rc == SNGB_OK) return;
    std::string m = sngb_strerror(rc);
    if ((rc >= SNGB_ERR_EPS && rc <= SNGB_ERR_ARG) || rc == SNGB_ERR_ZERO_VECTOR)
        throw py::value_error(m);
    if (rc == SNGB_ERR_CUDA) m += std::string(": ") + sngb_last_error_detail();
    throw std::runtime_error(m);
}

py::dict info_dict(const sngb_info& g) {
    py::dict d;
    d["distance_evals"] = g.distance_evals;
    d["edges"] = g.edges;
    d["graph_bytes"] = g.graph_bytes;
    d["cluster_count"] = g.cluster_count;
    d["core"] = g.core_count;
    d["border"] = g.border_count;
    d["noise"] = g.noise_count;
    d["draws"] = g.draws;
    d["collisions"] = g.collisions;
    d["irregular_vertices"] = g.irregular_vertices;
    d["pairs_evaluated"] = g.pairs_evaluated;
    d["band_rechecks"] = g.band_rechecks;
    d["band_1e6"] = g.band_1e6;
    d["fp32_flips"] = g.fp32_flips;
    d["filter_bits"] = g.filter_bits;
    d["num_gpus"] = g.num_gpus ? g.num_gpus : 1u;
    d["merge_rounds"] = g.merge_rounds;
    d["kernel_launches"] = g.kernel_launches;
    return d;
}

struct Call {
    py::array_t<float> f32;
    py::array_t<double> f64;
    bool use64 = false;
    uint64_t n = 0;
    uint32_t d = 0;
};

// float32 as given; float64 narrowed when fp32 holds every value exactly
Call points_of(const py::array& pts) {
    if (pts.ndim() != 2) throw py::value_error("points must be a 2-D [n, d] array");
    Call c;
    c.n = (uint64_t)pts.shape(0);
    c.d = (uint32_t)pts.shape(1);
    if (c.d == 0) throw py::value_error("dataset dimension must be >= 1");
    if (pts.dtype().is(py::dtype::of<float>())) {
        c.f32 = py::array_t<float, py::array::c_style | py::array::forcecast>::ensure(pts);
        return c;
    }
    c.f64 = py::array_t<double, py::array::c_style | py::array::forcecast>::ensure(pts);
    if (!c.f64) throw py::value_error("points must be a float32 or float64 array");
    const double* p = c.f64.data();
    const size_t m = (size_t)c.n * c.d;
    bool exact = true;
    for (size_t i = 0; i < m && exact; ++i) exact = (double)(float)p[i] == p[i] || std::isnan(p[i]);
    if (exact) {
        c.f32 = py::array_t<float>({(py::ssize_t)c.n, (py::ssize_t)c.d});
        float* q = c.f32.mutable_data();
        for (size_t i = 0; i < m; ++i) q[i] = (float)p[i];
    } else {
        c.use64 = true;
    }
    return c;
}

sngb_opts make_opts(const std::string& dist, std::optional<int> num_gpus,
                    const std::optional<std::vector<int32_t>>& devices,
                    std::vector<int32_t>& keep) {
    sngb_opts o{};
    o.device = -1;
    o.flags = metric_flags(dist);
    o.num_gpus = num_gpus.value_or(0);
    if (devices && !devices->empty()) {
        keep = *devices;
        o.devices = keep.data();
        if (o.num_gpus == 0 || o.num_gpus == 1) o.num_gpus = (int32_t)keep.size();
    }
    return o;
}

py::tuple run(bool exact, const py::array& points, double eps, int min_pts, double rate,
              uint64_t seed, std::optional<int> num_gpus, const std::string& dist,
              const std::optional<std::vector<int32_t>>& devices) {
    Call c = points_of(points);
    std::vector<int32_t> keep;
    const sngb_opts o = make_opts(dist, num_gpus, devices, keep);
    py::array_t<int32_t> labels((py::ssize_t)c.n);
    py::array_t<uint8_t> roles((py::ssize_t)c.n);
    int32_t* lp = c.n ? labels.mutable_data() : nullptr;
    uint8_t* rp = c.n ? roles.mutable_data() : nullptr;
    sngb_info g{};
    int rc;
    {
        py::gil_scoped_release nogil;
        if (exact)
            rc = c.use64 ? sngb_dbscan_exact_f64(c.f64.data(), c.n, c.d, eps, min_pts, &o, lp, rp, &g)
                         : sngb_dbscan_exact_f32(c.f32.data(), c.n, c.d, eps, min_pts, &o, lp, rp, &g);
        else
            rc = c.use64 ? sngb_dbscan_f64(c.f64.data(), c.n, c.d, eps, min_pts, rate, seed, &o, lp,
                                           rp, &g)
                         : sngb_dbscan_f32(c.f32.data(), c.n, c.d, eps, min_pts, rate, seed, &o, lp,
                                           rp, &g);
    }
    check(rc);
    return py::make_tuple(labels, roles, info_dict(g));
}

}  // namespace

PYBIND11_MODULE(_sngdbscan, m) {
    m.doc() = "SNG-DBSCAN (arXiv 2006.06743) on B200 GPUs: the reference's sng_dbscan / "
              "dbscan_exact through libsngb.so";
    m.def(
        "sng_dbscan",
        [](const py::array& points, double eps, int min_pts, double rate, uint64_t seed,
           std::optional<int> num_gpus, const std::string& dist,
           std::optional<std::vector<int32_t>> devices) {
            return run(false, points, eps, min_pts, rate, seed, num_gpus, dist, devices);
        },
        py::arg("points"), py::arg("eps"), py::arg("min_pts"), py::arg("rate") = 1.0,
        py::arg("seed") = 0, py::arg("num_gpus") = py::none(), py::arg("dist") = "euclidean",
        py::arg("devices") = py::none(),
        "sng::sng_dbscan (clusterer.hpp:42): -> (labels int32[n], roles uint8[n], info dict)");
    m.def(
        "dbscan_exact",
        [](const py::array& points, double eps, int min_pts, std::optional<int> num_gpus,
           const std::string& dist, std::optional<std::vector<int32_t>> devices) {
            return run(true, points, eps, min_pts, 1.0, 0, num_gpus, dist, devices);
        },
        py::arg("points"), py::arg("eps"), py::arg("min_pts"), py::arg("num_gpus") = py::none(),
        py::arg("dist") = "euclidean", py::arg("devices") = py::none(),
        "sng::dbscan_exact (clusterer.hpp:46-48): -> (labels, roles, info dict)");
    m.def("device_count", &sngb_device_count, "usable CUDA devices (0: no GPU, calls fail)");
    m.attr("NOISE") = -1;
    m.attr("CORE") = 0;
    m.attr("BORDER") = 1;
    m.attr("ABI_VERSION") = sngb_abi_version();
}
