// Builds against the C++ mirror (sngb/sng.hpp) exactly as a reference user
// would against sng/clusterer.hpp.  Exit codes: 0 ok, 2 wrong result,
// 3 no GPU (std::runtime_error), 4 unexpected exception text.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "sngb/io.hpp"
#include "sngb/sng.hpp"

int main() {
    // argument errors come first, with the reference's messages
    try {
        sng::SngParams bad;
        bad.eps = 0.0;
        sng::sng_dbscan(sng::Dataset(std::vector<double>{0.0, 1.0}, 1), bad);
        return 4;
    } catch (const std::invalid_argument& e) {
        if (std::string(e.what()) != "eps must be > 0") return 4;
    }
    // SPEC.md clusterer example: {0, 0.5, 10, 10.5}, eps=1, min_pts=1, rate=1
    sng::Dataset ds(std::vector<double>{0.0, 0.5, 10.0, 10.5}, 1);
    sng::SngParams p;
    p.eps = 1.0;
    p.min_pts = 1;
    p.rate = 1.0;
    sng::ClusterRunInfo info;
    try {
        sng::Clustering c = sng::sng_dbscan(ds, p, &info);
        const bool ok = c.cluster_count == 2 && c.assignment == std::vector<int>{0, 0, 1, 1} &&
                        info.edges == 2 && info.distance_evals == 12;
        std::printf("clusters=%d edges=%zu evals=%llu\n", c.cluster_count, info.edges,
                    (unsigned long long)info.distance_evals);
        if (!ok) return 2;
        // the same example as fp64 values fp32 cannot hold, through an SNGD file
        // and a label file: the fp64 entry point, same clustering
        const char* dir = std::getenv("DEMO_DIR");
        const std::string base = dir ? dir : ".";
        sng::save_binary(sng::Dataset(std::vector<double>{0.1, 0.6, 10.1, 10.6}, 1),
                         base + "/demo.sngd");
        sng::Dataset d64 = sng::load_binary(base + "/demo.sngd");
        if (!d64.is_fp64()) return 2;
        sng::Clustering c64 = sng::sng_dbscan(d64, p, &info);
        sng::save_clustering(c64, base + "/demo.labels");
        const bool ok64 = sng::load_labels(base + "/demo.labels") == c.assignment &&
                          info.gpu.filter_bits == 32;
        std::printf("fp64 via SNGD: clusters=%d ok=%d\n", c64.cluster_count, (int)ok64);
        if (!ok64) return 2;
        // Manhattan on the same example: |0 - 0.5| = 0.5 <= 1, clusters unchanged
        p.dist = sng::Distance::parse("manhattan");
        sng::Clustering cm = sng::sng_dbscan(ds, p, &info);
        std::printf("manhattan: clusters=%d\n", cm.cluster_count);
        if (cm.assignment != c.assignment) return 2;
        // dbscan_exact (clusterer.cpp:67-79): same clusters, n(n-1)/2 = 6 evaluations
        sng::ClusterRunInfo ei;
        sng::Clustering ce = sng::dbscan_exact(ds, 1.0, 1, sng::Distance::euclidean(), 0, &ei);
        std::uint64_t fe = 0;
        const auto edges = sng::full_graph_edges(ds, 1.0, sng::Distance::euclidean(), &fe);
        std::printf("exact: clusters=%d evals=%llu full_edges=%zu\n", ce.cluster_count,
                    (unsigned long long)ei.distance_evals, edges.size());
        if (ce.assignment != c.assignment || ei.distance_evals != 6 || fe != 6 ||
            edges.size() != 2 || edges[0] != std::make_pair(0u, 1u))
            return 2;
        // two row shards on GPU 0 (ABI 4 multi-GPU path, a repeated ordinal)
        sng::SngParams pm = p;
        pm.dist = sng::Distance::euclidean();
        pm.devices = {0, 0};
        sng::ClusterRunInfo mi;
        sng::Clustering cmg = sng::sng_dbscan(ds, pm, &mi);
        std::printf("multi: clusters=%d gpus=%u\n", cmg.cluster_count, mi.gpu.num_gpus);
        return (cmg.assignment == c.assignment && mi.gpu.num_gpus == 2) ? 0 : 2;
    } catch (const std::runtime_error& e) {
        std::printf("runtime_error: %s\n", e.what());
        return 3;
    }
}
