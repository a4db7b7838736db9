// sngb_cluster -- the `cluster` front-end of the reference's CLI (SPEC.md
// [MODULE] cli, cmd_cluster; the reference's proj/tools/CMakeLists.txt is a
// placeholder) over the C++ mirror and libsngb.so:
//
//   sngb_cluster --input DATA.sngd --eps E --min-pts M [--rate S] [--seed K]
//                [--dist euclidean|manhattan|cosine] [--output LABELS]
//                [--threads T] [--num-gpus N] [--exact]
//
// Reads an SNGD binary dataset (sngb/io.hpp), runs sng::sng_dbscan on the GPU
// (or sng::dbscan_exact with --exact), writes one label per line (noise "-1"),
// and prints  n=.. k=.. noise=.. edges=.. evals=.. ms=..  on stdout.
// Exit codes (SPEC cmd_cluster): 0 success (k = 0 included), 2 flag errors
// (usage on stderr; flags are validated before any computation), 3 I/O errors;
// 1 for a GPU / CUDA failure (there is no CPU fallback).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "sngb/io.hpp"
#include "sngb/sng.hpp"

namespace {

constexpr const char* kUsage =
    "usage: sngb_cluster --input PATH --eps E --min-pts M [--rate S (default 1.0)]\n"
    "                    [--seed K (default 0)] [--dist euclidean|manhattan|cosine]\n"
    "                    [--output PATH (default: INPUT.labels)] [--threads T]\n"
    "                    [--num-gpus N (default 1; -1: all)] [--exact]\n";

struct FlagError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

double to_double(const std::string& flag, const std::string& v) {
    char* end = nullptr;
    const double x = std::strtod(v.c_str(), &end);
    if (v.empty() || *end != '\0') throw FlagError(flag + ": '" + v + "' is not a number");
    return x;
}

long long to_int(const std::string& flag, const std::string& v) {
    char* end = nullptr;
    const long long x = std::strtoll(v.c_str(), &end, 10);
    if (v.empty() || *end != '\0') throw FlagError(flag + ": '" + v + "' is not an integer");
    return x;
}

struct Config {
    std::string input, output, dist = "euclidean";
    double eps = 0.0, rate = 1.0;
    long long min_pts = 0, threads = 0, num_gpus = 1;
    unsigned long long seed = 0;
    bool exact = false;
};

Config parse(int argc, char** argv) {
    std::map<std::string, std::string> kv;
    Config c;
    for (int i = 1; i < argc; ++i) {
        const std::string a = argv[i];
        if (a == "--exact") {
            c.exact = true;
            continue;
        }
        if (a == "--help" || a == "-h") throw FlagError("");
        if (a.rfind("--", 0) != 0) throw FlagError("unexpected argument '" + a + "'");
        if (i + 1 >= argc) throw FlagError(a + " needs a value");
        kv[a] = argv[++i];
    }
    static const char* known[] = {"--input", "--eps", "--min-pts", "--rate", "--seed",
                                  "--dist", "--output", "--threads", "--num-gpus"};
    for (const auto& [k, v] : kv) {
        bool ok = false;
        for (const char* q : known) ok = ok || k == q;
        if (!ok) throw FlagError("unknown flag " + k);
    }
    for (const char* req : {"--input", "--eps", "--min-pts"})
        if (!kv.count(req)) throw FlagError(std::string("missing ") + req);
    c.input = kv["--input"];
    c.eps = to_double("--eps", kv["--eps"]);
    c.min_pts = to_int("--min-pts", kv["--min-pts"]);
    if (kv.count("--rate")) c.rate = to_double("--rate", kv["--rate"]);
    if (kv.count("--seed")) c.seed = (unsigned long long)to_int("--seed", kv["--seed"]);
    if (kv.count("--threads")) c.threads = to_int("--threads", kv["--threads"]);
    if (kv.count("--num-gpus")) c.num_gpus = to_int("--num-gpus", kv["--num-gpus"]);
    if (kv.count("--dist")) c.dist = kv["--dist"];
    c.output = kv.count("--output") ? kv["--output"] : c.input + ".labels";
    // the library's checks, before any computation (clusterer.hpp:19-23, distance.hpp:37-43)
    sng::SngParams p;
    p.eps = c.eps;
    p.min_pts = (int)c.min_pts;
    p.rate = c.rate;
    try {
        if (c.min_pts < 1 || c.min_pts > 0x7fffffff) p.min_pts = 0;
        p.validate();
        (void)sng::Distance::parse(c.dist);
    } catch (const std::invalid_argument& e) {
        throw FlagError(e.what());
    }
    if (c.num_gpus == 0 || c.num_gpus < -1 || c.num_gpus > 16)
        throw FlagError("--num-gpus must be -1 or 1..16");
    return c;
}

}  // namespace

int main(int argc, char** argv) {
    Config cfg;
    try {
        cfg = parse(argc, argv);
    } catch (const FlagError& e) {
        if (*e.what()) std::fprintf(stderr, "sngb_cluster: %s\n", e.what());
        std::fputs(kUsage, stderr);
        return 2;
    }
    sng::Dataset data;
    try {
        data = sng::load_points(cfg.input);
    } catch (const sng::IoError& e) {
        std::fprintf(stderr, "sngb_cluster: %s\n", e.what());
        return 3;
    } catch (const sng::ParseError& e) {
        std::fprintf(stderr, "sngb_cluster: %s\n", e.what());
        return 3;
    } catch (const std::invalid_argument& e) {  // e.g. a non-finite value in the file
        std::fprintf(stderr, "sngb_cluster: %s\n", e.what());
        return 3;
    }
    sng::Clustering c;
    sng::ClusterRunInfo info;
    const auto t0 = std::chrono::steady_clock::now();
    try {
        const sng::Distance dist = sng::Distance::parse(cfg.dist);
        if (cfg.exact) {
            c = sng::dbscan_exact(data, cfg.eps, (int)cfg.min_pts, dist, (int)cfg.threads, &info,
                                  -1, (int)cfg.num_gpus);
        } else {
            sng::SngParams p;
            p.eps = cfg.eps;
            p.min_pts = (int)cfg.min_pts;
            p.rate = cfg.rate;
            p.seed = cfg.seed;
            p.dist = dist;
            p.threads = (int)cfg.threads;
            p.num_gpus = (int)cfg.num_gpus;
            c = sng::sng_dbscan(data, p, &info);
        }
    } catch (const std::invalid_argument& e) {
        std::fprintf(stderr, "sngb_cluster: %s\n", e.what());
        return 2;
    } catch (const std::runtime_error& e) {
        std::fprintf(stderr, "sngb_cluster: %s\n", e.what());
        return 1;
    }
    const double ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    try {
        sng::save_clustering(c, cfg.output);
    } catch (const sng::IoError& e) {
        std::fprintf(stderr, "sngb_cluster: %s\n", e.what());
        return 3;
    }
    std::printf("n=%zu k=%d noise=%zu edges=%zu evals=%llu ms=%.3f\n", c.size(), c.cluster_count,
                c.count_role(sng::PointRole::Noise), info.edges,
                (unsigned long long)info.distance_evals, ms);
    return 0;
}
