/*
 * sngb.h -- C ABI of the B200-native SNG-DBSCAN hot path (libsngb.so).
 *
 * The reference (arXiv 2006.06743 companion library, C++20) has no C ABI and
 * no GPU path; its hot path is the C++ call
 *
 *     Clustering sng::sng_dbscan(const Dataset&, const SngParams&, ClusterRunInfo*)
 *         -- proj/include/sng/clusterer.hpp:42, proj/src/clusterer.cpp:54-65
 *
 * which builds the subsampled eps-graph (sng::build_sampled_graph,
 * graph.hpp:65-66, graph.cpp:133-189) and clusters it (sng::cluster_graph,
 * clusterer.hpp:38, clusterer.cpp:7-52).  The entry points below are what a
 * binding of that path binds: plain pointers and sizes, no C++ or torch types.
 * The C++ mirror (paper_2006_06743_b200/cpp/include/sngb/sng.hpp) and the
 * Python mirror (paper_2006_06743_b200/__init__.py) sit on top of them and
 * map status codes back to the reference's exception types and messages.
 *
 * Semantics are the reference's, bit for bit: the same per-vertex Floyd
 * partner sets from the same (seed, vertex) counter streams (rng.hpp), the
 * same fp64 eps decision (distance.hpp:75-83; an fp32 or, for wide rows, an
 * 8-bit filter decides a pair only where its error bound proves the decision
 * identical, every other pair is re-evaluated in the reference's exact fp64
 * order), the same core mask, components, border ties
 * and relabelling (clusterer.cpp:7-52).  Points are fp32 row-major n x d
 * (the reference widens to fp64; fp32 -> fp64 widening is exact).
 *
 * There is no CPU fallback: every entry point returns SNGB_ERR_NO_DEVICE when
 * no CUDA device is usable.
 */
#ifndef SNGB_H
#define SNGB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SNGB_ABI_VERSION 4

/* Status codes.  1..6 carry the reference's std::invalid_argument messages. */
enum {
    SNGB_OK = 0,
    SNGB_ERR_EPS = 1,        /* "eps must be > 0"                 clusterer.hpp:20, graph.cpp:19 */
    SNGB_ERR_MINPTS = 2,     /* "min_pts must be >= 1"            clusterer.hpp:21, clusterer.cpp:8 */
    SNGB_ERR_RATE = 3,       /* "rate must lie in (0, 1]"         clusterer.hpp:22, graph.cpp:136 */
    SNGB_ERR_EMPTY = 4,      /* "dataset is empty"                graph.cpp:18 */
    SNGB_ERR_DIM = 5,        /* "dataset dimension must be >= 1"  dataset.hpp:22 */
    SNGB_ERR_NONFINITE = 6,  /* "dataset contains a non-finite value" dataset.hpp:26 */
    SNGB_ERR_TOO_LARGE = 7,  /* n must fit u32 vertex ids (graph.cpp:147) */
    SNGB_ERR_ARG = 8,        /* null pointer / bad row range */
    SNGB_ERR_NO_DEVICE = 9,  /* no usable CUDA device (there is no CPU fallback) */
    SNGB_ERR_CUDA = 10,      /* CUDA runtime error; see sngb_last_error_detail() */
    SNGB_ERR_CAPACITY = 11,  /* caller-provided output buffer too small; *count_out = needed */
    SNGB_ERR_ZERO_VECTOR = 12 /* "cosine distance is undefined for zero vectors" distance.hpp:97 */
};

/* opts.flags */
#define SNGB_FLAG_TIMING 0x1u /* record per-stage CUDA-event times into sngb_info */
/* The metric of Distance::within (distance.hpp:75-84); default Euclidean.
 * Manhattan: sum |a_k - b_k| <= eps; cosine: 1 - clamp(dot / (|a| |b|)) <= eps,
 * SNGB_ERR_ZERO_VECTOR when a row has a zero fp64 norm (n >= 2). */
#define SNGB_FLAG_MANHATTAN 0x2u
#define SNGB_FLAG_COSINE 0x4u

typedef struct sngb_opts {
    int32_t device;     /* CUDA ordinal; -1 = current device */
    uint32_t flags;     /* SNGB_FLAG_* */
    void* stream;       /* cudaStream_t to run on; NULL = library-owned stream */
    uint64_t row_begin; /* sampled-edge entry only: query rows [row_begin, row_end) */
    uint64_t row_end;   /*   (row_end == 0 means n) -- the multi-GPU row shard */
    /* ABI 4 -- several GPUs of this process (the reference's parallel_over_vertices
     * row split, graph.cpp:45-63, across devices).  Used by
     * sngb_dbscan_f32/_f64, sngb_dbscan_f32_device and sngb_dbscan_exact_f32[_device]:
     *   num_gpus 0 or 1  one GPU (`device`), the single-GPU path;
     *   num_gpus N > 1   query rows sharded over N GPUs: each uploads its row shard,
     *                    the replica is assembled over NVLink peer copies, each GPU
     *                    builds the edges of its rows, keys are routed to the owner
     *                    of their smaller endpoint, and the union-find forests are
     *                    merged to a fixed point by peer-memory all-reduces;
     *   num_gpus -1      every visible GPU.
     * devices: N CUDA ordinals (NULL: device, device+1, ... or 0.. when device is
     * -1).  An ordinal may repeat: its shards then share that GPU (same results).
     * The GPUs must have peer access to each other (NVLink / NVSwitch); the
     * device-buffer entry takes its points / labels on devices[0].  Results are
     * identical to the single-GPU call, bit for bit. */
    int32_t num_gpus;
    const int32_t* devices;
} sngb_opts;

/* ClusterRunInfo (clusterer.hpp:27-31) + BuildStats (graph.hpp:56-58) + GPU counters. */
typedef struct sngb_info {
    /* reference fields */
    uint64_t distance_evals; /* n * draws, exactly as graph.cpp:153,176,179 count them */
    uint64_t edges;          /* unique undirected edges (SampledGraph::edge_count) */
    uint64_t graph_bytes;    /* (n+1)*8 + 2*edges*4 (SampledGraph::storage_bytes) */
    int32_t cluster_count;   /* Clustering::cluster_count */
    uint32_t core_count, border_count, noise_count;
    /* sampling */
    uint64_t draws;              /* min(ceil(rate*n), n-1) */
    uint64_t collisions;         /* Floyd replacement draws (t already chosen -> j) */
    uint64_t irregular_vertices; /* vertices whose stream hit the Lemire reject test */
    /* eps-test exactness accounting (north star: traceability of fp32 decisions) */
    uint64_t pairs_evaluated;  /* pairs the GPU actually tested (incl. duplicate t draws) */
    uint64_t band_rechecks;    /* filter value inside the guard band -> exact fp64 recheck */
    uint64_t band_1e6;         /* of those, |s32 - eps^2| <= 1e-6 * eps^2 */
    uint64_t fp32_flips;       /* pairs where a bare fp32 test would have decided wrongly */
    uint64_t directed_accepts; /* accepted (u,v) emissions before symmetrise/dedup */
    /* stage times in ms (only with SNGB_FLAG_TIMING; CUDA events on the run stream) */
    float ms_total, ms_upload, ms_sample, ms_gather, ms_extras, ms_sort, ms_cluster, ms_download;
    uint64_t gather_pairs; /* pairs evaluated by the dominant gather kernel */
    uint64_t gather_bytes; /* its algorithmic bytes (see filter_bits) */
    uint64_t kernel_launches; /* hand-written kernels launched by this call (CUB not counted) */
    uint64_t library_launches; /* CUB radix-sort / select / scan kernels launched by this call */
    /* ABI 2: the filter the gather ran with -- 32: fp32 rows (gather_bytes = pairs * 4d);
     * 8: the exact 8-bit filter for wide rows (gather_bytes = pairs * (d + 4): the
     * row's bytes and its norm; band_rechecks counts its exact fp64 re-evaluations);
     * ABI 3 -- 16: the head filter for narrow rows (an exact reject on a head of a
     * few 8/16-bit coordinates per row, head_bytes each; gather_bytes = pairs *
     * head_bytes + survivors * 4d, survivors taking the fp32 test) */
    uint32_t filter_bits;
    uint32_t head_bytes;
    /* ABI 4 -- multi-GPU calls: GPUs used, fixed-point merge rounds, keys moved by
     * the owner routing (0 on one GPU); ms_merge: route + merge (SNGB_FLAG_TIMING) */
    uint32_t num_gpus;
    uint32_t merge_rounds;
    uint64_t routed_keys;
    float ms_merge;
    uint32_t reserved;
} sngb_info;

/* sng::sng_dbscan (clusterer.hpp:42) on HOST buffers: pts[n*d] fp32 row-major,
 * labels_out[n] (cluster id or -1 = kNoiseLabel), roles_out[n] (PointRole:
 * 0 Core, 1 Border, 2 Noise; dataset.hpp:74).  Upload, compute and download
 * run on opts->stream; returns when labels are on the host. */
int sngb_dbscan_f32(const float* pts, uint64_t n, uint32_t d, double eps, int32_t min_pts,
                    double rate, uint64_t seed, const sngb_opts* opts, int32_t* labels_out,
                    uint8_t* roles_out, sngb_info* info_out);

/* Same with DEVICE buffers (d_pts[n*d], d_labels[n], d_roles[n] on opts->device).
 * Returns after the work on opts->stream has completed. */
int sngb_dbscan_f32_device(const float* d_pts, uint64_t n, uint32_t d, double eps,
                           int32_t min_pts, double rate, uint64_t seed, const sngb_opts* opts,
                           int32_t* d_labels, uint8_t* d_roles, sngb_info* info_out);

/* sng::build_sampled_graph (graph.hpp:65-66) restricted to query rows
 * [opts->row_begin, opts->row_end): the sorted unique canonical edge keys
 * (u << 32 | v, u < v) of every accepted pair sampled BY those rows, written
 * to d_keys_out (device).  With the full row range this is exactly
 * SampledGraph::edges() (graph.cpp:104-111).  If *count_out > capacity the
 * call returns SNGB_ERR_CAPACITY and writes nothing. */
int sngb_sampled_edges_f32_device(const float* d_pts, uint64_t n, uint32_t d, double eps,
                                  double rate, uint64_t seed, const sngb_opts* opts,
                                  uint64_t* d_keys_out, uint64_t capacity, uint64_t* count_out,
                                  sngb_info* info_out);

/* Host-buffer variant of the above (keys_out on the host). */
int sngb_sampled_edges_f32(const float* pts, uint64_t n, uint32_t d, double eps, double rate,
                           uint64_t seed, const sngb_opts* opts, uint64_t* keys_out,
                           uint64_t capacity, uint64_t* count_out, sngb_info* info_out);

/* sng::dbscan_exact (clusterer.hpp:46-48, clusterer.cpp:67-79): classical DBSCAN
 * on the exact eps-graph, build_full_graph (graph.cpp:191-220: every unordered
 * pair once, distance_evals = n(n-1)/2), then cluster_graph.  Validation order:
 * eps, min_pts (clusterer.cpp:69-70), then empty / dim (graph.cpp:17-21); no rate.
 * Metric from opts->flags, multi-GPU from opts->num_gpus as above. */
int sngb_dbscan_exact_f32(const float* pts, uint64_t n, uint32_t d, double eps, int32_t min_pts,
                          const sngb_opts* opts, int32_t* labels_out, uint8_t* roles_out,
                          sngb_info* info_out);
int sngb_dbscan_exact_f32_device(const float* d_pts, uint64_t n, uint32_t d, double eps,
                                 int32_t min_pts, const sngb_opts* opts, int32_t* d_labels,
                                 uint8_t* d_roles, sngb_info* info_out);
int sngb_dbscan_exact_f64(const double* pts, uint64_t n, uint32_t d, double eps, int32_t min_pts,
                          const sngb_opts* opts, int32_t* labels_out, uint8_t* roles_out,
                          sngb_info* info_out);
/* sng::build_full_graph (graph.hpp:69-70): its canonical edges (SampledGraph::edges(),
 * u << 32 | v, sorted) into keys_out (host); SNGB_ERR_CAPACITY as the sampled entry. */
int sngb_full_edges_f32(const float* pts, uint64_t n, uint32_t d, double eps,
                        const sngb_opts* opts, uint64_t* keys_out, uint64_t capacity,
                        uint64_t* count_out, sngb_info* info_out);

/* Many small problems at once (the theory lab calls
 * sng_dbscan for many n <= 1e5 datasets, theory.cpp:239-256).  Each problem is
 * what one sngb_dbscan_f32 call would take (flags: SNGB_FLAG_MANHATTAN /
 * _COSINE); the problems run concurrently on up to SNGB_BATCH_SLOTS (default
 * 8) host workers with their own device contexts and streams, so their kernel
 * launches and host syncs overlap.  Per-problem status in `status`; returns
 * SNGB_OK or the first failing problem's status. */
typedef struct sngb_problem {
    const float* pts;
    uint64_t n;
    uint32_t d;
    uint32_t flags;
    double eps;
    double rate;
    uint64_t seed;
    int32_t min_pts;
    int32_t status; /* out */
    int32_t* labels_out;
    uint8_t* roles_out;
    sngb_info* info_out; /* optional */
} sngb_problem;
int sngb_dbscan_batch_f32(sngb_problem* problems, uint64_t count, const sngb_opts* opts);

/* fp64 input -- the reference's own Dataset type (dataset.hpp:69-71).  Values
 * that are not exactly fp32 are kept in fp64 on the device: the filter works on
 * them rounded to fp32 (or quantised to 8 bits from the fp64 values) with its
 * accept / reject thresholds widened by the rounding bound
 * sqrt(d) (2^-23 max|x| + 2^-149), and every pair in the band is re-evaluated
 * with the reference's fp64 operation order on the fp64 values.  Same results
 * as the reference, bit for bit. */
int sngb_dbscan_f64(const double* pts, uint64_t n, uint32_t d, double eps, int32_t min_pts,
                    double rate, uint64_t seed, const sngb_opts* opts, int32_t* labels_out,
                    uint8_t* roles_out, sngb_info* info_out);
int sngb_dbscan_f64_device(const double* d_pts, uint64_t n, uint32_t d, double eps,
                           int32_t min_pts, double rate, uint64_t seed, const sngb_opts* opts,
                           int32_t* d_labels, uint8_t* d_roles, sngb_info* info_out);
int sngb_sampled_edges_f64(const double* pts, uint64_t n, uint32_t d, double eps, double rate,
                           uint64_t seed, const sngb_opts* opts, uint64_t* keys_out,
                           uint64_t capacity, uint64_t* count_out, sngb_info* info_out);

/* sng::cluster_graph (clusterer.hpp:38) over canonical edge keys on the device
 * (any order, duplicates allowed -- they are sorted and deduplicated first,
 * graph.cpp:34-40).  This is the merge step of the multi-GPU path: every rank
 * all-gathers the shard keys and clusters them. */
int sngb_cluster_edges_device(const uint64_t* d_keys, uint64_t nkeys, uint64_t n,
                              int32_t min_pts, const sngb_opts* opts, int32_t* d_labels,
                              uint8_t* d_roles, sngb_info* info_out);

/* ---- Multi-GPU merge steps: local union-find per GPU, then a
 * fixed-point merge by NCCL all-reduce of full-length vertex arrays.
 *
 * Query rows are sharded; rank r owns the canonical keys (a<<32 | b, a < b)
 * whose smaller endpoint a lies in its row shard (after an all-to-all of the
 * keys its edge builder produced).  Vertex arrays are full length n < 2^31
 * and int32, so the caller can SUM / MIN all-reduce them between the steps.
 * Every call is synchronous on opts->stream (or the library stream), and a
 * key with a >= b or b >= n fails it with SNGB_ERR_ARG before any write.
 * Together they replace connected_components + core/border/relabel
 * (graph.cpp:222-247, clusterer.cpp:7-52) for an edge set split over ranks. */

/* Sort + deduplicate canonical keys (any order, duplicates allowed) into d_out
 * (capacity >= nkeys, must not alias d_keys); *count_out = unique count
 * (graph.cpp:34-40). */
int sngb_unique_keys_device(const uint64_t* d_keys, uint64_t nkeys, uint64_t n,
                            const sngb_opts* opts, uint64_t* d_out, uint64_t* count_out);

/* d_degree[v] += number of keys incident to v: the owned part of deg(v)
 * (graph.hpp:28); SUM-all-reduce over ranks gives the sampled degree. */
int sngb_degrees_device(const uint64_t* d_keys, uint64_t nkeys, uint64_t n, const sngb_opts* opts,
                        int32_t* d_degree);

/* Union-find over the keys whose endpoints are both core (degree >= min_pts,
 * clusterer.cpp:12-13; graph.cpp:228-235).  d_parent in: a forest with
 * parent[v] <= v (the identity on the first call, the MIN-all-reduced array
 * afterwards); out: every core vertex holds its root, the smallest vertex of
 * its set.  *changed_out = vertices whose entry changed; the merge has reached
 * its fixed point when that is 0 on every rank. */
int sngb_components_device(const uint64_t* d_keys, uint64_t nkeys, uint64_t n,
                           const int32_t* d_degree, int32_t min_pts, const sngb_opts* opts,
                           int32_t* d_parent, uint64_t* changed_out);

/* Border attachment over the keys (clusterer.cpp:26-37): for a non-core
 * endpoint b of a core vertex a, d_border[b] = min(d_border[b], d_parent[a]).
 * Initialise d_border to INT32_MAX ("no core neighbour"); MIN-all-reduce it. */
int sngb_border_device(const uint64_t* d_keys, uint64_t nkeys, uint64_t n, const int32_t* d_degree,
                       int32_t min_pts, const int32_t* d_parent, const sngb_opts* opts,
                       int32_t* d_border);

/* Labels and roles from the merged arrays (clusterer.cpp:17-51): identical on
 * every rank.  info (optional): cluster/core/border/noise counts. */
int sngb_relabel_device(uint64_t n, const int32_t* d_degree, int32_t min_pts,
                        const int32_t* d_parent, const int32_t* d_border, const sngb_opts* opts,
                        int32_t* d_labels, uint8_t* d_roles, sngb_info* info_out);

/* Status code -> message (the reference's exception text for codes 1..6). */
const char* sngb_strerror(int code);
/* Thread-local detail of the last SNGB_ERR_CUDA (CUDA error string + site). */
const char* sngb_last_error_detail(void);
int sngb_abi_version(void);
/* Number of usable CUDA devices (0 on a host without a GPU). */
int sngb_device_count(void);
/* Free the library-owned device pools of every device. */
void sngb_release_pools(void);

#ifdef __cplusplus
}
#endif
#endif /* SNGB_H */
