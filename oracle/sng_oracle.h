/*
 * sng_oracle.h -- CPU restatement of the SNG-DBSCAN hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the checker the CUDA path is compared
 * against; it is never linked into, loaded by, or called from the product
 * library (paper_2006_06743_b200/).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.
 *
 * Every function cites the reference file:line it restates
 * (paths relative to the reference's proj/ directory).
 *
 * Parity pin: the restatement is checked in tests/test_oracle.py against
 *   (1) the known-answer vectors of SURVEY.md Appendix A (computed from the
 *       compiled reference), and
 *   (2) the compiled reference itself (oracle/_ref/libsngref.so, built from
 *       /root/reference/proj/src/{graph,clusterer}.cpp by oracle/Makefile),
 *       through the golden fixtures in tests/golden/ made by
 *       tests/golden/make_golden.py.
 */
#ifndef SNG_ORACLE_H
#define SNG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* rng.hpp:9-13 */
uint64_t orc_mix(uint64_t z);
/* rng.hpp:23-24: Stream(seed, id).key_ */
uint64_t orc_stream_key(uint64_t seed, uint64_t stream_id);
/* rng.hpp:26: count successive next() outputs of Stream(seed, id) */
void orc_stream_next(uint64_t seed, uint64_t stream_id, uint64_t count, uint64_t* out);
/* rng.hpp:35-48: count successive next_below(bound) outputs of Stream(seed,id) */
void orc_stream_next_below(uint64_t seed, uint64_t stream_id, uint64_t bound, uint64_t count,
                           uint64_t* out);

/* graph.cpp:139-140: min(size_t(ceil(rate*double(n))), n-1) */
uint64_t orc_draws(uint64_t n, double rate);

/* graph.cpp:161-174: partner set of vertex u (Floyd over [0,n-2], shift >= u),
 * written sorted ascending to out[draws].  Returns draws. Requires draws < n-1. */
uint64_t orc_partners(uint64_t n, uint64_t draws, uint64_t seed, uint32_t u, uint32_t* out);

/* distance.hpp:75-83 Euclidean within() on fp64-widened fp32 rows. */
int orc_within(const float* a, const float* b, uint32_t d, double eps);

/* Counters mirroring ClusterRunInfo (clusterer.hpp:27-31). */
typedef struct {
    uint64_t distance_evals;
    uint64_t edges;
    uint64_t graph_bytes;
    int32_t cluster_count;
} orc_info;

/* graph.cpp:133-189 build_sampled_graph: canonical sorted unique edge keys
 * (u<<32 | v, u < v).  *keys_out is malloc'ed; caller frees with orc_free.
 * threads <= 0 -> all cores.  Returns 0, or a negative error code. */
int orc_sampled_edges(const float* pts, uint64_t n, uint32_t d, double eps, double rate,
                      uint64_t seed, int threads, uint64_t** keys_out, uint64_t* nkeys,
                      uint64_t* distance_evals);

/* The same restricted to the query rows [row_begin, row_end) -- the edges a
 * row shard of the multi-GPU path produces (graph.cpp:146-177 per vertex). */
int orc_sampled_edges_rows(const float* pts, uint64_t n, uint32_t d, double eps, double rate,
                           uint64_t seed, int threads, uint64_t row_begin, uint64_t row_end,
                           uint64_t** keys_out, uint64_t* nkeys, uint64_t* distance_evals);

/* clusterer.cpp:7-52 cluster_graph over canonical sorted unique keys. */
int orc_cluster_edges(const uint64_t* keys, uint64_t nkeys, uint64_t n, int32_t min_pts,
                      int32_t* labels, uint8_t* roles, int32_t* cluster_count);

/* clusterer.cpp:54-65 sng_dbscan. Error codes: -1 eps, -2 min_pts, -3 rate,
 * -4 empty dataset, -5 dim, -6 non-finite. */
int orc_sng_dbscan(const float* pts, uint64_t n, uint32_t d, double eps, int32_t min_pts,
                   double rate, uint64_t seed, int threads, int32_t* labels, uint8_t* roles,
                   orc_info* info);

void orc_free(void* p);

#ifdef __cplusplus
}
#endif
#endif
