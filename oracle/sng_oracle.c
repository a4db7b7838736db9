/*
 * sng_oracle.c -- CPU restatement of the SNG-DBSCAN hot path (plain C11).
 *
 * TEST INFRASTRUCTURE ONLY: the checker for the CUDA path, never part of the
 * product (see sng_oracle.h).  Citations are to the reference's proj/ tree.
 *
 * Arithmetic notes:
 *   - u64 integer work (mix / Stream / next_below / Floyd) is restated
 *     bit-exactly; the 128-bit Lemire product uses unsigned __int128 exactly
 *     as rng.hpp:37 does.
 *   - within() is evaluated in fp64 with the reference's sequential order
 *     (distance.hpp:77-82).  This file must be compiled WITHOUT -ffast-math
 *     and without FMA contraction (-ffp-contract=off), see oracle/Makefile.
 */
#include "sng_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#define ORC_GAMMA 0x9e3779b97f4a7c15ULL

/* rng.hpp:9-13 */
uint64_t orc_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* rng.hpp:23-24 */
uint64_t orc_stream_key(uint64_t seed, uint64_t stream_id) {
    return orc_mix(seed + ORC_GAMMA) ^ orc_mix(stream_id * 0xda942042e4dd58b5ULL + 0x8bb84b93962eacc9ULL);
}

typedef struct {
    uint64_t key;
    uint64_t counter;
} orc_stream;

/* rng.hpp:26 -- pre-increment counter */
static inline uint64_t stream_next(orc_stream* s) { return orc_mix(s->key + (++s->counter) * ORC_GAMMA); }

/* rng.hpp:35-48 */
static inline uint64_t stream_next_below(orc_stream* s, uint64_t bound) {
    uint64_t x = stream_next(s);
    unsigned __int128 m = (unsigned __int128)x * bound;
    uint64_t lo = (uint64_t)m;
    if (lo < bound) {
        const uint64_t threshold = (0 - bound) % bound;
        while (lo < threshold) {
            x = stream_next(s);
            m = (unsigned __int128)x * bound;
            lo = (uint64_t)m;
        }
    }
    return (uint64_t)(m >> 64);
}

void orc_stream_next(uint64_t seed, uint64_t stream_id, uint64_t count, uint64_t* out) {
    orc_stream s = {orc_stream_key(seed, stream_id), 0};
    for (uint64_t i = 0; i < count; ++i) out[i] = stream_next(&s);
}

void orc_stream_next_below(uint64_t seed, uint64_t stream_id, uint64_t bound, uint64_t count,
                           uint64_t* out) {
    orc_stream s = {orc_stream_key(seed, stream_id), 0};
    for (uint64_t i = 0; i < count; ++i) out[i] = stream_next_below(&s, bound);
}

/* graph.cpp:139-140 */
uint64_t orc_draws(uint64_t n, double rate) {
    uint64_t c = (uint64_t)ceil(rate * (double)n);
    return c < n - 1 ? c : n - 1;
}

/* ---- open-addressing u64 set: stands in for std::unordered_set (graph.cpp:164) ---- */
typedef struct {
    uint64_t* slot;
    uint64_t cap; /* power of two */
} u64set;

#define SET_EMPTY UINT64_MAX

static void set_init(u64set* s, uint64_t want) {
    uint64_t cap = 16;
    while (cap < 2 * want + 2) cap <<= 1;
    if (cap > s->cap) {
        free(s->slot);
        s->slot = (uint64_t*)malloc(cap * sizeof(uint64_t));
        s->cap = cap;
    }
    memset(s->slot, 0xff, s->cap * sizeof(uint64_t));
}

/* returns 1 if inserted, 0 if already present (unordered_set::insert().second) */
static inline int set_insert(u64set* s, uint64_t v) {
    uint64_t mask = s->cap - 1;
    uint64_t h = orc_mix(v) & mask;
    for (;;) {
        uint64_t cur = s->slot[h];
        if (cur == v) return 0;
        if (cur == SET_EMPTY) {
            s->slot[h] = v;
            return 1;
        }
        h = (h + 1) & mask;
    }
}

static int cmp_u32(const void* a, const void* b) {
    uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return (x > y) - (x < y);
}

/* graph.cpp:161-174: Floyd's sampling of `draws` distinct values from
 * [0, pool), pool = n-1, then shift indices >= u by one.  Output order is
 * irrelevant to the reference (pairs are sorted later, graph.cpp:36,69), so
 * the set is emitted in insertion order here and sorted by the caller. */
static uint64_t floyd_partners(u64set* set, uint64_t n, uint64_t draws, uint64_t seed, uint32_t u,
                               uint32_t* out) {
    orc_stream s = {orc_stream_key(seed, u), 0};
    const uint64_t pool = n - 1;
    uint64_t k = 0;
    set_init(set, draws);
    for (uint64_t j = pool - draws; j < pool; ++j) {
        uint64_t t = stream_next_below(&s, j + 1);
        uint64_t e = set_insert(set, t) ? t : (set_insert(set, j), j);
        out[k++] = (uint32_t)(e >= u ? e + 1 : e);
    }
    return k;
}

uint64_t orc_partners(uint64_t n, uint64_t draws, uint64_t seed, uint32_t u, uint32_t* out) {
    u64set set = {0, 0};
    uint64_t k = floyd_partners(&set, n, draws, seed, u, out);
    free(set.slot);
    qsort(out, k, sizeof(uint32_t), cmp_u32);
    return k;
}

/* distance.hpp:75-83: sequential fp64 sum of squared differences, no sqrt */
int orc_within(const float* a, const float* b, uint32_t d, double eps) {
    double s = 0.0;
    for (uint32_t k = 0; k < d; ++k) {
        const double t = (double)a[k] - (double)b[k];
        s += t * t;
    }
    return s <= eps * eps;
}

/* ---- LSD radix sort of u64 keys (replaces std::sort at graph.cpp:36,69) ---- */
static void radix_sort_u64(uint64_t* a, uint64_t m) {
    if (m < 2) return;
    uint64_t* tmp = (uint64_t*)malloc(m * sizeof(uint64_t));
    uint64_t maxv = 0;
    for (uint64_t i = 0; i < m; ++i)
        if (a[i] > maxv) maxv = a[i];
    uint64_t* src = a;
    uint64_t* dst = tmp;
    for (int shift = 0; shift < 64 && (maxv >> shift) != 0; shift += 16) {
        uint64_t cnt[65536 + 1];
        memset(cnt, 0, sizeof(cnt));
        for (uint64_t i = 0; i < m; ++i) cnt[((src[i] >> shift) & 0xffff) + 1]++;
        for (int b = 0; b < 65536; ++b) cnt[b + 1] += cnt[b];
        for (uint64_t i = 0; i < m; ++i) dst[cnt[(src[i] >> shift) & 0xffff]++] = src[i];
        uint64_t* t = src;
        src = dst;
        dst = t;
    }
    if (src != a) memcpy(a, src, m * sizeof(uint64_t));
    free(tmp);
}

static uint64_t sort_unique_u64(uint64_t* a, uint64_t m) {
    radix_sort_u64(a, m);
    uint64_t k = 0;
    for (uint64_t i = 0; i < m; ++i)
        if (k == 0 || a[i] != a[k - 1]) a[k++] = a[i];
    return k;
}

/* ---- per-vertex worker (graph.cpp:146-177) ---- */
typedef struct {
    const float* pts;
    uint64_t n;
    uint32_t d;
    double eps;
    uint64_t draws;
    uint64_t seed;
    uint64_t begin, end;
    uint64_t* keys;
    uint64_t nkeys, capkeys;
    uint64_t evals;
} worker_arg;

static void push_key(worker_arg* w, uint32_t u, uint32_t v) {
    if (w->nkeys == w->capkeys) {
        w->capkeys = w->capkeys ? 2 * w->capkeys : 1024;
        w->keys = (uint64_t*)realloc(w->keys, w->capkeys * sizeof(uint64_t));
    }
    uint32_t a = u < v ? u : v, b = u < v ? v : u; /* graph.cpp:183-186 */
    w->keys[w->nkeys++] = ((uint64_t)a << 32) | b;
}

static void* worker(void* p) {
    worker_arg* w = (worker_arg*)p;
    const uint64_t n = w->n;
    const uint32_t d = w->d;
    u64set set = {0, 0};
    uint32_t* partners = NULL;
    if (w->draws < n - 1) partners = (uint32_t*)malloc((w->draws ? w->draws : 1) * sizeof(uint32_t));
    for (uint64_t ui = w->begin; ui < w->end; ++ui) {
        const uint32_t u = (uint32_t)ui;
        const float* x = w->pts + (uint64_t)u * d;
        if (w->draws >= n - 1) { /* graph.cpp:157-159 exhaustive branch */
            for (uint64_t v = 0; v < n; ++v) {
                if (v == u) continue;
                ++w->evals;
                if (orc_within(x, w->pts + v * d, d, w->eps)) push_key(w, u, (uint32_t)v);
            }
        } else { /* graph.cpp:161-174 */
            uint64_t k = floyd_partners(&set, n, w->draws, w->seed, u, partners);
            for (uint64_t i = 0; i < k; ++i) {
                ++w->evals;
                if (orc_within(x, w->pts + (uint64_t)partners[i] * d, d, w->eps)) push_key(w, u, partners[i]);
            }
        }
    }
    free(partners);
    free(set.slot);
    return NULL;
}

static int resolve_threads(int threads, uint64_t n) { /* graph.cpp:23-31 */
    if (threads <= 0) {
        long hw = sysconf(_SC_NPROCESSORS_ONLN);
        threads = hw <= 0 ? 1 : (int)hw;
    }
    uint64_t cap = n / 256 + 1;
    return (int)((uint64_t)threads < cap ? (uint64_t)threads : cap);
}

int orc_sampled_edges(const float* pts, uint64_t n, uint32_t d, double eps, double rate,
                      uint64_t seed, int threads, uint64_t** keys_out, uint64_t* nkeys,
                      uint64_t* distance_evals) {
    return orc_sampled_edges_rows(pts, n, d, eps, rate, seed, threads, 0, n, keys_out, nkeys,
                                  distance_evals);
}

int orc_sampled_edges_rows(const float* pts, uint64_t n, uint32_t d, double eps, double rate,
                           uint64_t seed, int threads, uint64_t row_begin, uint64_t row_end,
                           uint64_t** keys_out, uint64_t* nkeys, uint64_t* distance_evals) {
    if (n == 0) return -4;
    if (!(eps > 0.0)) return -1;
    if (!(rate > 0.0) || rate > 1.0) return -3;
    if (row_begin > row_end || row_end > n) return -7;
    const uint64_t draws = orc_draws(n, rate);
    const uint64_t rows = row_end - row_begin;
    int workers = resolve_threads(threads, rows ? rows : 1);
    worker_arg* args = (worker_arg*)calloc((size_t)workers, sizeof(worker_arg));
    pthread_t* tids = (pthread_t*)calloc((size_t)workers, sizeof(pthread_t));
    const uint64_t chunk = (rows + workers - 1) / workers; /* graph.cpp:52 */
    int used = 0;
    for (int t = 0; t < workers; ++t) {
        uint64_t b = row_begin + t * chunk, e = b + chunk < row_end ? b + chunk : row_end;
        if (b >= e) break;
        args[t] = (worker_arg){pts, n, d, eps, draws, seed, b, e, NULL, 0, 0, 0};
        ++used;
    }
    if (used == 1) {
        worker(&args[0]);
    } else {
        for (int t = 0; t < used; ++t) pthread_create(&tids[t], NULL, worker, &args[t]);
        for (int t = 0; t < used; ++t) pthread_join(tids[t], NULL);
    }
    uint64_t total = 0, evals = 0;
    for (int t = 0; t < used; ++t) {
        total += args[t].nkeys;
        evals += args[t].evals;
    }
    uint64_t* keys = (uint64_t*)malloc((total ? total : 1) * sizeof(uint64_t));
    uint64_t off = 0;
    for (int t = 0; t < used; ++t) {
        if (args[t].nkeys) memcpy(keys + off, args[t].keys, args[t].nkeys * sizeof(uint64_t));
        off += args[t].nkeys;
        free(args[t].keys);
    }
    free(args);
    free(tids);
    *nkeys = sort_unique_u64(keys, total); /* graph.cpp:34-40 csr_from_pairs */
    *keys_out = keys;
    if (distance_evals) *distance_evals = evals;
    return 0;
}

/* union_find.hpp:10-41: path halving, union by size */
static uint32_t uf_find(uint32_t* parent, uint32_t x) {
    while (parent[x] != x) {
        parent[x] = parent[parent[x]];
        x = parent[x];
    }
    return x;
}

/* clusterer.cpp:7-52 cluster_graph (with graph.cpp:222-247 connected_components) */
int orc_cluster_edges(const uint64_t* keys, uint64_t nkeys, uint64_t n, int32_t min_pts,
                      int32_t* labels, uint8_t* roles, int32_t* cluster_count) {
    if (min_pts < 1) return -2;
    uint64_t* deg = (uint64_t*)calloc(n + 1, sizeof(uint64_t));
    for (uint64_t e = 0; e < nkeys; ++e) {
        deg[keys[e] >> 32]++;
        deg[keys[e] & 0xffffffffu]++;
    }
    /* CSR offsets (graph.cpp:84-102) so border scans see neighbour lists */
    uint64_t* off = (uint64_t*)calloc(n + 1, sizeof(uint64_t));
    for (uint64_t v = 0; v < n; ++v) off[v + 1] = off[v] + deg[v];
    uint32_t* nbr = (uint32_t*)malloc((off[n] ? off[n] : 1) * sizeof(uint32_t));
    uint64_t* cur = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
    memcpy(cur, off, n * sizeof(uint64_t));
    for (uint64_t e = 0; e < nkeys; ++e) {
        uint32_t u = (uint32_t)(keys[e] >> 32), v = (uint32_t)keys[e];
        nbr[cur[u]++] = v;
        nbr[cur[v]++] = u;
    }
    free(cur);

    uint8_t* core = (uint8_t*)malloc(n ? n : 1);
    for (uint64_t v = 0; v < n; ++v) core[v] = deg[v] >= (uint64_t)min_pts; /* clusterer.cpp:12-13 */

    uint32_t* parent = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
    uint32_t* size = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
    for (uint64_t v = 0; v < n; ++v) {
        parent[v] = (uint32_t)v;
        size[v] = 1;
    }
    for (uint64_t e = 0; e < nkeys; ++e) { /* graph.cpp:228-235 */
        uint32_t u = (uint32_t)(keys[e] >> 32), v = (uint32_t)keys[e];
        if (!core[u] || !core[v]) continue;
        uint32_t ru = uf_find(parent, u), rv = uf_find(parent, v);
        if (ru == rv) continue;
        if (size[ru] < size[rv]) {
            uint32_t t = ru;
            ru = rv;
            rv = t;
        }
        parent[rv] = ru;
        size[ru] += size[rv];
    }
    /* component ids by first appearance in vertex order (graph.cpp:237-245) */
    int32_t* root_id = (int32_t*)malloc((n ? n : 1) * sizeof(int32_t));
    int32_t* comp = (int32_t*)malloc((n ? n : 1) * sizeof(int32_t));
    int32_t count = 0;
    for (uint64_t v = 0; v < n; ++v) root_id[v] = -1;
    for (uint64_t v = 0; v < n; ++v) {
        comp[v] = -1;
        if (!core[v]) continue;
        uint32_t r = uf_find(parent, (uint32_t)v);
        if (root_id[r] < 0) root_id[r] = count++;
        comp[v] = root_id[r];
    }
    /* clusterer.cpp:17-39 */
    for (uint64_t v = 0; v < n; ++v) {
        labels[v] = -1;
        roles[v] = 2; /* Noise */
        if (core[v]) {
            labels[v] = comp[v];
            roles[v] = 0; /* Core */
        }
    }
    for (uint64_t v = 0; v < n; ++v) {
        if (core[v]) continue;
        int32_t best = -1;
        for (uint64_t k = off[v]; k < off[v + 1]; ++k) {
            uint32_t u = nbr[k];
            if (!core[u]) continue;
            if (best < 0 || comp[u] < best) best = comp[u];
        }
        if (best >= 0) {
            labels[v] = best;
            roles[v] = 1; /* Border */
        }
    }
    /* clusterer.cpp:41-51 relabel by smallest member */
    int32_t* remap = (int32_t*)malloc((count ? count : 1) * sizeof(int32_t));
    for (int32_t c = 0; c < count; ++c) remap[c] = -1;
    int32_t next = 0;
    for (uint64_t v = 0; v < n; ++v) {
        int32_t c = labels[v];
        if (c < 0) continue;
        if (remap[c] < 0) remap[c] = next++;
        labels[v] = remap[c];
    }
    *cluster_count = next;
    free(remap);
    free(root_id);
    free(comp);
    free(parent);
    free(size);
    free(core);
    free(nbr);
    free(off);
    free(deg);
    return 0;
}

int orc_sng_dbscan(const float* pts, uint64_t n, uint32_t d, double eps, int32_t min_pts,
                   double rate, uint64_t seed, int threads, int32_t* labels, uint8_t* roles,
                   orc_info* info) {
    /* clusterer.hpp:19-23 then graph.cpp:17-21 */
    if (!(eps > 0.0)) return -1;
    if (min_pts < 1) return -2;
    if (!(rate > 0.0) || rate > 1.0) return -3;
    if (n == 0) return -4;
    if (d == 0) return -5;
    for (uint64_t i = 0; i < n * d; ++i)
        if (!isfinite(pts[i])) return -6;
    uint64_t* keys = NULL;
    uint64_t nkeys = 0, evals = 0;
    int rc = orc_sampled_edges(pts, n, d, eps, rate, seed, threads, &keys, &nkeys, &evals);
    if (rc) return rc;
    int32_t count = 0;
    rc = orc_cluster_edges(keys, nkeys, n, min_pts, labels, roles, &count);
    free(keys);
    if (info) {
        info->distance_evals = evals;
        info->edges = nkeys;
        info->graph_bytes = (n + 1) * 8 + 2 * nkeys * 4; /* graph.hpp:41-43 */
        info->cluster_count = count;
    }
    return rc;
}

void orc_free(void* p) { free(p); }
