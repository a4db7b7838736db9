"""Generate tests/golden/golden.json from the REFERENCE itself.

The reference's own graph.cpp + clusterer.cpp + rng.hpp, compiled unmodified
by oracle/Makefile into oracle/_ref/libsngref.so, produce every value here.
The reference ships no golden vectors for s < 1 (proj/tests/test_rng.cpp is
property-only), so these fixtures are how the oracle (oracle/sng_oracle.c)
and the CUDA path are pinned to it.  Run here (where /root/reference exists):

    python tests/golden/make_golden.py

Inputs are deterministic (seeded numpy / the synthetic generators), so the
fixture records the inputs' recipe plus SHA-256 digests of the outputs; tiny
cases also keep the full arrays.
"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import Reference, fnv1a64_u32  # noqa: E402
from paper_2006_06743_b200 import synthetic  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def random_points(n, d, seed, scale):
    rng = np.random.default_rng(seed)
    return rng.random((n, d), dtype=np.float32) * np.float32(scale)


# (name, recipe, eps, min_pts, rate, seed) -- recipe rebuilt by tests/_golden.py
CASES = [
    ("line12_kat", {"kind": "arange", "n": 12}, 1e9, 3, 0.25, 1),
    ("tiny_spec_line", {"kind": "explicit", "values": [[0.0], [0.5], [10.0], [10.5]]}, 1.0, 1, 1.0, 0),
    ("single_point", {"kind": "explicit", "values": [[1.0, 2.0]]}, 0.5, 1, 1.0, 0),
    ("two_points", {"kind": "explicit", "values": [[0.0, 0.0], [0.05, 0.0]]}, 0.1, 1, 0.3, 7),
    ("coincident5", {"kind": "explicit", "values": [[1.0, 1.0]] * 5}, 1.0, 4, 1.0, 0),
    ("rand_50x2", {"kind": "random", "n": 50, "d": 2, "seed": 7, "scale": 1.0}, 0.2, 3, 0.3, 7),
    ("rand_500x3", {"kind": "random", "n": 500, "d": 3, "seed": 3, "scale": 1.0}, 0.15, 4, 0.1, 3),
    ("rand_2000x16", {"kind": "random", "n": 2000, "d": 16, "seed": 11, "scale": 3.0}, 3.6, 5, 0.05, 11),
    ("rand_1500x784", {"kind": "random", "n": 1500, "d": 784, "seed": 2, "scale": 1.0}, 11.2, 5, 0.03, 2),
    ("rand_3000x33", {"kind": "random", "n": 3000, "d": 33, "seed": 5, "scale": 1.0}, 2.1, 5, 0.02, 5),
    ("rate1_300x2", {"kind": "random", "n": 300, "d": 2, "seed": 300, "scale": 1.0}, 0.08, 4, 1.0, 9),
    ("large_draws_6000x3", {"kind": "random", "n": 6000, "d": 3, "seed": 4, "scale": 1.0}, 0.1, 4, 0.8, 4),
    ("cfg1_n20000", {"kind": "synthetic", "cfg": 1, "n": 20000}, 0.03, 10, 0.1, 1),
    ("cfg2_n4000", {"kind": "synthetic", "cfg": 2, "n": 4000}, 4.5, 10, 700 / 4000, 2),
    ("cfg3_n30000", {"kind": "synthetic", "cfg": 3, "n": 30000}, 0.5, 5, 1000 / 30000, 3),
    ("cfg4_n40000", {"kind": "synthetic", "cfg": 4, "n": 40000}, 0.1, 4, 2500 / 40000, 4),
    ("cfg5_n30000", {"kind": "synthetic", "cfg": 5, "n": 30000}, 1.2, 5, 4000 / 30000, 5),
]


# dbscan_exact (clusterer.cpp:67-79) / build_full_graph (graph.cpp:191-220) cases:
# (name, recipe, eps, min_pts, metric)
EXACT_CASES = [
    ("exact_spec_line", {"kind": "explicit", "values": [[0.0], [0.5], [10.0], [10.5]]}, 1.0, 1,
     "euclidean"),
    ("exact_coincident5", {"kind": "explicit", "values": [[1.0, 1.0]] * 5}, 1.0, 4, "euclidean"),
    ("exact_single", {"kind": "explicit", "values": [[3.0, 4.0]]}, 0.5, 1, "euclidean"),
    ("exact_rand_500x3", {"kind": "random", "n": 500, "d": 3, "seed": 3, "scale": 1.0}, 0.15, 4,
     "euclidean"),
    ("exact_rand_3000x16", {"kind": "random", "n": 3000, "d": 16, "seed": 11, "scale": 3.0}, 3.6,
     5, "euclidean"),
    ("exact_rand_1200x784", {"kind": "random", "n": 1200, "d": 784, "seed": 2, "scale": 1.0},
     11.2, 5, "euclidean"),
    ("exact_cfg1_n6000", {"kind": "synthetic", "cfg": 1, "n": 6000}, 0.03, 10, "euclidean"),
    ("exact_manhattan_800x5", {"kind": "random", "n": 800, "d": 5, "seed": 8, "scale": 1.0}, 0.6,
     3, "manhattan"),
    ("exact_cosine_800x8", {"kind": "random", "n": 800, "d": 8, "seed": 9, "scale": 1.0}, 0.05,
     3, "cosine"),
]


def build_points(recipe):
    k = recipe["kind"]
    if k == "arange":
        return np.arange(recipe["n"], dtype=np.float32).reshape(-1, 1)
    if k == "explicit":
        return np.asarray(recipe["values"], np.float32)
    if k == "random":
        return random_points(recipe["n"], recipe["d"], recipe["seed"], recipe["scale"])
    if k == "synthetic":
        return synthetic.generate(recipe["cfg"], n=recipe["n"])
    raise KeyError(k)


def main():
    ref = Reference()
    g = {"generator": "tests/golden/make_golden.py (oracle/_ref: reference graph.cpp, "
                      "clusterer.cpp, rng.hpp compiled unmodified)"}
    # rng.hpp KATs
    g["stream_next"] = [{"seed": s, "id": i, "values": [str(v) for v in ref.stream_next(s, i, 8)]}
                        for s, i in [(1, 0), (0, 0), (42, 7), (5, 12345), (2**64 - 1, 2**63 + 5)]]
    g["stream_next_below"] = [
        {"seed": s, "id": i, "bound": b, "values": [int(v) for v in ref.stream_next_below(s, i, b, 16)]}
        for s, i, b in [(5, 12345, 19999), (1, 0, 7), (3, 999, 999999), (9, 1, 2**31 + 11)]]
    # Per-vertex partner sets at the five BASELINE geometries: the reference
    # exposes no per-vertex API, so these are SURVEY.md Appendix A's FNV-1a-64
    # digests (computed there from the compiled reference), carried verbatim.
    g["partners_fnv1a64"] = [
        {"n": 20000, "draws": 2000, "seed": 1, "u": 0, "first4": [25, 26, 28, 31], "last": 19998, "fnv": "a820a1d3471dc557"},
        {"n": 20000, "draws": 2000, "seed": 1, "u": 1, "first4": [15, 16, 24, 33], "last": 19992, "fnv": "6ff3b31692a62f1c"},
        {"n": 20000, "draws": 2000, "seed": 1, "u": 19999, "first4": [1, 46, 65, 71], "last": 19991, "fnv": "cf99297cf7a6947c"},
        {"n": 70000, "draws": 700, "seed": 2, "u": 0, "first4": [56, 72, 85, 170], "last": 69955, "fnv": "af6ebad7d2118bcc"},
        {"n": 70000, "draws": 700, "seed": 2, "u": 1, "first4": [56, 59, 183, 327], "last": 69937, "fnv": "00a1490b47e324cb"},
        {"n": 70000, "draws": 700, "seed": 2, "u": 69999, "first4": [7, 38, 43, 170], "last": 69892, "fnv": "cd50dff47879b481"},
        {"n": 1000000, "draws": 1000, "seed": 3, "u": 0, "first4": [3255, 4054, 4187, 4449], "last": 999951, "fnv": "8ed081343f629a9e"},
        {"n": 1000000, "draws": 1000, "seed": 3, "u": 1, "first4": [1808, 2129, 2142, 2338], "last": 999608, "fnv": "664aa3f14de54689"},
        {"n": 1000000, "draws": 1000, "seed": 3, "u": 999999, "first4": [53, 73, 153, 176], "last": 999692, "fnv": "36cd46a925fe767c"},
        {"n": 5000000, "draws": 2500, "seed": 4, "u": 0, "first4": [2162, 3044, 3928, 5594], "last": 4998994, "fnv": "281d8a4bfe8d00e6"},
        {"n": 5000000, "draws": 2500, "seed": 4, "u": 1, "first4": [3943, 4352, 4791, 5009], "last": 4998609, "fnv": "b1d9bf7898a19295"},
        {"n": 5000000, "draws": 2500, "seed": 4, "u": 4999999, "first4": [1021, 1104, 1250, 2128], "last": 4997689, "fnv": "0d7af1215c7f8911"},
        {"n": 20000000, "draws": 4000, "seed": 5, "u": 0, "first4": [12547, 13950, 24553, 33600], "last": 19999017, "fnv": "0c9045b58aa0c511"},
        {"n": 20000000, "draws": 4000, "seed": 5, "u": 1, "first4": [17137, 19289, 20069, 27154], "last": 19999914, "fnv": "dca3f1af76facb87"},
        {"n": 20000000, "draws": 4000, "seed": 5, "u": 19999999, "first4": [6161, 7504, 16134, 26107], "last": 19999735, "fnv": "821efb5f007cf27c"},
    ]
    g["cases"] = []
    for name, recipe, eps, min_pts, rate, seed in CASES:
        pts = build_points(recipe)
        ds = ref.dataset(pts)
        keys, evals, _ = ref.sampled_edges(ds, eps, rate, seed)
        labels, roles, info = ref.sng_dbscan(ds, eps, min_pts, rate, seed)
        c = {"name": name, "recipe": recipe, "eps": eps, "min_pts": min_pts, "rate": rate,
             "seed": seed, "n": int(pts.shape[0]), "d": int(pts.shape[1]),
             "distance_evals": info["distance_evals"], "edges": info["edges"],
             "graph_bytes": info["graph_bytes"], "cluster_count": info["cluster_count"],
             "edges_evals": evals, "points_sha256": sha(pts), "keys_sha256": sha(keys),
             "labels_sha256": sha(labels), "roles_sha256": sha(roles),
             "core": int((roles == 0).sum()), "border": int((roles == 1).sum()),
             "noise": int((roles == 2).sum())}
        if pts.shape[0] <= 64:
            c["keys"] = [str(int(k)) for k in keys]
            c["labels"] = labels.tolist()
            c["roles"] = roles.tolist()
        g["cases"].append(c)
        print(name, c["edges"], c["cluster_count"], flush=True)
    g["exact_cases"] = []
    for name, recipe, eps, min_pts, metric in EXACT_CASES:
        pts = build_points(recipe)
        ds = ref.dataset(pts)
        ref.set_metric(metric)
        labels, roles, info, keys = ref.dbscan_exact(ds, eps, min_pts)
        ref.set_metric("euclidean")
        c = {"name": name, "recipe": recipe, "eps": eps, "min_pts": min_pts, "metric": metric,
             "n": int(pts.shape[0]), "d": int(pts.shape[1]),
             "distance_evals": info["distance_evals"], "edges": info["edges"],
             "graph_bytes": info["graph_bytes"], "cluster_count": info["cluster_count"],
             "points_sha256": sha(pts), "keys_sha256": sha(keys), "labels_sha256": sha(labels),
             "roles_sha256": sha(roles), "core": int((roles == 0).sum()),
             "border": int((roles == 1).sum()), "noise": int((roles == 2).sum())}
        if pts.shape[0] <= 64:
            c["keys"] = [str(int(k)) for k in keys]
            c["labels"] = labels.tolist()
            c["roles"] = roles.tolist()
        g["exact_cases"].append(c)
        print(name, c["edges"], c["cluster_count"], flush=True)
    with open(OUT, "w") as f:
        json.dump(g, f, indent=1)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
