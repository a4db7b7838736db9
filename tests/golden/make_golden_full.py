"""Generate tests/golden/golden_full.json: the REFERENCE's results on the five
BASELINE configs at FULL size.

The reference's own graph.cpp + clusterer.cpp (oracle/_ref/libsngref.so,
compiled unmodified by oracle/Makefile) run once per config through
``sngref_full_run`` = build_sampled_graph (graph.cpp:133-189) followed by
cluster_graph (clusterer.cpp:7-52), which is sng_dbscan (clusterer.cpp:54-65)
with the canonical edge list kept.  The fixture stores SHA-256 digests of the
points, the canonical edge keys (u<<32|v, sorted), labels and roles, the
reference counters, plus 64 per-block label/role digests so a GPU mismatch
can be located without the reference.

Cost on the 8-core CPU container: cfg2 ~15 s, cfg3 ~25 s, cfg4 ~3-4 min,
cfg5 ~25 min.  Run here (where /root/reference exists):

    python tests/golden/make_golden_full.py [cfg ...]

Existing entries for configs not named on the command line are kept.
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import Reference  # noqa: E402
from paper_2006_06743_b200 import synthetic  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_full.json")
BLOCKS = 64


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def block_digests(a: np.ndarray, blocks: int = BLOCKS):
    """First 16 hex digits of the SHA-256 of each of `blocks` contiguous slices."""
    n = len(a)
    cuts = [(n * i) // blocks for i in range(blocks + 1)]
    return [sha(a[cuts[i]:cuts[i + 1]])[:16] for i in range(blocks)]


def run(cfg: int, ref: Reference) -> dict:
    w = synthetic.CONFIGS[cfg]
    t0 = time.time()
    pts = synthetic.generate(cfg)
    gen_s = time.time() - t0
    ds = ref.dataset(pts)
    labels, roles, info, keys = ref.full_run(ds, w.eps, w.min_pts, w.rate, w.seed, threads=0)
    del ds
    return {
        "cfg": cfg, "workload": w.name, "n": w.n, "d": w.d, "eps": w.eps, "min_pts": w.min_pts,
        "rate": w.rate, "seed": w.seed, "draws": w.draws,
        "distance_evals": info["distance_evals"], "edges": info["edges"],
        "graph_bytes": info["graph_bytes"], "cluster_count": info["cluster_count"],
        "core": int((roles == 0).sum()), "border": int((roles == 1).sum()),
        "noise": int((roles == 2).sum()),
        "points_sha256": sha(pts), "keys_sha256": sha(keys), "labels_sha256": sha(labels),
        "roles_sha256": sha(roles),
        "labels_blocks": block_digests(labels), "roles_blocks": block_digests(roles),
        "ref_ms": info["ms"], "ref_threads": ref.hw_threads(), "gen_s": gen_s,
    }


def main(argv):
    cfgs = [int(a) for a in argv] or [1, 2, 3, 4, 5]
    ref = Reference()
    g = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            g = json.load(f)
    g["generator"] = ("tests/golden/make_golden_full.py (oracle/_ref: reference graph.cpp, "
                      "clusterer.cpp, rng.hpp compiled unmodified; one build_sampled_graph + "
                      "cluster_graph per config)")
    g.setdefault("configs", {})
    for c in cfgs:
        e = run(c, ref)
        g["configs"][str(c)] = e
        print(f"cfg{c}: edges={e['edges']} k={e['cluster_count']} core={e['core']} "
              f"border={e['border']} noise={e['noise']} ref {e['ref_ms'] / 1e3:.1f} s",
              flush=True)
        with open(OUT, "w") as f:
            json.dump(g, f, indent=1)
    print("wrote", OUT)


if __name__ == "__main__":
    main(sys.argv[1:])
