"""k_floyd_head (SNGB_FUSED=1) vs the two-kernel default (SNGB_FUSED=0) A/B
(not part of the product): step time and stages, labels, roles and counters
compared bit for bit.

    python tools/fh_ab.py 4 5
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2006_06743_b200 as sng  # noqa: E402
from paper_2006_06743_b200 import synthetic  # noqa: E402

for cfg in [int(c) for c in sys.argv[1:]] or [5]:
    w = synthetic.CONFIGS[cfg]
    x = torch.from_numpy(synthetic.generate(cfg)).cuda()
    outs = {}
    for fused in ("0", "1"):
        os.environ["SNGB_FUSED"] = fused
        sng.sng_dbscan_device(x, w.eps, w.min_pts, w.rate, w.seed, timing=True)
        runs = [sng.sng_dbscan_device(x, w.eps, w.min_pts, w.rate, w.seed, timing=True) for _ in range(3)]
        lab, rol, gi = runs[-1]
        rec = {"cfg": cfg, "fused": fused, "ms_total": statistics.median(r[2].ms_total for r in runs),
               "ms_sample": statistics.median(r[2].ms_sample for r in runs),
               "ms_gather": statistics.median(r[2].ms_gather for r in runs)}
        keys = ("edges", "collisions", "irregular_vertices", "gather_pairs", "pairs_evaluated",
                "cluster_count", "core_count", "noise_count")
        rec.update({k: getattr(gi, k) for k in keys if hasattr(gi, k)})
        outs[fused] = (lab.cpu(), rol.cpu(), {k: rec.get(k) for k in keys})
        print(json.dumps(rec), flush=True)
    a, b = outs["0"], outs["1"]
    print(json.dumps({"cfg": cfg, "labels_equal": bool(torch.equal(a[0], b[0])),
                      "roles_equal": bool(torch.equal(a[1], b[1])), "counters_equal": a[2] == b[2]}),
          flush=True)
    del x
    torch.cuda.empty_cache()
