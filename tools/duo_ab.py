"""k_duo (SNGB_FUSED=3) vs the two kernels A/B (not part of the product), with the
labels, roles and counters compared bit for bit.

    python tools/duo_ab.py 4 5
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2006_06743_b200 as sng  # noqa: E402
from paper_2006_06743_b200 import synthetic  # noqa: E402

variants = [("two_kernels", {"SNGB_FUSED": "0"}),
            ("two_kernels_pipe", {"SNGB_FUSED": "0", "SNGB_FLOYD_PIPE": "1"}),
            ("headpipe", {"SNGB_FUSED": "4"}),
            ("headpipe_g256", {"SNGB_FUSED": "4", "SNGB_FHP_GRAB": "256"})]
if os.environ.get("DUO_AB_DUO"):
    variants.append(("duo", {"SNGB_FUSED": "3"}))
for cfg in [int(c) for c in sys.argv[1:]] or [5]:
    w = synthetic.CONFIGS[cfg]
    x = torch.from_numpy(synthetic.generate(cfg)).cuda()
    outs = {}
    for name, env in variants:
        for k in ("SNGB_FUSED", "SNGB_DUO_SPLIT", "SNGB_DUO_GRAB", "SNGB_FLOYD_PIPE", "SNGB_FHP_GRAB"):
            os.environ.pop(k, None)
        os.environ.update(env)
        sng.sng_dbscan_device(x, w.eps, w.min_pts, w.rate, w.seed, timing=True)
        runs = [sng.sng_dbscan_device(x, w.eps, w.min_pts, w.rate, w.seed, timing=True) for _ in range(3)]
        lab, rol, gi = runs[-1]
        rec = {"cfg": cfg, "variant": name,
               "ms_total": statistics.median(r[2].ms_total for r in runs),
               "ms_sample": statistics.median(r[2].ms_sample for r in runs),
               "ms_gather": statistics.median(r[2].ms_gather for r in runs),
               "collisions": gi.collisions, "irregular": gi.irregular_vertices, "edges": gi.edges}
        outs[name] = (lab.cpu(), rol.cpu(), gi.edges, gi.collisions)
        print(json.dumps(rec), flush=True)
    a = outs["two_kernels"]
    for name, _ in variants[1:]:
        b = outs[name]
        same = bool(torch.equal(a[0], b[0]) and torch.equal(a[1], b[1]) and a[2:] == b[2:])
        print(json.dumps({"cfg": cfg, "variant": name, "equals_two_kernels": same}), flush=True)
    del x
    torch.cuda.empty_cache()
