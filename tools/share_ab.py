"""Shared draws (gather writes t, k_floyd_pipe reads) vs regenerating A/B (not part of
the product), with labels, roles and counters compared bit for bit.

    python tools/share_ab.py 4 5
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2006_06743_b200 as sng  # noqa: E402
from paper_2006_06743_b200 import synthetic  # noqa: E402

KEYS = ("SNGB_SHARE_T", "SNGB_SHARE_SERIAL", "SNGB_TBUF_MB", "SNGB_SAMPLER_RPB")
variants = [("regenerate", {"SNGB_SHARE_T": "0"}),
            ("share", {}),
            ("share_serial", {"SNGB_SHARE_SERIAL": "1"}),
            ("share_1gb", {"SNGB_TBUF_MB": "1024"}),
            ("share_16gb", {"SNGB_TBUF_MB": "16384"}),
            ("share_rpb8", {"SNGB_SAMPLER_RPB": "8"}),
            ("share_rpb64", {"SNGB_SAMPLER_RPB": "64"}),
            ("share_serial_rpb64_16gb", {"SNGB_SHARE_SERIAL": "1", "SNGB_SAMPLER_RPB": "64", "SNGB_TBUF_MB": "16384"})]
for cfg in [int(c) for c in sys.argv[1:]] or [5]:
    w = synthetic.CONFIGS[cfg]
    x = torch.from_numpy(synthetic.generate(cfg)).cuda()
    outs = {}
    for name, env in variants:
        for k in KEYS:
            os.environ.pop(k, None)
        os.environ.update(env)
        sng.sng_dbscan_device(x, w.eps, w.min_pts, w.rate, w.seed, timing=True)
        runs = [sng.sng_dbscan_device(x, w.eps, w.min_pts, w.rate, w.seed, timing=True) for _ in range(3)]
        lab, rol, gi = runs[-1]
        rec = {"cfg": cfg, "variant": name,
               "ms_total": statistics.median(r[2].ms_total for r in runs),
               "ms_sample": statistics.median(r[2].ms_sample for r in runs),
               "ms_gather": statistics.median(r[2].ms_gather for r in runs),
               "launches": gi.kernel_launches,
               "collisions": gi.collisions, "irregular": gi.irregular_vertices, "edges": gi.edges}
        outs[name] = (lab.cpu(), rol.cpu(), gi.edges, gi.collisions)
        print(json.dumps(rec), flush=True)
    a = outs["regenerate"]
    for name, _ in variants[1:]:
        b = outs[name]
        same = bool(torch.equal(a[0], b[0]) and torch.equal(a[1], b[1]) and a[2:] == b[2:])
        print(json.dumps({"cfg": cfg, "variant": name, "equals_regenerate": same}), flush=True)
    del x
    torch.cuda.empty_cache()
