"""k_floyd_pipe vs k_floyd_lean A/B (not part of the product): the sampler
alone (SNGB_OVERLAP=0: ms_sample) and the default step, with the labels, roles
and counters of both kernels compared bit for bit.

    python tools/pipe_ab.py 4 5
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
    for pipe in ("0", "1"):
        os.environ["SNGB_FLOYD_PIPE"] = pipe
        rec = {"cfg": cfg, "kernel": "k_floyd_pipe" if pipe == "1" else "k_floyd_lean"}
        for ov in ("0", None):
            if ov is None:
                os.environ.pop("SNGB_OVERLAP", None)
            else:
                os.environ["SNGB_OVERLAP"] = ov
            sng.sng_dbscan_device(x, w.eps, w.min_pts, w.rate, w.seed, timing=True)
            runs = [sng.sng_dbscan_device(x, w.eps, w.min_pts, w.rate, w.seed, timing=True) for _ in range(3)]
            tag = "alone" if ov == "0" else "step"
            rec[f"ms_sample_{tag}"] = statistics.median(r[2].ms_sample for r in runs)
            rec[f"ms_gather_{tag}"] = statistics.median(r[2].ms_gather for r in runs)
            rec[f"ms_total_{tag}"] = statistics.median(r[2].ms_total for r in runs)
            lab, rol, gi = runs[-1]
            outs[pipe] = (lab.cpu(), rol.cpu(), gi.edges, gi.collisions, gi.irregular_vertices)
        rec["collisions"] = outs[pipe][3]
        rec["irregular"] = outs[pipe][4]
        print(json.dumps(rec), flush=True)
    a, b = outs["0"], outs["1"]
    same = bool(torch.equal(a[0], b[0]) and torch.equal(a[1], b[1]) and a[2:] == b[2:])
    print(json.dumps({"cfg": cfg, "pipe_equals_lean": same, "edges": a[2]}), flush=True)
    del x
    torch.cuda.empty_cache()
