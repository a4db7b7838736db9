"""k_floyd_lean rows per block on cfg4 in the default step (not part of the product)."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2006_06743_b200 as sng
from paper_2006_06743_b200 import synthetic
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
w = synthetic.CONFIGS[cfg]
x = torch.from_numpy(synthetic.generate(cfg)).cuda()
for pipe in ("0", "1"):
    os.environ["SNGB_FLOYD_PIPE"] = pipe
    for ov in (None, "0"):
        for rpb in ("8", "16", "32", "64", "128"):
            os.environ["SNGB_SAMPLER_RPB"] = rpb
            if ov is None: os.environ.pop("SNGB_OVERLAP", None)
            else: os.environ["SNGB_OVERLAP"] = ov
            sng.sng_dbscan_device(x, w.eps, w.min_pts, w.rate, w.seed, timing=True)
            runs = [sng.sng_dbscan_device(x, w.eps, w.min_pts, w.rate, w.seed, timing=True) for _ in range(5)]
            print(json.dumps({"cfg": cfg, "pipe": pipe, "overlap": ov or "auto", "rpb": rpb,
                              "ms_total": round(statistics.median(r[2].ms_total for r in runs), 3),
                              "ms_sample": round(statistics.median(r[2].ms_sample for r in runs), 3),
                              "ms_gather": round(statistics.median(r[2].ms_gather for r in runs), 3)}), flush=True)
